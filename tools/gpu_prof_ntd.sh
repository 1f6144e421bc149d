PROFILE_BATCH=1 python tools/profile_kernels.py 1 > gpurun_out/pk1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_apply -s 1 -c 1 -o gpurun_out/ntd_apply_1sys -f env PROFILE_BATCH=1 python tools/profile_kernels.py 1 > gpurun_out/ncu_ntd1.log 2>&1; echo "ncu rc=$?"
