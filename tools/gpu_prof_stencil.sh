timeout 300 python tools/profile_stencil_single.py 5 > gpurun_out/ps5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_spmv_dot|k_true_res" -s 2 -c 2 -o gpurun_out/stencil_single5 -f python tools/profile_stencil_single.py 5 > gpurun_out/ncu_st5.log 2>&1; echo "ncu rc=$?"
