timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_more.py -x -q -k "reduction or relres or config4 or golden or stencil" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_q.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
PROFILE_BATCH=64 timeout 300 python tools/profile_kernels.py 4 > gpurun_out/pk4.log 2>&1 && \
PROFILE_BATCH=64 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:skew::k_apply -s 1 -c 1 -o gpurun_out/ilu0_apply_batch4 -f env PROFILE_BATCH=64 python tools/profile_kernels.py 4 > gpurun_out/ncu_ilu4.log 2>&1; echo "ncu ilu rc=$?"
