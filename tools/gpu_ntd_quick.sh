timeout 900 python -m pytest tests/test_gpu_parity_more.py -x -q -k "line_width or config4_system0" > gpurun_out/pytest_ntd.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ntd.log
for c in "1 1" "2 1" "3 1" "4 1" "4 8" "4 64" "5 1"; do timeout 300 python tools/ntd_time.py $c; done
