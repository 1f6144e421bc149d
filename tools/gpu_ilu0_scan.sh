timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ilu0 or mappings or combined or golden or reduction" > gpurun_out/pytest_ilu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_ilu.log
for c in "3 1" "4 1" "5 1"; do timeout 300 python tools/ilu0_hp_scan.py $c; done > gpurun_out/ilu0_hp_scan.txt 2>&1; cat gpurun_out/ilu0_hp_scan.txt
