timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q -k "ilu0 or mappings or golden or batch or config3" > gpurun_out/pytest_skew.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_skew.log
for c in "4 1" "4 8" "4 64"; do QUICK=0 timeout 300 python tools/ilu0_hp_scan.py $c 2>&1 | grep "skew\|cfg"; done
timeout 300 python tools/batch_variants.py skew 64
timeout 300 python tools/batch_variants.py auto 64
