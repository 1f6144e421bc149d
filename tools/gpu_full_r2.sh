timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python tools/phase_timing.py 64 > gpurun_out/phase64.txt 2>&1; cat gpurun_out/phase64.txt
timeout 300 python tools/phase_timing.py 8 > gpurun_out/phase8.txt 2>&1; cat gpurun_out/phase8.txt
