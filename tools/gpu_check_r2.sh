# Round-2 check on one B200: GPU tests, smoke, bench (N=1 with configs), self-launched 2-rank bench on one GPU.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$TWO_RANK" ]; then
NTD_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err; echo "bench w2 rc=$?"; tail -c 600 gpurun_out/bench_w2.json; grep -c "NCCL\|rank" gpurun_out/bench_w2.err
fi
