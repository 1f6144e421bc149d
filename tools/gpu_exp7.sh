timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_gpu.log
for G in 8 16; do NTD_STREAM_GROUPS=$G timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$G.json 2>&1; echo "B64 G=$G $(python -c "
import json; d=json.load(open('gpurun_out/bench_g$G.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'])")"; done
for G in 1 2 4 8; do NTD_STREAM_GROUPS=$G timeout 600 python bench.py --systems 8 --no-cpu-baseline > gpurun_out/bench_b8g$G.json 2>&1; echo "B8 G=$G $(python -c "
import json; d=json.load(open('gpurun_out/bench_b8g$G.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'])")"; done
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"; cat gpurun_out/bench_cfg5.json; tail -3 gpurun_out/bench_cfg5.err
