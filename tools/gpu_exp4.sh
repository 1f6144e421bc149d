timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for G in 4 8; do NTD_STREAM_GROUPS=$G timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$G.json 2> gpurun_out/bench_g$G.err; echo "G=$G rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_g$G.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['apply_ms'], d['roofline']['frac'], d['kernels_ms'], d['iterations'])"; done
