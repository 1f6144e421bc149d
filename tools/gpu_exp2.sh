for b in 1 64; do for v in p0_t0 p1_t0 p0_t1 p1_t1; do echo "B=$b $v"; for r in 1 2; do ./tools/micro_apply_$v $b | head -1; done; done; done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/batch_scan.py 1,64 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_new.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['apply_ms'], d['roofline']['frac'], d['kernels_ms'], d['iterations'])"
