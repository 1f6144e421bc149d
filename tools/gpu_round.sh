# Round check on one B200: GPU tests, smoke, bench (+ reference arm), launch list, ncu of the NTD apply.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -2 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ts::k_apply -c 1 -o gpurun_out/ntd_apply_full -f python tools/profile_kernels.py ${PROFILE_SYSTEMS:-4} > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:skew::k_apply -c 1 -o gpurun_out/ilu0_apply_full -f python tools/profile_kernels.py ${PROFILE_SYSTEMS:-4} > gpurun_out/ncu_full_ilu0.log 2>&1; echo "ncu3 rc=$?"
timeout 300 python tools/phase_timing.py 64 > gpurun_out/phase_timing.txt 2>&1; echo "phase rc=$?"; cat gpurun_out/phase_timing.txt
