# Round-2 evidence: latencies, bench, launch list, ncu of the NTD and ILU0 sweeps as the bench launches them.
./tools/micro_lat2.bin > gpurun_out/micro_lat2.txt 2>&1; ./tools/micro_tput2.bin > gpurun_out/micro_tput2.txt 2>&1; ./tools/micro_line_ts.bin > gpurun_out/micro_line_ts.txt 2>&1; cat gpurun_out/micro_lat2.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
PROFILE_BATCH=64 timeout 300 python tools/profile_kernels.py 4 > gpurun_out/pk4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ts::k_apply -s 1 -c 1 -o gpurun_out/ntd_apply_batch4 -f env PROFILE_BATCH=64 python tools/profile_kernels.py 4 > gpurun_out/ncu_ntd4.log 2>&1; echo "ncu ntd rc=$?"
PROFILE_BATCH=64 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:skew::k_apply -s 1 -c 1 -o gpurun_out/ilu0_apply_batch4 -f env PROFILE_BATCH=64 python tools/profile_kernels.py 4 > gpurun_out/ncu_ilu4.log 2>&1; echo "ncu ilu rc=$?"
