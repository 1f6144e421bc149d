python tools/profile_ilu0.py 1 1 hp > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 2 -o gpurun_out/ilu0_hp_cfg1 -f python tools/profile_ilu0.py 1 1 hp > gpurun_out/ncu_hp1.log 2>&1; echo "ncu1 rc=$?"
python tools/profile_ilu0.py 5 1 hp > gpurun_out/p5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 2 -o gpurun_out/ilu0_hp_cfg5 -f python tools/profile_ilu0.py 5 1 hp > gpurun_out/ncu_hp5.log 2>&1; echo "ncu5 rc=$?"
