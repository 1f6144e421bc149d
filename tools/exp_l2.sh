for v in h0 h1; do
  export NTD_LIB_OVERRIDE=$PWD/build/var/libntdgpu_$v.so
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "apply" 2>&1 | tail -1)
  s=$(timeout 300 python tools/batch_scan.py 1,64 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('B%d ntd %.3f iter %.3f' % (d['B'], d['ntd_apply'], d['ms_per_iter']), end=' | ')
    except Exception: pass")
  b=$(timeout 300 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print(round(d['value']), round(d['e2e']['value']))")
  echo "$v :: $r :: $s :: bench $b"
done
unset NTD_LIB_OVERRIDE
cp build/var/libntdgpu_h1.so paper_1909_09771_b200/libntdgpu.so
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:sl::k_apply -c 1 -o gpurun_out/ntd_h1 -f python tools/profile_kernels.py 8 > /dev/null 2>&1; echo ncu rc=$?
