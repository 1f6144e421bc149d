for v in w16pf4ps8 w16pf2ps8 w24pf2ps4 w24pf1ps4 w32pf1ps4; do
  export NTD_LIB_OVERRIDE=$PWD/build/var/libntdgpu_$v.so
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "ilu0 or combined" 2>&1 | tail -1)
  s=$(timeout 300 python tools/batch_scan.py 1,8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('B%d ilu %.3f iter %.3f' % (d['B'], d['ilu0_apply'], d['ms_per_iter']), end=' | ')
    except Exception: pass")
  b=$(timeout 300 python bench.py --no-cpu-baseline --steps 2 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print(round(d['value']), round(d['e2e']['value']))")
  echo "$v :: $r :: $s :: bench $b"
done
