for v in w16 w32; do
  export NTD_LIB_OVERRIDE=$PWD/build/var/libntdgpu_$v.so
  r=$(timeout 300 python tools/ilu0_check.py 2>&1 | tail -1)
  s=$(timeout 300 python tools/batch_scan.py 1,8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('B%d ilu %.3f iter %.3f' % (d['B'], d['ilu0_apply'], d['ms_per_iter']), end=' | ')
    except Exception: pass")
  echo "$v :: $r :: $s"
done
