for v in un1 un2 un4; do
  export NTD_LIB_OVERRIDE=$PWD/build/var/libntdgpu_$v.so
  b=$(timeout 300 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print(round(d['value']), round(d['e2e']['value']), {k:round(v['frac'],3) for k,v in d['stencil_roofline'].items()}, d['iterations']['within_1_of_reference'])")
  echo "$v :: $b"
done
