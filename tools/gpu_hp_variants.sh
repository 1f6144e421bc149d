for lib in "" build/var/libntdgpu_nozf.so build/var/libntdgpu_noout.so build/var/libntdgpu_none.so; do
  echo "== variant ${lib:-base}"
  for c in "1 1" "4 1" "5 1"; do VARIANT_LIB=$lib QUICK=1 timeout 300 python tools/ilu0_hp_scan.py $c 2>&1 | tail -2; done
done
