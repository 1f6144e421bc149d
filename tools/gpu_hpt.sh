VARIANT_LIB=build/var/libntdgpu_hpt.so timeout 120 python tools/hp_timing.py 1
VARIANT_LIB=build/var/libntdgpu_hpt.so timeout 120 python tools/hp_timing.py 4 48 3
