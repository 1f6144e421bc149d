for p in auto skew hp:2:16 hp:4:8 hp:8:4 hp:2:12; do timeout 300 python tools/batch_variants.py $p 64; done
for p in auto skew hpmin; do timeout 300 python tools/batch_variants.py $p 8; done
