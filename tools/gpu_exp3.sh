for b in 1 64; do for v in pf0 pf2 pf4; do echo "B=$b $v"; for r in 1 2; do ./tools/micro_apply_$v $b | head -1; done; done; done
for v in tpf0 tpf2; do echo "timing $v"; ./tools/micro_apply_$v 1; done
