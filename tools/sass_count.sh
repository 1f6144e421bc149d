#!/bin/bash
# Instruction mix of sl::k_apply<K,D> in an object file (offline proxy for the line-step cost).
# usage: tools/sass_count.sh obj.o [K] [D]
K=${2:-3}; D=${3:-7}
cuobjdump -sass -fun "_ZN2sl7k_applyILi${K}ELi${D}EEEvPKdS2_PdS3_S2_iiiPKi" $1 | grep -E "^\s+/\*[0-9a-f]{4,}\*/" | \
 sed -E 's#^\s+/\*[0-9a-f]+\*/\s+##; s#^@!?U?P[0-9T]+\s+##' | awk '{split($1,a,"."); c[a[1]]++; n++} END {printf "total %d\n", n; for (k in c) printf "%s %d\n", k, c[k]}' | sort -k2 -n -r | head -22 | tr '\n' ' '; echo
