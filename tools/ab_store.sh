#!/bin/bash
# A/B: block STORE / V-cycle at C4 (K=2 L=7, 4 blocks) + coupled applies (C2, C4-op, C5-op) per variant
for rep in 1 2; do
  for v in "$@"; do
    s=$(SPK_LIB_PATH=_variants/$v.so K=2 L=7 NB=4 DEG=3 python tools/prof_vcycle.py 2>&1 | grep -E "block STORE|residual |cheb step|V-cycle" | awk '{print $1,$2,$3}' | paste -sd' ')
    c=""
    for cfg in 4,6,3 2,7,4 3,6,3; do
      IFS=, read K L Q <<< "$cfg"
      t=$(SPK_LIB_PATH=_variants/$v.so K=$K L=$L Q=$Q TARGETS=0 python tools/prof_apply.py 2>&1 | grep " us" | awk '{print $5}')
      c="$c k$K:$t"
    done
    echo "$v | $s | $c"
  done
done
