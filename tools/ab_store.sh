#!/bin/bash
# A/B: block STORE at C4 (K=2 L=7 4 blocks) + coupled applies (C2, C4-op, C5-op) for libspk variants
for rep in 1 2; do
  for v in "$@"; do
    s=$(SPK_LIB_PATH=_variants/$v.so K=2 L=7 NB=4 DEG=3 python tools/prof_vcycle.py 2>&1 | grep -E "block STORE|V-cycle" | awk '{print $1,$2,$3}' | paste -sd' ')
    c=""
    for cfg in "4 6 3" "2 7 4" "3 6 3"; do
      set -- $cfg
      t=$(SPK_LIB_PATH=_variants/$v.so K=$1 L=$2 Q=$3 TARGETS=0 python tools/prof_apply.py 2>&1 | grep " us" | awk '{print $5}')
      c="$c k$1:$t"
      set -- "$@"
    done
    echo "$v | $s | $c"
  done
done
