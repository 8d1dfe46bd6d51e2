#!/bin/bash
# A/B timing of libspk variants in one GPU session: tools/ab.sh v1 v2 ...  (configs via $CFGS)
CFGS=${CFGS:-"4,6,3 2,7,4 3,6,3"}
for rep in 1 2; do
  for v in "$@"; do
    for c in $CFGS; do
      IFS=, read K L Q <<< "$c"
      r=$(SPK_LIB_PATH=_variants/$v.so K=$K L=$L Q=$Q TARGETS=0 python tools/prof_apply.py 2>&1 | grep " us" | tail -1)
      echo "$v $r"
    done
  done
done
