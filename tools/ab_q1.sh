#!/bin/bash
for rep in 1 2; do for v in "$@"; do
  s=$(SPK_LIB_PATH=_variants/$v.so K=3 L=6 NB=1 DEG=3 python tools/prof_vcycle.py 2>&1 | grep -E "block STORE|residual |cheb step|V-cycle" | awk '{print $1,$2,$3}' | paste -sd' ')
  s2=$(SPK_LIB_PATH=_variants/$v.so K=2 L=7 NB=1 DEG=3 python tools/prof_vcycle.py 2>&1 | grep -E "block STORE|V-cycle" | awk '{print $1,$2,$3}' | paste -sd' ')
  echo "$v | k3: $s | k2: $s2"
done; done
