#!/bin/bash
# time K3 of every tools/diag/sweep/lib_*.so variant on a config: time_variants.sh CONFIG [names...]
cfg=${1:-C2}; shift
names=("$@")
if [ ${#names[@]} -eq 0 ]; then names=($(ls tools/diag/sweep/ | sed -n 's/^lib_\(.*\)\.so$/\1/p')); fi
for n in "${names[@]}"; do
  timeout 300 python tools/diag/sweep_time.py tools/diag/sweep/lib_$n.so $cfg 2>&1 | tail -1
done
