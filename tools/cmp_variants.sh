#!/bin/bash
# Compare library variants on one config: tools/cmp_variants.sh CFG name1 name2 ...
cfg=$1; shift
for v in "$@"; do
  for i in 1 2; do
    echo "== $v"
    EG_LIB_PATH=$PWD/paper_0904_3151_b200/_native/libeg_$v.so timeout 300 python tools/blocks_sweep.py --config $cfg --blocks auto --reps 3 2>&1 | tail -2
  done
done
