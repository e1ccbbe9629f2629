#!/bin/bash
# MSM-stage variants on one config: tools/msm_cmp.sh cfg3 "lib1 lib2 ..." ["ENV=.. ENV2=.."]
c=${1:-cfg3}; libs=${2:-libepsgraph_b200}; L=$PWD/paper_0904_3151_b200/_native
for v in $libs; do
  echo "-- $v"; EG_LIB_PATH=$L/$v.so timeout 300 python tools/msm_bench.py --config $c --iters 8 2>&1 | tail -3
done
shift 2
for e in "$@"; do
  echo "-- env $e"; env $e timeout 300 python tools/msm_bench.py --config $c --iters 8 2>&1 | tail -3
done
