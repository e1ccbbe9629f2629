#!/bin/bash
# MSM stage of every config under the previous round's block count and under the
# plan's own choice (digests must agree): python tools/msm_bench.py per line.
for cfg in cfg3 cfg5 cfg2 cfg4; do
  case $cfg in cfg3) old=7;; cfg5) old=5;; cfg2) old=3;; cfg4) old=3;; esac
  for b in $old 0; do timeout 900 python tools/msm_bench.py --config $cfg --blocks $b --iters 4 2>&1 | tail -2 | head -1 | cut -c1-150; done
done
