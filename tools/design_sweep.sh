#!/bin/bash
# MSM stage of one config under the complete design and the table's covering
# designs (plan codes 10000 + 100 v + m); digests must agree.
CFG=${CFG:-cfg3}
for b in ${PLANS:-7 10804 10904 11004 11105 11205 0}; do
  timeout 600 python tools/msm_bench.py --config $CFG --blocks $b --iters 6 2>&1 | tail -2
done
