#!/bin/bash
# Tuning sweep of the MSM launch shape on cfg3 (per-class CUDA-event ms).
for t in ${TARGETS:-384 768 1536}; do
  for u in ${UNITS:-4 8 16}; do
    echo "== target=$t units=$u"
    EG_MSM_TARGET=$t EG_MSM_UNITS=$u EG_PROFILE=1 python tools/run_build.py --config ${CFG:-cfg3} --reps 2 2>&1 | grep -E "^profiled|^1 " | tail -2
  done
done
