#!/bin/bash
# cfg3 MSM-stage sweep over units per batch (two-stream default).
for u in ${UNITS:-8 12 16}; do
  echo "== units=$u"
  EG_MSM_UNITS=$u EG_PROFILE=1 timeout 200 python tools/run_build.py --config ${CFG:-cfg3} --reps 1 2>&1 | grep -E "^profiled" | tail -1 | python -c "import sys,re; l=sys.stdin.read(); print(re.findall(r\"'(msm_stage|msm_scatter|msm_group|msm_hist)': ([0-9.]+)\", l))"
done
