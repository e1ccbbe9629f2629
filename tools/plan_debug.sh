for c in cfg3 cfg2 cfg5 cfg4; do EG_PLAN_DEBUG=1 timeout 400 python tools/blocks_sweep.py --config $c --blocks auto --reps 2 2>&1 | grep -E "eg_msm_plan|blocks=" | sort | uniq | head -30; done
