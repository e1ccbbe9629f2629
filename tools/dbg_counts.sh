# repeated builds: counts must be identical run to run and across block counts
for b in 7 6 8; do EG_MSM_BLOCKS=$b timeout 200 python tools/run_build.py --config cfg3 --reps 4 2>&1 | grep -E "^[0-9] " | cut -c1-150; done
for c in cfg5 cfg2; do timeout 300 python tools/run_build.py --config $c --reps 3 2>&1 | grep -E "^[0-9] " | cut -c1-150; done
