# auto-planned build of every config: device-side stage times + counts
for c in cfg3 cfg2 cfg1 cfg5 cfg4; do
  timeout 300 python tools/blocks_sweep.py --config $c --blocks auto --reps 2 2>&1 | tail -2
done
