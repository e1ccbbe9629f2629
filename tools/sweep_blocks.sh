# device time of the MSM stage per forced block count (tools/blocks_sweep.py)
timeout 300 python tools/blocks_sweep.py --config cfg3 --blocks auto,6,7,8,9,10 --reps 3 | grep blocks=
timeout 200 python tools/blocks_sweep.py --config cfg2 --blocks auto,3,4,5 --reps 3 | grep blocks=
timeout 400 python tools/blocks_sweep.py --config cfg5 --blocks auto,4,5,6,7 --reps 1 | grep blocks=
timeout 400 python tools/blocks_sweep.py --config cfg4 --blocks auto,3,4 --reps 1 | grep blocks=
