timeout 300 python tools/blocks_sweep.py --config cfg3 --blocks 12,auto,6,7,8,9,10,16
timeout 200 python tools/blocks_sweep.py --config cfg2 --blocks 8,auto,3,4,5,6,10
timeout 300 python tools/blocks_sweep.py --config cfg4 --blocks 16,auto,3,4,6,8,12 --reps 1
timeout 400 python tools/blocks_sweep.py --config cfg5 --blocks 16,auto,6,8,10,12 --reps 1
timeout 100 python tools/blocks_sweep.py --config cfg1 --blocks 8,auto,4,6
