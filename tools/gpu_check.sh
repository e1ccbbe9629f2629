# GPU parity suite + one profiled cfg3 build (the usual iteration check)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/blocks_sweep.py --config ${CFG:-cfg3} --blocks auto --reps 3 | tail -2
