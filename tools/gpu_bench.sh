timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --config cfg1 --no-cpu-baseline --no-quality --e2e-steps 0 --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['ms_per_step'],3))"
