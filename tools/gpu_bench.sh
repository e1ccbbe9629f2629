timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-quality --e2e-steps 0 --steps 12 2> gpurun_out/b.err > gpurun_out/b.json; grep step_ms gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['match'])"
