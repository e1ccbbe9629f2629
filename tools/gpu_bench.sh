timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 12 2> gpurun_out/b.err > gpurun_out/b.json; grep step_ms gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['match'], d['quality']['recall'])"
for c in cfg4 cfg5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-quality --e2e-steps 0 --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()}, d['counts']['edges'])"; done
