timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for c in cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-quality --e2e-steps 0 --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), round(d['stage_ms']['msm_stage'],3), d['counts']['edges'], (d.get('parity') or {}).get('match'))"; done
for w in 8; do timeout 600 python tools/rank_sim.py --world $w --ranks 1 2>&1 | grep world=; done
