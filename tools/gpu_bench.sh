timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in 1 8; do timeout 600 python tools/rank_sim.py --world $w --ranks 2 2>&1 | grep world=; done
timeout 900 python bench.py --no-cpu-baseline --no-quality --e2e-steps 0 --steps 12 2> gpurun_out/b.err > gpurun_out/b.json; grep step_ms gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], d['parity']['match'])"
