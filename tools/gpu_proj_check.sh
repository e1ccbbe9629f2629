# full GPU parity suite + bench line (no CPU baseline) + projection band print
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -m pytest tests -m gpu -q -s -k "tc_projection_error_band" 2>&1 | grep "tc band" | head -8
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_h16.json 2>gpurun_out/bench_h16.err; tail -2 gpurun_out/bench_h16.err; python -c "
import json; d=json.load(open('gpurun_out/bench_h16.json')); print(d['ms_per_step'], {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['match'])"
