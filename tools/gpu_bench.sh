timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; grep step_ms gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null
for c in cfg1 cfg2 cfg4 cfg5; do timeout 900 python bench.py --config $c --no-quality --steps 5 > gpurun_out/bench_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['ms_per_step'],2), d['value'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-quality --e2e-steps 0 --soak-s 0 > /dev/null 2>&1; echo ncu=$?
