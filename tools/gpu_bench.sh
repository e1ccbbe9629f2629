timeout 900 python bench.py --config cfg4 --no-cpu-baseline --no-quality --e2e-steps 0 --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python tools/run_build.py --config cfg4 --reps 1 > /dev/null 2>&1; echo ncu=$?
