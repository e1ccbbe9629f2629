timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; grep step_ms gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['quality']['recall'], {k: round(v,3) for k,v in d['stage_ms'].items()})"
