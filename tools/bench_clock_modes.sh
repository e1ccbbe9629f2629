# step-time jitter under different host settings (cfg3, 20 steps)
for v in "EG_BENCH_CLOCKS=between" "EG_BENCH_CLOCKS=between PYTHONGC=off" "EG_BENCH_CLOCKS=off" "EG_BENCH_CLOCKS=between CUDA_DEVICE_MAX_CONNECTIONS=32"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 > /tmp/b.json 2> /tmp/b.err
  echo "== $v $(python -c "import json; d=json.load(open('/tmp/b.json')); print(round(d['ms_per_step'],2), d['clocks'])")"
  grep -E "step_ms" /tmp/b.err
done
nproc; uptime; ps aux --sort=-%cpu | head -8
