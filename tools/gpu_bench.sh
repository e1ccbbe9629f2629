for v in "EG_BENCH_CLOCKS=between" "EG_BENCH_CLOCKS=none"; do
env $v timeout 900 python bench.py --no-cpu-baseline --no-quality --e2e-steps 0 --steps 12 2>&1 >/dev/null | grep step_ms | sed "s/^/$v /"
done
