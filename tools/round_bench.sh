#!/bin/bash
# Bench lines of every config + the cfg3 launch list + one full ncu capture
# of the top kernel (each profiled command ran clean without ncu first).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do
  python bench.py --config $c --steps 5 --no-quality > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
EG_REFERENCE_BUDGET_S=60 python bench.py --impl reference --steps 5 > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.err
python tools/run_build.py --config cfg3 --reps 3 > gpurun_out/run_build.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv \
  python tools/run_build.py --config cfg3 --reps 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_msm_group -s 2 -c 1 \
  -o gpurun_out/ncu_msm_group python tools/run_build.py --config cfg3 --reps 2 > gpurun_out/ncu_group.log 2>&1
echo done
