#!/bin/bash
# DRAM traffic per stage (ncu metrics) for every config -> gpurun_out/r2_traffic.json
for c in cfg1:20000 cfg2:10500000 cfg3:1600000 cfg4:4000000 cfg5:20000000; do
  cfg=${c%%:*}; n=${c##*:}
  python tools/run_build.py --config $cfg --reps 2 > /dev/null 2>&1 || continue
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/traffic_$cfg.csv python tools/run_build.py --config $cfg --reps 2 > /dev/null 2>&1
  python tools/traffic.py $cfg $n gpurun_out/traffic_$cfg.csv gpurun_out/r2_traffic.json
done
