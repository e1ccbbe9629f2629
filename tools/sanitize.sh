#!/bin/bash
# compute-sanitizer over the kernel families (summaries -> gpurun_out/sanitize_*.log)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for w in cfg1 cfg3_small tiers exact; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_run.py $w > gpurun_out/sanitize_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${w}.log | tail -1)"
  done
done
