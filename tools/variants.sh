#!/bin/bash
# Compare group-tier compile variants on cfg3 (MSM stage ms)
run() { EG_PROFILE=1 timeout 200 python tools/run_build.py --config cfg3 --reps 1 2>&1 | grep -E "^profiled" | tail -1 | python -c "import sys,re; l=sys.stdin.read(); print(re.findall(r\"'(msm_stage|msm_group)': ([0-9.]+)\", l))"; }
echo "== default"; run
echo "== cap1024 nt128 (target 768)"; EG_MSM_TARGET=768 EG_LIB_PATH=$PWD/paper_0904_3151_b200/_native/libeg_c1024_t128.so run
echo "== cap1024 nt256 (target 768)"; EG_MSM_TARGET=768 EG_LIB_PATH=$PWD/paper_0904_3151_b200/_native/libeg_c1024_t256.so run
echo "== cap2048 nt512"; EG_LIB_PATH=$PWD/paper_0904_3151_b200/_native/libeg_c2048_t512.so run
