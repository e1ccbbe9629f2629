#!/bin/bash
# Experiment: time the TC projection with parts disabled
# (1 = no epilogue, 2 = no convert, 4 = R once, 8 = no fused fp64 norms)
for f in ${FLAGS:-0 1 4 8 9 12 13}; do
  EG_TC_EXP=$f timeout 120 python tools/tc_proj.py 2>&1 | grep EXP
done
EG_PROJECT_UNFUSED=1 timeout 120 python tools/tc_proj.py 2>&1 | grep EXP | sed 's/^/unfused /'
