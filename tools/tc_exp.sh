#!/bin/bash
# Experiment: time the TC projection with parts disabled (1=no epilogue, 2=no convert, 4=R once)
for f in 0 1 2 4 3 5 6 7; do
  EG_TC_EXP=$f timeout 120 python tools/tc_proj.py 2>&1 | grep EXP
done
