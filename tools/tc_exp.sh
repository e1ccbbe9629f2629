#!/bin/bash
# Experiment: time the TC projection with parts disabled (1=no epilogue, 2=no convert, 4=R once)
for f in 0 1 2 4 7; do
  echo "== EG_TC_EXP=$f"
  EG_TC_EXP=$f timeout 60 python tools/tc_proj.py 2>&1 | tail -1
done
