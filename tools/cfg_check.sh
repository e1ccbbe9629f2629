#!/bin/bash
# Per-config profiled build times (device ms per class), bounded by timeouts.
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg5}; do
  echo "== $c ${EG_LIB_PATH:+(lib $EG_LIB_PATH)}"
  EG_PROFILE=1 timeout ${TMO:-300} python tools/run_build.py --config $c --reps 1 2>&1 | grep -E "^profiled|^0 " | tail -2
done
