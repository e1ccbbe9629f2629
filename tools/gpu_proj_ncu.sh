# projection-only timing (ring variants) + projection parity subset
timeout 600 python -m pytest tests -m gpu -x -q -k "projection or fused or tc_" 2>&1 | tail -4
for v in "2 8" "3 8" "2 3"; do set -- $v; EG_H16_OSLOTS=$1 EG_H16_XSLOTS=$2 timeout 300 python tools/tc_proj.py 2>&1 | tail -1 | sed "s/^/o=$1 x=$2 /"; done
for e in 1 4 16; do EG_TC_EXP=$e timeout 300 python tools/tc_proj.py 2>&1 | tail -1; done
