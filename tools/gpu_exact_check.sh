timeout 600 python -m pytest tests/test_exact.py -x -q 2>&1 | tail -15
timeout 300 python tools/recall.py cfg1 2>&1 | tail -2
timeout 600 python tools/recall.py cfg3 --n 200000 2>&1 | tail -2
timeout 900 python tools/recall.py cfg3 2>&1 | tail -2
