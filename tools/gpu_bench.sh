for lp in 8 4; do for c in cfg4 cfg5; do EG_VERIFY_LP=$lp timeout 900 python bench.py --config $c --no-cpu-baseline --no-quality --e2e-steps 0 --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('lp=$lp $c', round(d['ms_per_step'],2), round(d['stage_ms'].get('verify',0),2), d['counts']['edges'])"; done; done
EG_VERIFY_LP=4 timeout 900 python -m pytest tests -m gpu -x -q -k "cfg or exact or small" 2>&1 | tail -2
