for kb in 128 160 212; do EG_HIST_SMEM_KB=$kb timeout 900 python bench.py --no-cpu-baseline --no-quality --e2e-steps 0 --steps 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('kb=$kb', round(d['ms_per_step'],3), round(d['stage_ms']['msm_stage'],3), d['parity']['match'])"; done
