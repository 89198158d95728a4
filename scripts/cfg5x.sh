#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
for cfg in "38 2" "80 1" "100 1" "60 1"; do set -- $cfg; for c in cfg5 cfg2; do HPS_GPU_TMA_ROWS=$1 HPS_GPU_RED_WAVES=$2 timeout 400 python bench.py --config $c --no-cpu-baseline --steps 30 --e2e-steps 4 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('rows $1 waves $2 $c', round(d['ms_per_step']*1000,1))"; done; done
