#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
for rep in 1 2; do for k in 2 1; do for c in cfg2 cfg5 cfg1; do HPS_GPU_POOL_CTAS=$k timeout 400 python bench.py --config $c --no-cpu-baseline --steps 30 --e2e-steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ctas $k $c', round(d['ms_per_step']*1000,1), 'e2e', round(d['e2e']['value']/1e6,2))"; done; done; done
