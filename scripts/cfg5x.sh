#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
for rep in 1 2; do for w in 512 1024 2048 256; do for c in cfg1; do HPS_GPU_DEDUP_PER_CTA=$w timeout 400 python bench.py --config $c --no-cpu-baseline --steps 30 --e2e-steps 4 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('per_cta $w $c', round(d['ms_per_step']*1000,1))"; done; done; done
