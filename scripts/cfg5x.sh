#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
for k in 4 2 1 8; do HPS_GPU_POOLM_CTAS=$k timeout 400 python bench.py --config cfg3 --no-cpu-baseline --steps 20 --e2e-steps 4 --trace 4 2>&1 | grep "pool \|count \|place\|reduce_short\|^{" | cut -c1-130 | sed "s/^/ctas $k /"; done
