#!/bin/bash
# One ncu --set full capture of each step kernel of the headline config (cold, serialised).
TAG=${1:-n}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_probe|k_seg_alloc|PlaceOp|k_lookup_1hot_tma|k_reduce_short|k_long|k_radix_pass|LongRegOp|k_radix_hist" \
  -s 40 -c 10 -o gpurun_out/full_cfg2_${TAG} python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
