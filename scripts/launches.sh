#!/bin/bash
# Per-launch kernel times (ncu timing pass, cold + serialised) for the bench configs.
# Usage (under gpurun): bash scripts/launches.sh TAG [configs...]
TAG=${1:-r1}; shift
CFGS=${@:-cfg2}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_${c}_${TAG}.csv python bench.py --config $c --steps 3 --warmup 3 --pool 1 \
    --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python profiles/summarize_launches.py gpurun_out/launches_${c}_${TAG}.csv > gpurun_out/launches_${c}_${TAG}_summary.txt
done
