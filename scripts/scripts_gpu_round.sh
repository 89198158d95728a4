#!/bin/bash
# One GPU round: parity tests, bench lines for cfg2 (headline) / cfg3 / cfg1, and ncu launch lists.
# Usage (under gpurun): bash scripts_gpu_round.sh TAG
TAG=${1:-r}
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
for c in cfg2 cfg3 cfg1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/bench_${c}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-400
done
for c in cfg2 cfg3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|k_" --csv --log-file gpurun_out/launches_${c}_${TAG}.csv python bench.py --config $c --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
