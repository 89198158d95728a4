#!/bin/bash
# Quick iteration on one B200: parity suite + smoke + headline/cfg3/cfg5 bench lines.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -25 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in cfg2 cfg3 cfg5; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-250
done
bash scripts/launches.sh ${TAG} cfg2 cfg3
for c in cfg2 cfg3; do grep -v "insert\|fill_slots\|gen_keys" gpurun_out/launches_${c}_${TAG}_summary.txt; done
