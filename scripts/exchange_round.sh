#!/bin/bash
# The multi-GPU placements on one B200 (NCCL world of one: the exchange code path runs end
# to end; all-to-alls are local). Tag $1.
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.log
for pl in distributed hybrid; do
  timeout 600 python bench.py --config cfg2 --placement $pl --force-exchange --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2_${pl}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_cfg2_${pl}_${TAG}.json | cut -c1-260
done
timeout 600 python bench.py --config cfg3 --placement localized --force-exchange --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg3_localized_${TAG}.json 2>&1; tail -1 gpurun_out/bench_cfg3_localized_${TAG}.json | cut -c1-260
timeout 600 python bench.py --config cfg5 --placement distributed --force-exchange --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg5_distributed_${TAG}.json 2>&1; tail -1 gpurun_out/bench_cfg5_distributed_${TAG}.json | cut -c1-260
