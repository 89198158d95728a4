#!/bin/bash
# Batch-pipelining iteration: prefetch parity tests, full GPU suite, bench lines + timelines.
TAG=${1:-p}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefetch.py -x -q -p no:cacheprovider > gpurun_out/pytest_prefetch_${TAG}.log 2>&1; tail -25 gpurun_out/pytest_prefetch_${TAG}.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
for c in cfg2 cfg3 cfg5 cfg1; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-300; tail -3 gpurun_out/bench_${c}_${TAG}.err
done
bash scripts/trace.sh ${TAG} cfg2 cfg3
