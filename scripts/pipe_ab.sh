#!/bin/bash
# A/B: pipelined vs unpipelined steps, all training configs. Tag $1.
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefetch.py -x -q -p no:cacheprovider > gpurun_out/pytest_prefetch_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_prefetch_${TAG}.log
for c in cfg2 cfg3 cfg5 cfg1; do
  for p in "" "--no-pipeline"; do
    timeout 400 python bench.py --config $c --no-cpu-baseline $p > gpurun_out/bench_${c}${p}_${TAG}.json 2> gpurun_out/bench_${c}${p}_${TAG}.err
    echo "$c $p $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${c}${p}_${TAG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,2), 'M/s e2e', round(d['e2e']['value']/1e6,2), d.get('full_batch_n1',{}).get('ms_per_step'))" 2>&1 | tail -1)"
  done
done
bash scripts/trace.sh ${TAG} cfg2 cfg3 > /dev/null 2>&1; grep "^#" gpurun_out/trace_cfg2_${TAG}.txt gpurun_out/trace_cfg3_${TAG}.txt
