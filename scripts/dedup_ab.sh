#!/bin/bash
# A/B: flat (3-kernel) vs persistent dedup x pipelined / not. Tag $1.
TAG=${1:-dd}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
for c in cfg2 cfg3 cfg5 cfg1; do
  for d in flat persistent; do
    for p in "" "--no-pipeline"; do
      HPS_GPU_DEDUP=$d timeout 400 python bench.py --config $c --no-cpu-baseline $p > gpurun_out/bench_${c}_${d}${p}_${TAG}.json 2> gpurun_out/bench_${c}_${d}${p}_${TAG}.err
      echo "$c $d $p $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${c}_${d}${p}_${TAG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,2), 'M/s e2e', round(d['e2e']['value']/1e6,2), d.get('full_batch_n1',{}).get('ms_per_step'))" 2>&1 | tail -1)"
    done
  done
done
for p in "" "--no-pipeline"; do
  timeout 400 python bench.py --config cfg2 --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 8 $p > /dev/null 2> gpurun_out/trace_cfg2${p}_${TAG}.txt; grep "^#" gpurun_out/trace_cfg2${p}_${TAG}.txt
done
timeout 400 python bench.py --config cfg3 --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 8 --no-pipeline > /dev/null 2> gpurun_out/trace_cfg3_${TAG}.txt; grep "^#" gpurun_out/trace_cfg3_${TAG}.txt
