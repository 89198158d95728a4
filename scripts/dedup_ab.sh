#!/bin/bash
# A/B: dedup variants (lead / flat / persistent) x pipelined or not. Tag $1.
# env: CFGS (configs), DEDUPS (variants), PIPES ("pipe nopipe"), TESTS=0 to skip the GPU suite.
TAG=${1:-dd}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
for c in ${CFGS:-cfg2 cfg3 cfg5 cfg1}; do
  for d in ${DEDUPS:-lead flat persistent}; do
    for p in ${PIPES:-pipe nopipe}; do
      fl=""; [ "$p" = "pipe" ] && fl="--pipeline"
      f=gpurun_out/bench_${c}_${d}_${p}_${TAG}
      HPS_GPU_DEDUP=$d timeout 400 python bench.py --config $c --no-cpu-baseline $fl > $f.json 2> $f.err
      echo "$c $d $p $(python -c "import json,sys; d=json.loads(open('$f.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,2), 'M/s e2e', round(d['e2e']['value']/1e6,2), d.get('full_batch_n1',{}).get('ms_per_step'))" 2>&1 | tail -1)"
    done
  done
done
for c in ${TRACE:-cfg2}; do
  for p in ${PIPES:-pipe nopipe}; do
    fl=""; [ "$p" = "pipe" ] && fl="--pipeline"
    HPS_GPU_DEDUP=${TRACE_DEDUP:-lead} timeout 400 python bench.py --config $c --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 8 $fl > /dev/null 2> gpurun_out/trace_${c}_${p}_${TAG}.txt; echo "== trace $c $p"; grep "^#" gpurun_out/trace_${c}_${p}_${TAG}.txt
  done
done
