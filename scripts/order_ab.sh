#!/bin/bash
# A/B: dedup beside the pooling (default) vs dedup first on the main stream, x dedup variant.
TAG=${1:-oa}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
HPS_GPU_DEDUP_FIRST=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_first_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_first_${TAG}.log
fi
for c in ${CFGS:-cfg2 cfg3 cfg5 cfg1}; do
  for first in 0 1; do for d in persistent flat; do
    for rep in 1 2; do
      HPS_GPU_DEDUP_FIRST=$first HPS_GPU_DEDUP=$d timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 --full-batch 0 > gpurun_out/oa_${c}_${first}_${d}_${rep}.json 2>/dev/null
      echo "$c first=$first $d rep$rep $(python -c "import json; d=json.loads(open('gpurun_out/oa_${c}_${first}_${d}_${rep}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1)"
    done
  done; done
done
HPS_GPU_DEDUP_FIRST=1 HPS_GPU_DEDUP=flat timeout 300 python bench.py --config cfg2 --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 8 --full-batch 0 > /dev/null 2> gpurun_out/trace_first_${TAG}.txt; grep "^#" gpurun_out/trace_first_${TAG}.txt
