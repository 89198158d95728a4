#!/bin/bash
# A/B for the multi-hot / narrow-row configs: short-reduce path (register vs cp.async row stream).
mkdir -p gpurun_out
for c in cfg3 cfg1; do
  for m in 0 64 16; do
    for rep in 1 2; do
      HPS_GPU_TMA_MIN_DIM=${m/0/128} timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 --full-batch 0 > gpurun_out/c3_${c}_${m}_${rep}.json 2>/dev/null
      echo "$c tma_min_dim=${m/0/128} rep$rep $(python -c "import json; d=json.loads(open('gpurun_out/c3_${c}_${m}_${rep}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1)"
    done
  done
done
HPS_GPU_TMA_MIN_DIM=64 timeout 300 python -m pytest tests/test_gpu_paths.py -q -p no:cacheprovider -k "dim_sweep or config3 or bulk" 2>&1 | tail -2
