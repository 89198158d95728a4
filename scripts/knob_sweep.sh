#!/bin/bash
# A/B knob sweep on one B200 (config $CFG, default cfg2): pooling CTAs/SM x dedup variant,
# short-reduce row-stream depth. One bench line each (3 repeats of the step timing).
TAG=${1:-ks}
CFG=${CFG:-cfg2}
mkdir -p gpurun_out
run() {
  local name=$1; shift
  for rep in 1 2; do
    env "$@" timeout 300 python bench.py --config $CFG --no-cpu-baseline --e2e-steps 2 --full-batch 0 > gpurun_out/ks_${name}_${rep}.json 2>/dev/null
    echo "$name rep$rep $(python -c "import json; d=json.loads(open('gpurun_out/ks_${name}_${rep}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1)"
  done
}
for d in persistent flat; do
  for p in 1 2 4; do run ${d}_pool$p HPS_GPU_DEDUP=$d HPS_GPU_POOL_CTAS=$p; done
done
for u in 8 16; do run pipeU$u HPS_GPU_PIPE_U=$u; done
run nopdl HPS_GPU_NO_PDL=1
