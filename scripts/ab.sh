#!/bin/bash
# Generic A/B on one B200: AB_CFGS configs x variants ("name:ENV=V,ENV2=V2" or "name:" for
# the default), AB_REPS repeats each, interleaved; prints the step time of each run.
CFGS=${AB_CFGS:-cfg2}
REPS=${AB_REPS:-3}
mkdir -p gpurun_out
for cfg in $CFGS; do
  for rep in $(seq 1 $REPS); do
    for v in "$@"; do
      name=${v%%:*}; envs=${v#*:}
      out=gpurun_out/ab_${cfg}_${name}_${rep}.json
      env ${envs//,/ } timeout 300 python bench.py --config $cfg --steps ${AB_STEPS:-20} --no-cpu-baseline --e2e-steps ${AB_E2E:-2} --full-batch 0 > $out 2>/dev/null
      echo "$cfg $name rep$rep $(python -c "import json; d=json.loads(open('$out').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,1), 'us', 'e2e', round(d['e2e']['value']/1e6,1))" 2>&1 | tail -1)"
    done
  done
done
