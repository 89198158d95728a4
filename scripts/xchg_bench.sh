#!/bin/bash
# Exchange paths on one GPU (NCCL world of one): distributed / hybrid (cfg2), localized (cfg3).
for spec in "cfg2 distributed" "cfg2 hybrid" "cfg3 localized" "cfg5 distributed"; do
  set -- $spec
  echo -n "$1 $2: "
  timeout 900 python bench.py --config $1 --placement $2 --force-exchange --steps 10 --warmup 3 --no-cpu-baseline \
    2> gpurun_out/xchg_$1_$2.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step', round(d['value']/1e6,2), 'M/s', d['config']['parallelism'], 'xbytes', d.get('nvlink',{}).get('bytes_per_step_rank0'))" || tail -5 gpurun_out/xchg_$1_$2.err
done
