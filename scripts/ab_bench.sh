#!/bin/bash
# A/B: bench lines with and without an env toggle. Usage: bash scripts/ab_bench.sh ENVVAR cfg...
VAR=$1; shift
for c in "$@"; do
  for v in 0 1; do
    echo -n "$c $VAR=$v "
    env $VAR=$v timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step', round(d['e2e']['value']/1e6,2), 'M e2e', round(d['roofline']['kernel_ms']*1000,1), 'us lookup')"
  done
done
