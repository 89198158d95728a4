#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg2 cfg5; do timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e']['value'], d['unique_keys'])"; done
