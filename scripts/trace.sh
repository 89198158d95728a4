#!/bin/bash
# In-graph kernel timelines for the bench configs (bench.py --trace), tag $1.
TAG=${1:-t}; shift
CFGS=${@:-cfg2 cfg3}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 8 > gpurun_out/trace_${c}_${TAG}.json 2> gpurun_out/trace_${c}_${TAG}.txt
  echo "== $c"; tail -1 gpurun_out/trace_${c}_${TAG}.json | cut -c1-160; grep "^#" gpurun_out/trace_${c}_${TAG}.txt
done
