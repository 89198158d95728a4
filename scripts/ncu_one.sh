#!/bin/bash
# ncu --set full of one kernel (regex $2) from the bench config $3 (default cfg2), tag $1.
TAG=$1; K=$2; C=${3:-cfg2}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 4 -c 1 \
  -o gpurun_out/one_${TAG} python bench.py --config $C --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/ncu_one_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_one_${TAG}.log
