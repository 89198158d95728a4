#!/bin/bash
# Iteration loop on one B200: parity suite + smoke + in-graph timelines + bench lines. Tag $1.
TAG=${1:-i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/trace.sh ${TAG} cfg2 cfg3 cfg5
HPS_GPU_NO_FORK=1 bash scripts/trace.sh ${TAG}_nofork cfg2
