#!/bin/bash
# compute-sanitizer over the step kernels (small shapes). Tag $1.
TAG=${1:-s}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 3 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke_${TAG}.log 2>&1; echo "memcheck smoke rc=$?"; tail -3 gpurun_out/memcheck_smoke_${TAG}.log
timeout 1200 $CS --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_table.py -q -x -p no:cacheprovider -k "skewed or multi_hot or one_hot or insert_on_miss" > gpurun_out/memcheck_table_${TAG}.log 2>&1; echo "memcheck table rc=$?"; tail -3 gpurun_out/memcheck_table_${TAG}.log
timeout 1200 $CS --tool racecheck --error-exitcode 3 python -m pytest tests/test_gpu_table.py -q -x -p no:cacheprovider -k "skewed and sgd" > gpurun_out/racecheck_table_${TAG}.log 2>&1; echo "racecheck table rc=$?"; tail -3 gpurun_out/racecheck_table_${TAG}.log
timeout 1200 $CS --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_cache.py -q -x -p no:cacheprovider > gpurun_out/memcheck_cache_${TAG}.log 2>&1; echo "memcheck cache rc=$?"; tail -3 gpurun_out/memcheck_cache_${TAG}.log
timeout 1200 $CS --tool racecheck --error-exitcode 3 python -m pytest tests/test_gpu_cache.py -q -x -p no:cacheprovider -k "randomized and 256-8-0 or read_through" > gpurun_out/racecheck_cache_${TAG}.log 2>&1; echo "racecheck cache rc=$?"; tail -3 gpurun_out/racecheck_cache_${TAG}.log
