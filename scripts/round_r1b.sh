#!/bin/bash
# Re-entry check of HEAD on one B200: parity suite, smoke, bench lines, launch list, one ncu --set full.
TAG=${1:-r1b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_${TAG}.txt
nproc >> gpurun_out/gpu_${TAG}.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_cfg2_${TAG}.json 2> gpurun_out/bench_cfg2_${TAG}.err; tail -1 gpurun_out/bench_cfg2_${TAG}.json | cut -c1-300
for c in cfg3 cfg5 cfg1; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-200
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.json | cut -c1-200
bash scripts/launches.sh ${TAG} cfg2 cfg3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce_short|k_lookup_1hot|k_radix_pass|k_long" -s 8 -c 4 -o gpurun_out/full_cfg2_${TAG} python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
ls -la gpurun_out
