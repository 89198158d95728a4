#!/bin/bash
# Evidence for profiles/: bench line (with CPU baseline), per-launch list, one ncu --set full
# capture of the dominant kernels, device info. Usage (under gpurun): bash scripts/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_${TAG}.txt
nproc >> gpurun_out/gpu_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/gpu_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_cfg2_full_${TAG}.json 2> gpurun_out/bench_cfg2_full_${TAG}.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_cfg2_${TAG}.csv python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce_short|k_lookup_1hot|k_radix_pass" -s 6 -c 3 -o gpurun_out/full_cfg2_${TAG} python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > /dev/null 2>&1
ls -la gpurun_out
