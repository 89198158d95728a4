#!/bin/bash
# Evidence for profiles/: parity suite, bench lines (headline with CPU baseline + other
# configs + the reference arm), in-graph timelines, per-launch list, and one ncu --set full
# capture of each step kernel. Usage (under gpurun): bash scripts/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_${TAG}.txt
nproc >> gpurun_out/gpu_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/gpu_${TAG}.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_cfg2_${TAG}.json 2> gpurun_out/bench_cfg2_${TAG}.err; tail -1 gpurun_out/bench_cfg2_${TAG}.json | cut -c1-200
for c in cfg3 cfg5 cfg1; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-200
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.json | cut -c1-200
bash scripts/trace.sh ${TAG} cfg2 cfg3 cfg5 cfg1 > /dev/null 2>&1
bash scripts/launches.sh ${TAG} cfg2 cfg3
# step kernels (eager steps: probe, pooling, dedup, ..., short reduce, long reduce)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_probe|k_lookup_1hot_tma|k_dedup|k_reduce_short|k_long<" \
  -s 15 -c 5 -o gpurun_out/full_cfg2_${TAG} python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/ncu_full_${TAG}.log 2>&1
# the roofline kernel: the fused inference lookup (bench's lookup_only leg)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tma<\(bool\)0>" \
  -c 1 -o gpurun_out/full_fwd_cfg2_${TAG} python bench.py --steps 3 --warmup 3 --pool 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/ncu_fwd_${TAG}.log 2>&1
ls gpurun_out | grep ${TAG}
# config 4 (HPS cache) sweeps, f32 and f16 rows
timeout 900 python bench_cache.py --reps 30 > gpurun_out/bench_cfg4_${TAG}.jsonl 2> gpurun_out/bench_cfg4_${TAG}.err
timeout 900 python bench_cache.py --reps 30 --no-cpu --dtype f16 > gpurun_out/bench_cfg4_f16_${TAG}.jsonl 2>&1
tail -1 gpurun_out/bench_cfg4_${TAG}.jsonl | cut -c1-300
