#!/bin/bash
# Round-2 final evidence on one B200: the standard evidence script (GPU suite, smoke, probe A/B,
# per-step ncu traffic, bench lines, traces, launch lists) + config-4 cache sweep + the
# three-tier miss-path bench.
TAG=${1:-r2i}
bash scripts/round2_evidence.sh $TAG
timeout 900 python bench_cache.py --reps 30 --no-cpu > gpurun_out/bench_cfg4_${TAG}.jsonl 2>&1; tail -2 gpurun_out/bench_cfg4_${TAG}.jsonl | cut -c1-300
timeout 600 python scripts/bench_tiered.py > gpurun_out/bench_tiered_${TAG}.jsonl 2> gpurun_out/bench_tiered_${TAG}.err; cat gpurun_out/bench_tiered_${TAG}.jsonl | cut -c1-200
