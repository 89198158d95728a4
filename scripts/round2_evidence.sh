#!/bin/bash
# Round-2 evidence on one B200: GPU suite, smoke, probe A/B, per-step ncu DRAM traffic of the
# training configs, bench lines (headline with CPU baseline + others), launch lists, timelines.
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout 600 python scripts/probe_ab.py > gpurun_out/probe_ab_${TAG}.jsonl 2> gpurun_out/probe_ab_${TAG}.err; cat gpurun_out/probe_ab_${TAG}.jsonl
for c in ${STEP_CFGS:-cfg2 cfg3 cfg5}; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_" --csv --log-file gpurun_out/step_${c}_${TAG}.csv python scripts/profile_step.py $c 3 > /dev/null 2>&1
  python profiles/step_traffic.py gpurun_out/step_${c}_${TAG}.csv $(python -c "
import sys; sys.path.insert(0,'.'); from paper_2210_08803_b200 import workload as W; print({'cfg1':W.config1,'cfg2':W.config2,'cfg3':W.config3,'cfg5':W.config5}['$c']().name)") gpurun_out/ncu_step_traffic_${TAG}.json
done
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py > gpurun_out/bench_cfg2_${TAG}.json 2> gpurun_out/bench_cfg2_${TAG}.err; tail -1 gpurun_out/bench_cfg2_${TAG}.json | cut -c1-300
for c in cfg3 cfg5 cfg1; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2>&1; tail -1 gpurun_out/bench_${c}_${TAG}.json | cut -c1-200
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.json | cut -c1-200
timeout 400 python bench.py --config cfg2 --no-cpu-baseline --force-exchange --placement distributed > gpurun_out/bench_cfg2_xdist_${TAG}.json 2>&1; tail -1 gpurun_out/bench_cfg2_xdist_${TAG}.json | cut -c1-200
bash scripts/trace.sh ${TAG} cfg2 cfg3 cfg5 cfg1 > /dev/null 2>&1
bash scripts/launches.sh ${TAG} cfg2 cfg3
fi
ls gpurun_out | grep ${TAG}
