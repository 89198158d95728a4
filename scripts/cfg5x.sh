timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for m in 8 16; do echo "== mult $m"; HPS_GPU_BT_MULT=$m bash scripts/trace.sh v12f cfg1 cfg2 2>&1 | grep "count\|reduce_short\|=="; for c in cfg1 cfg2; do tail -1 gpurun_out/trace_${c}_v12f.json | cut -c100-180; done; done
