timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg2 cfg5; do for r in 38 36; do echo "== $c rows=$r"; HPS_GPU_TMA_ROWS=$r timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 --e2e-steps 2 | cut -c100-190; done; done
bash scripts/trace.sh v12b cfg2 2>&1 | grep -v "^{"
