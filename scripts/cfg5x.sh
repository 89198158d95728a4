timeout 900 python -m pytest tests/test_gpu_table.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg3 cfg1; do timeout 400 python bench.py --config $c --no-cpu-baseline --steps 10 --e2e-steps 2 --trace 4 2>&1 | grep "reduce_short\|reduce_long\|^{" | cut -c1-170; done
