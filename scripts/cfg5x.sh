timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg2 cfg1 cfg3 cfg5; do echo "== $c"; timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 --e2e-steps 2 --trace 8 2>&1 | grep "count\|seg_alloc\|reduce_short\|^{" | cut -c1-150; done
