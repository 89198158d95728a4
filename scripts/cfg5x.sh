timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg3 cfg2 cfg5 cfg1; do echo "== $c"; timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 --e2e-steps 2 --trace 4 2>&1 | grep "pool \|count \|place\|reduce_short\|^{" | cut -c1-150; done
