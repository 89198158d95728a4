timeout 600 python -m pytest tests/test_gpu_table.py -x -q -k "adam or insert" 2>&1 | tail -2
for f in "" "--no-graph"; do timeout 300 python bench.py --config cfg5 --no-cpu-baseline --steps 10 --e2e-steps 2 $f | cut -c1-200; done
timeout 300 python bench.py --config cfg2 --no-cpu-baseline --steps 10 --e2e-steps 2 | cut -c1-200
