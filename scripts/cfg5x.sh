timeout 600 python -m pytest tests/test_gpu_cache.py tests/test_gpu_table.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench_cache.py --reps 30 --no-cpu > gpurun_out/cache_graph4.jsonl 2>&1; head -13 gpurun_out/cache_graph4.jsonl | cut -c40-150; tail -2 gpurun_out/cache_graph4.jsonl | cut -c1-250
