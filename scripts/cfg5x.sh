#!/bin/bash
# Scratch A/B runner for one gpurun call (rewritten per experiment; see DESIGN.md §3 "Tried and reverted").
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench_cache.py --reps 30 --no-cpu > gpurun_out/cache_graph5.jsonl 2>&1; head -3 gpurun_out/cache_graph5.jsonl | cut -c40-150; tail -2 gpurun_out/cache_graph5.jsonl | cut -c1-200
