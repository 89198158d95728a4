for d in persistent flat lead; do for p in 1 0; do
  echo "== dedup $d pipeline $p"; HPS_GPU_DEDUP=$d HPS_PIPELINE=$p timeout 300 python -m pytest tests/test_gpu_table.py -q -p no:cacheprovider -k "adam_graph_step or pipelined_host" 2>&1 | grep -E "passed|failed|vs eager|Mismatched elements" | head -5
done; done
