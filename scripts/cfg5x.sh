cp paper_2210_08803_b200/libhps_gpu.so /tmp/base.so
for v in base m8; do
  if [ $v = base ]; then cp /tmp/base.so paper_2210_08803_b200/libhps_gpu.so; else cp variants_$v.so paper_2210_08803_b200/libhps_gpu.so; fi
  for c in cfg3 cfg2; do
  echo "== $v $c"; timeout 400 python bench.py --config $c --no-cpu-baseline --steps 20 --e2e-steps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('frac',d['roofline']['frac'],'kernel_ms',d['roofline']['kernel_ms'],'step',d['ms_per_step'])"
  done
done
cp /tmp/base.so paper_2210_08803_b200/libhps_gpu.so
