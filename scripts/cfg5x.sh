HPS_BENCH_E2E_CPU=1 timeout 400 python bench.py --config cfg2 --no-cpu-baseline --steps 20 2>&1 | grep "^#\|^{" | cut -c1-120
python - <<'PY'
import time, torch
x=torch.zeros(1).cuda(); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(1000): pass
print("noop", (time.perf_counter()-t)*1e3)
PY
