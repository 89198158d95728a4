"""Debug: batch-table occupancy and step timing across cfg2 steps (eager, no graph)."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2210_08803_b200 import Context, workload as W
from paper_2210_08803_b200.sharded import build_tables, TrainStep
cfg = W.config2()
ctx = Context(0)
t = build_tables(ctx, cfg, 0, 1)
st = TrainStep(ctx, t, cfg, 0, 1, use_graph=False)
gen = W.BatchGen(cfg)
bs = [st.stage_batch(*gen.batch(s)[:2]) for s in range(3)]
d = torch.randn(cfg.batch * cfg.n_slots, cfg.dim, device="cuda") * 0.01
v = ctypes.c_uint64(0)
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st.run(bs[i % 3], d, step=i + 1)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ctx.lib.hps_gpu_debug_batch_table_used(t.h, ctypes.byref(v))
    print(f"step {i}: {dt*1e6:.0f} us wall, batch table used {v.value}", flush=True)
