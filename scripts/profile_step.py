"""A few eager training steps of one config (for ncu: per-kernel DRAM bytes of a step).
Usage: python scripts/profile_step.py cfg2 [steps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_08803_b200 import Context  # noqa: E402
from paper_2210_08803_b200 import workload as W  # noqa: E402
from paper_2210_08803_b200.sharded import TrainStep, build_tables  # noqa: E402

CFG = {"cfg1": W.config1, "cfg2": W.config2, "cfg3": W.config3, "cfg5": W.config5}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = CFG[name]()
    ctx = Context(0)
    tables = build_tables(ctx, cfg)
    ts = TrainStep(ctx, tables, cfg, use_graph=False)
    gen = W.BatchGen(cfg)
    rs = np.random.default_rng(0)
    dout = torch.from_numpy((rs.standard_normal((cfg.batch * cfg.n_slots, cfg.dim)) * 0.01).astype(np.float32)).cuda()
    for s in range(steps):
        keys, offs, _, _ = gen.batch(s)
        ts.run(ts.stage_batch(keys, offs), dout, step=s + 1)
    torch.cuda.synchronize()
    print("steps done", name, ts.last_counts())


if __name__ == "__main__":
    main()
