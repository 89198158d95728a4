"""A/B of the index probe scheme on one B200 (north_star (1): warp-cooperative probing).

One 40M-row table (config 2's largest Criteo table, index load 0.5 = 2^27 slots x 16 B),
1,437,696 lookups per launch (config 2's global batch: 55,296 x 26), three key mixes:
all present, 10 % absent, all absent. Each variant (group 1 = per-thread linear probe, the
product; 2/4/8 = warp-cooperative windows) is timed with CUDA events over 20 launches after
warm-up, L2 flushed between launches. Prints one JSON line per (mix, group)."""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_08803_b200 import Context, EmbeddingTableGroup  # noqa: E402
from paper_2210_08803_b200 import _lib as L  # noqa: E402
from paper_2210_08803_b200 import workload as W  # noqa: E402


def main():
    ctx = Context(0)
    cap, n = 39_884_406, 55_296 * 26
    g = EmbeddingTableGroup(ctx, [cap], 4, [0], "sgd", n, n, 1)
    for first in range(0, cap, 1 << 24):
        g.insert(0, ctx.gen_keys(W.table_seed(1, 0), first, min(1 << 24, cap - first)), return_rows=False)
    ctx.sync()
    rs = np.random.default_rng(0)
    present = W.table_keys(1, 0, rs.integers(0, cap, n))
    absent = rs.integers(0, 2**63, n).astype(np.uint64) | np.uint64(1 << 63)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for mix, frac in (("present", 0.0), ("absent_10pct", 0.1), ("absent", 1.0)):
        m = rs.random(n) < frac
        q = torch.from_numpy(np.where(m, absent, present).view(np.int64)).cuda()
        for grp in (1, 2, 4, 8):
            f = lambda: L.check(ctx.lib.hps_gpu_debug_find_variant(g.h, 0, C.c_void_p(q.data_ptr()), n,
                                                                   C.c_void_p(out.data_ptr()), grp), "find")
            for _ in range(3):
                f()
            ts = []
            for _ in range(20):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                f()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            us = float(np.median(ts)) * 1000
            print(json.dumps({"mix": mix, "group": grp, "us": round(us, 2), "mkeys_per_s": round(n / us, 1),
                              "probe": "per-thread linear" if grp == 1 else f"warp-cooperative x{grp}"}), flush=True)


if __name__ == "__main__":
    main()
