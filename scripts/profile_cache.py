"""Config-4 read-throughs at one batch size (for ncu: per-kernel times of the orchestrator
lookup). Same setup as bench_cache.py (100M-row dim-128 table, 10M-row cache, Zipf 1.05),
a short warm-up, then 3 eager lookups of `batch` keys.
Usage: python scripts/profile_cache.py [batch] [warm_batches]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_08803_b200 import Context, EmbeddingTableGroup, HotCache  # noqa: E402
from paper_2210_08803_b200 import workload as W  # noqa: E402
from paper_2210_08803_b200.api import CachedLookup  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    keys_n, cap, dim, seed = 100_000_000, 10_000_000, 128, 0x5EED0004
    ctx = Context(0)
    table = EmbeddingTableGroup(ctx, [keys_n], dim, [0], "sgd", batch, batch, seed)
    tseed = W.table_seed(seed, 0)
    for first in range(0, keys_n, 1 << 24):
        table.insert(0, ctx.gen_keys(tseed, first, min(1 << 24, keys_n - first)), return_rows=False)
    cache = HotCache(ctx, cap, dim, 8, 0, batch)
    rt = CachedLookup(cache, table)
    w = torch.arange(1, keys_n + 1, dtype=torch.float64, device="cuda").pow_(-1.05)
    cdf = torch.cumsum(w, 0)
    del w
    H = float(cdf[-1].item())
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    tt = torch.tensor(tseed - (1 << 64) if tseed >= (1 << 63) else tseed, dtype=torch.int64, device="cuda")

    def keys(m):
        r = torch.searchsorted(cdf, torch.rand(m, dtype=torch.float64, device="cuda", generator=gen) * H,
                               right=True).clamp_(max=keys_n - 1)
        z = tt ^ ((r * 2654435761) % keys_n)
        z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * -4658895280553007687
        z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * -7723592293110705685
        return z ^ ((z >> 31) & ((1 << 33) - 1))

    for _ in range(warm):
        rt.lookup(keys(batch))
    torch.cuda.synchronize()
    for _ in range(3):
        rt.lookup(keys(batch))
    torch.cuda.synchronize()
    print("done", rt.sources(), int(rt.n_unique.item()))


if __name__ == "__main__":
    main()
