"""Miss-path latency of the three-tier orchestrator (hps_gpu_tiered_lookup) on a
config-4-shaped stream, scaled to a PDB that fits the box's scratch disk: K keys (dim 128) in
the PDB, the VDB sized to 20 % of them, the GPU cache to 5 %, Zipf(1.05) query keys. After a
warm-up (the migrations fill L2/L1 the way a serving process would), each batch size is timed
on the host (the call returns before its migrations; the await is timed separately) and the
per-key source mix is reported. One JSON line per batch size.

  python scripts/bench_tiered.py [--keys 2000000] [--reps 20] [--root /tmp/hps_pdb_bench]
"""
import argparse
import json
import os
import shutil
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=2_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--zipf", type=float, default=1.05)
    ap.add_argument("--root", default="/tmp/hps_pdb_bench")
    args = ap.parse_args()
    import torch
    from paper_2210_08803_b200 import Context, HotCache
    from paper_2210_08803_b200 import tiers as T
    from paper_2210_08803_b200 import workload as W

    K, D = args.keys, args.dim
    shutil.rmtree(args.root, ignore_errors=True)
    ctx = Context(0)
    rs = np.random.default_rng(0)
    keys = W.table_keys(0x5EED0004, 0, np.arange(K, dtype=np.int64))
    t0 = time.perf_counter()
    pdb = T.Pdb(args.root)
    pdb.create_table("emb", D)
    chunk = 1 << 18
    for a in range(0, K, chunk):
        k = keys[a:a + chunk]
        pdb.put_batch("emb", k, rs.standard_normal((len(k), D)).astype(np.float32), np.ones(len(k), np.uint64))
    pdb.close()
    pdb = T.Pdb(args.root)  # reopen: the index rebuilt from the segments
    load_s = time.perf_counter() - t0
    vdb = T.Vdb(8, max(1, K // 5 // 8), D, "evict_oldest_version")
    max_batch = 16384
    cache = HotCache(ctx, max(8, K // 20 // 8 * 8), D, 8, 0, max_batch)
    tl = T.TieredLookup(cache, vdb, pdb, "emb", max_batch)
    z = W.Zipf(K, args.zipf)

    def batch(n):
        r = W.rng(int(rs.integers(0, 2**62)), np.arange(n, dtype=np.uint64))
        return torch.from_numpy(keys[z.ranks(r)].view(np.int64)).cuda()

    t0 = time.perf_counter()
    for _ in range(40):  # warm-up: fills L1 and L2 through the migrations
        tl.lookup(batch(max_batch))
        tl.await_migrations()
    warm_s = time.perf_counter() - t0
    print(json.dumps({"setup": True, "keys": K, "dim": D, "pdb_load_s": round(load_s, 2), "warmup_s": round(warm_s, 2),
                      "vdb_entries": vdb.size(), "cache_entries": cache.size()}), flush=True)
    b = 1
    while b <= max_batch:
        lat, aw, src = [], [], {"L1": 0, "L2": 0, "L3": 0, "Default": 0}
        for _ in range(args.reps):
            kb = batch(b)
            torch.cuda.synchronize()
            t = time.perf_counter()
            tl.lookup(kb)
            torch.cuda.synchronize()
            lat.append(time.perf_counter() - t)
            t = time.perf_counter()
            tl.await_migrations()
            aw.append(time.perf_counter() - t)
            for k, v in tl.sources().items():
                src[k] += v
        tot = sum(src.values())
        p50 = float(np.median(lat))
        print(json.dumps({"batch": b, "p50_us": round(p50 * 1e6, 1), "p95_us": round(float(np.percentile(lat, 95)) * 1e6, 1),
                          "await_p50_us": round(float(np.median(aw)) * 1e6, 1), "keys_per_s": round(b / p50),
                          "source_frac": {k: round(v / tot, 4) for k, v in src.items()}}), flush=True)
        b *= 4
    tl.close()
    pdb.close()
    shutil.rmtree(args.root, ignore_errors=True)


if __name__ == "__main__":
    main()
