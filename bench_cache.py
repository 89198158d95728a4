"""bench_cache.py — BASELINE config 4: HPS inference cache batch sweep on one B200.

100M-key dim-128 fp32 backing table resident in HBM (51.2 GB; this sweep times the all-GPU
read-through, so the "lower tier" is a GPU table — the host VDB/PDB miss path is timed by
scripts/bench_tiered.py), a GPU cache at 10 % capacity (10M rows, 8 ways,
1.25M sets, aging 10 x capacity), Zipf(1.05) query keys. After a warm-up of >= 10 x
capacity accesses, each batch size 1, 2, 4, ... 131072 is timed as one orchestrator
read-through (cache query -> misses read from the table -> misses migrated into the
cache) with CUDA events; prints one JSON line per batch size (p50/p95 latency, hit rate,
keys/s) and a summary line. The CPU oracle cache (tests/oracle_lib, the checker — not the
product) is timed on the same query stream at small scale for reference.

  python bench_cache.py [--keys 100000000] [--capacity 10000000] [--reps 50] [--scale 1.0]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=100_000_000)
    ap.add_argument("--capacity", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--zipf", type=float, default=1.05)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--max-batch", type=int, default=131072)
    ap.add_argument("--warmup-mult", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16"], help="cache row storage (binary16 halves the bytes)")
    ap.add_argument("--eager", action="store_true", help="no CUDA graphs (default: one graph per batch size)")
    ap.add_argument("--phases", action="store_true", help="debug: per-call times (query / read-through / insert) at the max batch")
    args = ap.parse_args()

    import torch
    from paper_2210_08803_b200 import Context, EmbeddingTableGroup, HotCache
    from paper_2210_08803_b200 import workload as W
    from paper_2210_08803_b200.api import CachedLookup

    ctx = Context(0)
    seed = 0x5EED0004
    t0 = time.perf_counter()
    table = EmbeddingTableGroup(ctx, [args.keys], args.dim, [0], "sgd", args.max_batch, args.max_batch, seed)
    tseed = W.table_seed(seed, 0)
    chunk = 1 << 24
    for first in range(0, args.keys, chunk):
        table.insert(0, ctx.gen_keys(tseed, first, min(chunk, args.keys - first)))
    ctx.sync()
    cache = HotCache(ctx, args.capacity, args.dim, 8, 0, args.max_batch, dtype=args.dtype)
    rt = CachedLookup(cache, table)
    setup_s = time.perf_counter() - t0

    # Zipf(s) over the table's rows on the GPU: inverse CDF (float64) + seeded affine permutation
    n = args.keys
    w = torch.arange(1, n + 1, dtype=torch.float64, device="cuda").pow_(-args.zipf)
    cdf = torch.cumsum(w, 0)
    del w
    H = float(cdf[-1].item())
    perm = W.affine_perm(seed + 4, n)
    a_mul = int(perm(np.array([1]))[0] - perm(np.array([0]))[0]) % n
    c_add = int(perm(np.array([0]))[0])
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    tseed_t = torch.tensor(tseed - (1 << 64) if tseed >= (1 << 63) else tseed, dtype=torch.int64, device="cuda")

    def zipf_keys(m):
        u = torch.rand(m, dtype=torch.float64, device="cuda", generator=gen) * H
        r = torch.searchsorted(cdf, u, right=True).clamp_(max=n - 1)
        idx = (r * a_mul + c_add) % n
        return mix64_t(tseed_t ^ idx)

    def mix64_t(z):  # splitmix64 finaliser on int64 tensors (wrapping arithmetic)
        z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * -4658895280553007687  # 0xbf58476d1ce4e5b9
        z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * -7723592293110705685  # 0x94d049bb133111eb
        return z ^ ((z >> 31) & ((1 << 33) - 1))

    # warm-up: >= warmup_mult x capacity accesses in max-size batches
    t1 = time.perf_counter()
    n_warm = int(args.warmup_mult * args.capacity)
    for _ in range(0, n_warm, args.max_batch):
        rt.lookup(zipf_keys(args.max_batch))
    ctx.sync()
    warm_s = time.perf_counter() - t1

    if args.phases:  # per-stage device times of the cache query inside each lookup (stderr)
        os.environ["HPS_GPU_CACHE_PHASES"] = "1"
        for _ in range(3):
            rt.lookup(zipf_keys(args.max_batch))
        ctx.sync()
        del os.environ["HPS_GPU_CACHE_PHASES"]

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6541.8))

    results = []
    b = 1
    while b <= args.max_batch:
        reps = args.reps if b <= 8192 else max(10, args.reps // 4)
        batches = [zipf_keys(b) for _ in range(reps)]
        if not args.eager:  # capture this size's graph outside the timed calls
            rt.lookup_graphed(zipf_keys(b))
            ctx.sync()
        cache.reset_stats()
        lat = []
        for kb in batches:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if args.eager:
                rt.lookup(kb)
            else:
                rt.lookup_graphed(kb)
            e1.record()
            e1.synchronize()
            lat.append(e0.elapsed_time(e1) * 1000.0)
        s = cache.stats()
        lat = np.array(lat)
        src = rt.sources()  # the last batch's per-key sources
        n_hit, n_miss = src["L1"], src["L2"] + src["Default"]
        # SURVEY §8(d) cache-query bytes over the INPUT keys: Q(k + 8 ways) + H(2 D e + 18) + M 12
        row = args.dim * (2 if args.dtype == "f16" else 4)
        alg = b * (8 + 8 * 8) + n_hit * (2 * row + 18) + n_miss * 12
        p50 = float(np.median(lat))
        line = {"config": "cfg4-hps-cache", "dtype": args.dtype, "graph": not args.eager, "batch": b, "p50_us": p50,
                "p95_us": float(np.percentile(lat, 95)), "keys_per_s": b / (p50 / 1e6),
                "hit_rate": s["hits"] / max(1, s["queries"]),  # over the distinct keys the cache saw
                "key_hit_rate": n_hit / b, "unique_frac": int(rt.n_unique.item()) / b,
                "alg_bytes": alg, "achieved_gbs": alg / (p50 * 1e3), "frac_hbm": alg / (p50 * 1e3) / hbm_peak}
        results.append(line)
        print(json.dumps(line), flush=True)
        b *= 2

    # ideal static hit rate: top-capacity Zipf mass
    ideal = float(cdf[args.capacity - 1].item() / H)
    cpu = None
    if not args.no_cpu:
        from tests import oracle_lib as O
        oc = O.OracleCache(min(args.capacity, 1 << 20), args.dim, 8, 0)
        q = W.mix64(np.arange(200_000, dtype=np.uint64))
        vec = np.ones((len(q), args.dim), np.float32)
        t2 = time.perf_counter()
        for i in range(0, len(q), 4096):
            fi, fv, mi = oc.query(q[i:i + 4096])
            oc.insert(q[i:i + 4096][mi], vec[:len(mi)], np.zeros(len(mi), np.uint64))
        dt = time.perf_counter() - t2
        cpu = {"keys_per_s": len(q) / dt, "cores": 1, "kind": "port",
               "sample": "200k cold keys, 4096-key batches, query + insert of misses, 1M-row cache"}
    summary = {"config": "cfg4-hps-cache", "dtype": args.dtype, "summary": True, "keys": args.keys, "capacity": args.capacity,
               "dim": args.dim, "zipf": args.zipf, "ideal_static_hit_rate": ideal,
               "hit_rate_at_max_batch": results[-1]["hit_rate"],
               "key_hit_rate_at_max_batch": results[-1]["key_hit_rate"], "frac_hbm_max_batch": results[-1]["frac_hbm"], "p50_us_batch1": results[0]["p50_us"],
               "p50_us_max_batch": results[-1]["p50_us"], "keys_per_s_max_batch": results[-1]["keys_per_s"],
               "setup_s": setup_s, "warmup_s": warm_s, "warmup_accesses": n_warm, "cpu_baseline": cpu}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
