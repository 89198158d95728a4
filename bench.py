"""bench.py — DLRM-shape embedding fwd+bwd+update samples/s on B200 (BASELINE.json metric).

Workload (N=1 default): BASELINE config 2, the MLPerf-DLRM shape — 26 tables at the
Criteo-1TB cardinalities capped at 40M (187.8M rows, 96.1 GB fp32 at dim 128), one key
per slot, sum pooling, sparse SGD, 6,912 samples per GPU per step (8 GPUs x 6,912 =
the config's global batch 55,296). One step = hps_gpu_lookup_pooled (train) +
hps_gpu_backward_update on synthetic keys; d_out (the dense model's gradient, out of
scope) is a pre-generated device tensor. Multi-GPU: distributed slot sharding
(owner = key_hash mod G) through paper_2210_08803_b200.sharded.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg1|cfg3|cfg5] [--impl ours|reference]

cfg5 = one hashed table over a 1e9-key space (power-law keys), dim 128, Adam; rows
materialise on first touch (insert-on-miss inside the step, HPS_LOOKUP_INSERT).

Prints ONE JSON line (rank 0). `--impl reference` times the CPU implementation of the
same step (the oracle port, all host threads) on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2210_08803_b200 import workload as W  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "round1", "ncu_traffic.json")
STEP_TRAFFIC_PATH = os.path.join(ROOT, "profiles", "round2", "ncu_step_traffic.json")


def ncu_traffic(workload, path=TRAFFIC_PATH):
    """DRAM bytes (read + write) from a committed ncu capture, or None: per launch of the fused
    lookup (TRAFFIC_PATH), or per training step summed over its kernels (STEP_TRAFFIC_PATH,
    profiles/step_traffic.py)."""
    try:
        with open(path) as f:
            d = json.load(f)[workload]
        return int(d["dram_read"]) + int(d["dram_write"])
    except Exception:
        return None
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg5"])
    ap.add_argument("--batch-per-gpu", type=int, default=None)
    ap.add_argument("--placement", default="auto",
                    choices=["auto", "distributed", "distributed-py", "localized", "hybrid"],
                    help="multi-GPU slot placement (auto: localized for cfg3, distributed otherwise)")
    ap.add_argument("--hot-budget-gb", type=float, default=0.0625, help="hybrid: replicated hot rows per GPU")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="distributed placement through the C-ABI: NCCL all-to-alls, or peer-memory kernels")
    ap.add_argument("--force-exchange", action="store_true",
                    help="run the multi-GPU exchange path (NCCL world of one) on a single GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool", type=int, default=4, help="distinct synthetic batches rotated through")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--pipeline", action="store_true",
                    help="batch pipelining: each step prefetches (records + dedups) the next batch on a slot stream")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--table-scale", type=float, default=1.0, help="debug only: shrink cardinalities")
    ap.add_argument("--sustain-s", type=float, default=2.0,
                    help="untimed steps run under the clock sampler right before the timed steps")
    ap.add_argument("--full-batch", type=int, default=55296,
                    help="N=1 cfg2: also time steps at BASELINE's literal global batch (0 = off)")
    ap.add_argument("--trace", type=int, default=0,
                    help="debug: after timing, replay N steps with the in-graph kernel timeline on (stderr)")
    return ap.parse_args()


def get_config(args):
    if args.config == "cfg1":
        cfg = W.config1()
    elif args.config == "cfg2":
        cfg = W.config2()
    elif args.config == "cfg3":
        cfg = W.config3()
    else:
        cfg = W.config5()
    if args.batch_per_gpu:
        cfg.batch = args.batch_per_gpu
    if args.table_scale != 1.0:
        cfg.cards = [max(1, int(c * args.table_scale)) for c in cfg.cards]
    return cfg


def workload_config(cfg, world, args):
    """The workload the line is quoted on — identical in the GPU arm and the reference arm."""
    xchg = world > 1 or args.force_exchange
    placement = args.placement if args.placement != "auto" else ("localized" if args.config == "cfg3" else "distributed")
    return {"workload": cfg.name, "batch_per_gpu": cfg.batch, "global_batch": cfg.batch * world,
            "tables": len(cfg.cards), "rows": int(sum(cfg.cards)), "dim": cfg.dim, "hot": cfg.hot,
            "combiner": cfg.combiner, "optimizer": cfg.optimizer, "keyspace": cfg.keyspace,
            "parallelism": f"{placement}-slot x{world}" if xchg else "single"}


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------------------
def algorithmic_bytes(N, U, n_bags, dim, n_state, multi):
    e, k, P = 4, 8, 16
    f = 4 if multi else 0
    fwd = N * (k + P + dim * e) + n_bags * (dim * e + f)
    bwd = n_bags * (dim * e + f) + N * k + U * (P + 2 * dim * e * (1 + n_state))
    return fwd, bwd


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[3 + j].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------------------
# CPU side: the reference arm and the cpu_baseline leg (oracle port; checker, not product)
# ---------------------------------------------------------------------------------------
def cpu_step_runner(cfg, threads):
    from tests import oracle_lib as O
    import ctypes as C
    L = O.lib()
    L.orc_sparse_create.restype = C.c_void_p
    L.orc_sparse_create.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int, C.c_uint64, C.c_float]
    L.orc_sparse_step.restype = C.c_int
    L.orc_sparse_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_int]
    L.orc_sparse_destroy.argtypes = [C.c_void_p]
    st = np.asarray(cfg.slots(), dtype=np.uint32)
    opt = {"sgd": 0, "adagrad": 1, "adam": 2}[cfg.optimizer]
    h = L.orc_sparse_create(len(cfg.cards), cfg.dim, O.P(st), len(st), opt, cfg.seed, 0.0)
    from paper_2210_08803_b200.api import opt_params
    p = opt_params(cfg.optimizer, cfg.lr, eps=cfg.eps)
    o7 = np.array([p.lr, p.eps, p.beta1, p.beta2, p.one_minus_beta1, p.one_minus_beta2, p.lr_t], dtype=np.float32)
    comb = 1 if cfg.combiner == "mean" else 0

    def step(keys, offs, dout, out):
        return L.orc_sparse_step(h, O.P(keys), O.P(offs), cfg.batch, comb, O.P(dout), O.P(o7), O.P(out), threads)

    return step, lambda: L.orc_sparse_destroy(h)


def run_cpu(cfg, steps, warmup, threads, budget_s=None):
    """Time the oracle port of one full per-GPU step. Returns (samples/s, sample description)."""
    gen = W.BatchGen(cfg)
    batches = [gen.batch(s) for s in range(min(4, steps + warmup))]
    step, close = cpu_step_runner(cfg, threads)
    rs = np.random.default_rng(0)
    n_bags = cfg.batch * cfg.n_slots
    dout = (rs.standard_normal((n_bags, cfg.dim)) * 0.01).astype(np.float32)
    out = np.empty((n_bags, cfg.dim), dtype=np.float32)
    for s in range(warmup):
        k, o, _, _ = batches[s % len(batches)]
        step(k, o, dout, out)
    t0 = time.perf_counter()
    done = 0
    for s in range(steps):
        k, o, _, _ = batches[s % len(batches)]
        step(k, o, dout, out)
        done += 1
        if budget_s and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    close()
    return cfg.batch * done / dt, f"{done} full steps of {cfg.batch} samples x {cfg.n_slots} slots (rows materialised on first touch)"


def host_info():
    """The CPU the baseline ran on: nproc, affinity, model name."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model}


def reference_arm(args, cfg, rank, world):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    val, sample = run_cpu(cfg, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": "DLRM-shape embedding fwd+bwd+update samples/s", "value": val,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * cfg.batch / val, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": workload_config(cfg, world, args),
        "cpu_baseline": {"value": val, "unit": "samples/s", "cores": threads, "kind": "port", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": val, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


TRACE_NAMES = {0: "probe", 1: "pool", 2: "seg_alloc", 3: "place", 4: "long_hist", 5: "long_pass0",
               6: "long_pass1", 7: "long_pass2", 8: "long_pass3", 9: "long_reg", 10: "reduce_short",
               11: "reduce_long", 12: "reset_counts", 13: "count", 14: "|count_local", 15: "|count_global",
               16: "|count_cas", 17: "|count_probe", 18: "scale_dout", 19: "<step-in", 20: ">step-out", 21: "ins_claim",
               22: "ins_commit", 23: "ins_finish"}


def print_trace(ctx, n, step):
    """In-graph kernel timeline (hps_gpu_debug_trace): median start/end of each traced kernel
    relative to the step's first kernel, over n replays (L2 flushed before each)."""
    import ctypes
    lib = ctx.lib
    buf = (ctypes.c_uint64 * 64)()
    lib.hps_gpu_debug_trace(1, None)
    recs = []
    for i in range(n):
        step(i)
        lib.hps_gpu_debug_trace(2, buf)
        r = {k: (buf[2 * k], buf[2 * k + 1]) for k in TRACE_NAMES if buf[2 * k] != (1 << 64) - 1 or buf[2 * k + 1]}
        s0 = min((v[0] for v in r.values() if v[0] != (1 << 64) - 1), default=0)
        r = {k: (v[0] if v[0] != (1 << 64) - 1 else v[1], v[1]) for k, v in r.items()}  # end-only markers
        r = {k: (v[0], v[1] if v[1] else v[0]) for k, v in r.items()}  # began but no warp did work (empty list)
        if r:
            t0 = min(v[0] for v in r.values())
            recs.append({k: ((a - t0) / 1000.0, (b - t0) / 1000.0) for k, (a, b) in r.items()})
    lib.hps_gpu_debug_trace(0, None)
    keys = sorted({k for r in recs for k in r}, key=lambda k: float(np.median([r[k][0] for r in recs if k in r])))
    print(f"# in-graph timeline, us (median of {len(recs)} steps)", file=sys.stderr)
    for k in keys:
        st = float(np.median([r[k][0] for r in recs if k in r]))
        en = float(np.median([r[k][1] for r in recs if k in r]))
        print(f"#   {TRACE_NAMES[k]:<14s} {st:8.1f} -> {en:8.1f}  ({en - st:6.1f})", file=sys.stderr)


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = get_config(args)
    if cfg.keyspace:  # every step sees a fresh batch, so new keys keep materialising inside the timed steps
        args.pool = max(args.pool, args.warmup + args.steps + args.trace)
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2210_08803_b200 import Context, opt_params
    from paper_2210_08803_b200.sharded import (build_tables, build_tables_hybrid, build_tables_localized,
                                               hybrid_hot_set, localized_plan, TrainStep)

    torch.cuda.set_device(local)
    xchg = world > 1 or args.force_exchange
    full_batch = 0
    if xchg:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29512")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = Context(local)
    t_setup = time.perf_counter()
    placement = args.placement if args.placement != "auto" else ("localized" if args.config == "cfg3" else "distributed")
    owned = localized_plan(cfg, world) if xchg and placement == "localized" else None
    hot = None
    if xchg and placement == "hybrid":
        hot, tables = build_tables_hybrid(ctx, cfg, rank, world, hybrid_hot_set(cfg, int(args.hot_budget_gb * 1e9)))
    elif owned is None:
        full_batch = args.full_batch if (world == 1 and not xchg and args.config == "cfg2") else 0
        tables = build_tables(ctx, cfg, rank, world, batch_cap=full_batch)
    else:
        tables = build_tables_localized(ctx, cfg, owned, rank, world)
    gen = W.BatchGen(cfg)
    step_fn = TrainStep(ctx, tables, cfg, rank, world, use_graph=not args.no_graph, owned=owned, hybrid_hot=hot,
                        force_exchange=xchg, pipeline=args.pipeline, cabi=placement != "distributed-py",
                        transport=args.transport)
    pool = []
    rs = np.random.default_rng(rank)
    n_bags = cfg.batch * cfg.n_slots
    for s in range(args.pool):
        keys, offs, _, _ = gen.batch(s * world + rank)
        pool.append(step_fn.stage_batch(keys, offs))
    douts = [torch.from_numpy((rs.standard_normal((n_bags, cfg.dim)) * 0.01).astype(np.float32)).cuda()
             for _ in range(min(args.pool, 2))]
    setup_s = time.perf_counter() - t_setup

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    # Step sequence. Call c runs batch idx(c) with d_out douts[c % 2] and names batch idx(c+1)
    # as the next one (prefetched inside the step: TrainStep pipelining), so the step graphs are
    # keyed by (c mod 4). A hashed table (config 5) times FRESH batches: the warm-up and the
    # sustained-clock steps cycle over pool[0:W), the timed steps use pool[W:W+K) (their keys
    # materialise inside the timed steps).
    P = len(pool)
    n_warm_pool = args.warmup if cfg.keyspace else P
    timed0 = args.warmup if cfg.keyspace else 0

    def pre_idx(c):
        return c % n_warm_pool

    calls = [0]

    def one(i, idx=None, nxt=None):
        c = calls[0]
        b = pool[pre_idx(c) if idx is None else idx]
        nb = pool[pre_idx(c + 1) if nxt is None else nxt]
        step_fn.run(b, douts[c % len(douts)], step=c + 1, next_b=nb)
        calls[0] += 1

    def timed_idx(i):
        return (timed0 + i) % P if not cfg.keyspace else timed0 + i

    for i in range(args.warmup):
        one(i)
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    # the clocks are sampled over a sustained run of the same step (>= args.sustain_s of
    # untimed steps: the timed K steps alone last a few ms, shorter than nvidia-smi's
    # sampling period) that runs straight into the timed steps
    t_sus, n_sus = time.perf_counter(), 0
    while time.perf_counter() - t_sus < args.sustain_s:
        for _ in range(50):
            one(args.warmup + n_sus)
            n_sus += 1
        torch.cuda.synchronize()
    # bridge (untimed): the batch the last step prefetched, naming the first timed batch next
    one(0, idx=pre_idx(calls[0]), nxt=timed_idx(0))
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xff)  # evict L2 between timed iterations (not inside the step events)
        starts[i].record(stream)
        one(i, idx=timed_idx(i), nxt=timed_idx(i + 1) if i + 1 < args.steps else pre_idx(calls[0] + 1))
        ends[i].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ctx.sync()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    N, U = step_fn.last_counts()
    # the dominant kernel alone: one hps_gpu_lookup_pooled launch (k_lookup_*) between events
    for i in range(3):  # warm-up: the inference kernel's first launch pays its lazy module load
        step_fn.lookup_only(pool[i % len(pool)])
    torch.cuda.synchronize()
    fwd_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        fwd_ev[i][0].record(stream)
        step_fn.lookup_only(pool[i % len(pool)])
        fwd_ev[i][1].record(stream)
    torch.cuda.synchronize()
    fwd_ms = [a.elapsed_time(b) for a, b in fwd_ev]
    if args.trace:
        def traced(i):  # stamps around the step mark its start/end latency in the stream
            flush.fill_(i & 0xff)
            ctx.lib.hps_gpu_debug_stamp(ctypes.c_void_p(stream.cuda_stream), 19)
            if cfg.keyspace:  # fresh batches, as the timed steps (their keys materialise in the step)
                one(i, idx=timed0 + args.steps + i, nxt=timed0 + args.steps + i + 1 if i + 1 < args.trace else None)
            else:
                one(i)
            ctx.lib.hps_gpu_debug_stamp(ctypes.c_void_p(stream.cuda_stream), 20)
        print_trace(ctx, args.trace, traced)
    ms = float(np.mean(step_ms))
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * cfg.batch / (ms_max / 1000.0)

    # BASELINE's literal global batch (55,296 samples) as ONE GPU's step: the same tables,
    # a TrainStep at that batch, K timed steps (L2 flushed between them)
    full = None
    if full_batch > cfg.batch:
        cfg_f = W.Config(**{**cfg.__dict__, "batch": full_batch})
        step_f = TrainStep(ctx, tables, cfg_f, rank, world, use_graph=not args.no_graph, pipeline=args.pipeline)
        gen_f = W.BatchGen(cfg_f)
        pool_f = [step_f.stage_batch(*gen_f.batch(5000 + s)[:2]) for s in range(2)]
        dout_f = torch.from_numpy((rs.standard_normal((full_batch * cfg.n_slots, cfg.dim)) * 0.01)
                                  .astype(np.float32)).cuda()
        n_w = max(4, args.warmup + args.warmup % 2)
        for i in range(n_w):
            step_f.run(pool_f[i % 2], dout_f, step=i + 1, next_b=pool_f[(i + 1) % 2])
        torch.cuda.synchronize()
        ev_f = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            ev_f[i][0].record(stream)
            step_f.run(pool_f[i % 2], dout_f, step=100 + i, next_b=pool_f[(i + 1) % 2])
            ev_f[i][1].record(stream)
        torch.cuda.synchronize()
        ms_f = float(np.mean([a.elapsed_time(b) for a, b in ev_f]))
        Nf, Uf = step_f.last_counts()
        ff, fb = algorithmic_bytes(Nf, Uf, full_batch * cfg.n_slots, cfg.dim, 0, False)
        full = {"batch_per_gpu": full_batch, "ms_per_step": ms_f, "value": full_batch / (ms_f / 1000.0),
                "unit": "samples/s", "unique_keys": Uf, "key_occurrences": Nf,
                "step_algorithmic_bytes": ff + fb, "step_frac": (ff + fb) / (ms_f / 1000.0) / 1e9 / hbm_peak()[0]}
        del step_f, pool_f, dout_f

    # algorithmic bytes of the last step's batch on this rank
    fwd_b, bwd_b = algorithmic_bytes(N, U, n_bags, cfg.dim, {"sgd": 0, "adagrad": 1, "adam": 2}[cfg.optimizer],
                                     cfg.hot > 1)
    peak, peak_kind = hbm_peak()
    fwd_ms_mean = float(np.mean(fwd_ms))
    fwd_gbs = fwd_b / (fwd_ms_mean / 1000.0) / 1e9
    step_gbs = (fwd_b + bwd_b) / (ms / 1000.0) / 1e9

    # e2e: the same step through the C-ABI from pinned HOST keys + a D2H read of the step result
    e2e_steps = args.e2e_steps or args.steps
    host_batches = []
    for s in range(min(args.pool, 4)):
        keys, offs, _, _ = gen.batch(1000 + s * world + rank)
        host_batches.append(step_fn.stage_host(keys, offs))
    # warm every (host buffer, d_out) pairing the timed loop uses (one-hot steps capture a
    # CUDA graph per pairing on first use; capture must not land in the timed region)
    # (pairings x 2 result slots: the pipelined loop below alternates slots)
    n_pair = len(host_batches) * len(douts) // math.gcd(len(host_batches), len(douts))
    n_pair = n_pair * 2 // math.gcd(n_pair, 2)
    nh = len(host_batches)
    for i in range(max(2, n_pair) + 1):
        step_fn.run_host_async(host_batches[i % nh], douts[i % len(douts)], step=10_000 + i,
                               slot=i % 2, next_b=host_batches[(i + 1) % nh])
        step_fn.read_host_result(i % 2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d = d2h = 0
    # one step in flight: step i's result (D2H into pinned memory) is read on the host after
    # step i+1 is enqueued; every step moves its inputs H2D and its result D2H
    e2e0 = max(2, n_pair) + 1  # continue the warm-up's batch sequence (the next batch is prefetched)
    for i in range(e2e_steps):
        j = e2e0 + i
        bi, bo = step_fn.run_host_async(host_batches[j % nh], douts[j % len(douts)],
                                        step=20_000 + i, slot=j % 2, next_b=host_batches[(j + 1) % nh])
        if i:
            _ = step_fn.read_host_result((j - 1) % 2)
        h2d, d2h = bi, bo
    _ = step_fn.read_host_result((e2e0 + e2e_steps - 1) % 2)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    t = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = world * cfg.batch / (float(t.item()) / 1000.0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        cval, sample = run_cpu(cfg, steps=30, warmup=2, threads=threads, budget_s=20.0)
        cpu = {"value": cval, "unit": "samples/s", "cores": threads, "kind": "port", "sample": sample,
               "host": host_info()}

    if rank == 0:
        line = {
            "metric": "DLRM-shape embedding fwd+bwd+update samples/s",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": workload_config(cfg, world, args),
            "run": {"l2": "flushed between timed steps (256 MB write)", "graph": step_fn.graph_mode,
                    "insert_on_miss": step_fn.insert_missing},
            # the timed unit: one training step (lookup + backward + update, one CUDA graph);
            # algorithmic bytes per SURVEY.md §8(d) over the step's N occurrences / U unique rows
            "roofline": {"bound": "hbm",
                         "kernel": "training step: probe, dedup, pooling, short + long reduce with the fused "
                                   "optimizer (one CUDA graph)",
                         "achieved": step_gbs, "peak": peak, "unit": "GB/s", "frac": step_gbs / peak,
                         "peak_kind": peak_kind,
                         "traffic": ncu_traffic(cfg.name, STEP_TRAFFIC_PATH) if world == 1 else None,
                         "traffic_source": "ncu dram__bytes_read+write summed over one eager step's kernels, "
                                           "cold caches (profiles/round2/ncu_step_traffic.json)",
                         "algorithmic_bytes": fwd_b + bwd_b, "ms": ms,
                         "fused_lookup": {
                             "kernel": "k_lookup_1hot_tma<0> (inference: hash+probe+gather+pool)" if cfg.hot == 1
                             else "k_lookup_multi (inference: hash+probe+gather+pool)",
                             "achieved": fwd_gbs, "frac": fwd_gbs / peak, "algorithmic_bytes": fwd_b,
                             "kernel_ms": fwd_ms_mean, "traffic": ncu_traffic(cfg.name) if world == 1 else None}},
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": step_fn.kernels_per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "unique_keys": U, "key_occurrences": N, "setup_s": setup_s,
        }
        if full is not None:
            line["full_batch_n1"] = full
        if xchg:
            xb = step_fn.exchange.exchanged_bytes(cfg.dim)
            line["nvlink"] = {"bytes_per_step_rank0": xb, "achieved_gbs": xb / (ms_max / 1000.0) / 1e9,
                              "peak_gbs": 770.0, "peak_kind": "measured peer copy (B200_PROFILING.md)",
                              "frac": xb / (ms_max / 1000.0) / 1e9 / 770.0}
            line["roofline"]["kernel"] = (
                {"distributed": "distributed forward (bucketize + all-to-all + gather + all-to-all + pool)",
                 "localized": "localized forward (regroup + all-to-all + owner lookup + all-to-all + place)",
                 "hybrid": "hybrid forward (hot probe + cold all-to-all + gather + all-to-all + pool)"}[step_fn.placement])
        print(json.dumps(line), flush=True)
    if xchg:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
