"""Synthetic DLRM/Criteo-shaped workloads (host side).

Everything is a pure function of documented seeds so the CUDA path and the CPU
oracle consume byte-identical inputs:
  mix64(x)            splitmix64 finaliser (a bijection on u64)
  rng(seed, ctr)      mix64(seed + (ctr+1) * 0x9E3779B97F4A7C15)  (counter-based splitmix64)
  table_key(t, i)     mix64(table_seed(t) ^ i): distinct keys per table, i in [0, card_t)
  uniform index       floor(u53 * card)
  zipf index          inverse CDF over k^-s, then a seeded affine
                      permutation rank -> index (so hot keys are not adjacent rows)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
MASK64 = (1 << 64) - 1

# MLPerf DLRM Criteo-1TB per-feature cardinalities capped at 40M (public values).
CRITEO_1TB_CAPPED = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63, 38532951, 2953546, 403346, 10,
                     2208, 11938, 155, 4, 976, 14, 39979771, 25641295, 39664984, 585935, 12972, 108, 36]


def mix64(x):
    """splitmix64 finaliser on uint64 numpy arrays (or a python int)."""
    scalar = not isinstance(x, np.ndarray)
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return int(z) if scalar else z


def rng(seed: int, ctr: np.ndarray) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed & MASK64) + (c + np.uint64(1)) * GOLDEN)


def table_seed(config_seed: int, t: int) -> int:
    return mix64((config_seed * 0x100000001B3 + t + 1) & MASK64)


def table_keys(config_seed: int, t: int, idx: np.ndarray) -> np.ndarray:
    """Key of row-index `idx` of table t: mix64(table_seed ^ idx)."""
    return mix64(np.uint64(table_seed(config_seed, t)) ^ np.asarray(idx, dtype=np.uint64))


def uniform_index(r: np.ndarray, card: int) -> np.ndarray:
    u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return np.minimum(np.floor(u * card).astype(np.int64), card - 1)


class Zipf:
    """Inverse-CDF Zipf(s) sampler over ranks 1..n."""

    def __init__(self, n: int, s: float):
        self.n, self.s = n, s
        w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
        self.cdf = np.cumsum(w)
        self.H = float(self.cdf[-1])

    def prob(self, k: int) -> float:
        return (k ** -self.s) / self.H

    def ranks(self, r: np.ndarray) -> np.ndarray:
        """0-based ranks from uniform u64 draws."""
        u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * self.H
        return np.minimum(np.searchsorted(self.cdf, u, side="right"), self.n - 1).astype(np.int64)


def affine_perm(seed: int, n: int):
    """A seeded bijection on [0, n): i -> (a*i + c) mod n with gcd(a, n) == 1."""
    a = (mix64(seed) % n) | 1 if n > 1 else 1
    while math.gcd(a, n) != 1:
        a = (a + 2) % n or 1
    c = mix64(seed ^ 0x5A5A) % n if n > 1 else 0
    assert n < (1 << 31), "affine_perm: int64 products need n < 2^31"
    return lambda i: (np.asarray(i, dtype=np.int64) * a + c) % n


@dataclass
class Config:
    """One BASELINE.json configuration (per GPU shape)."""
    name: str
    cards: List[int]
    dim: int
    batch: int                      # samples per GPU per step
    hot: int = 1                    # keys per bag (1 = one-hot); multi-hot uses 1..2*hot-1
    zipf_s: Optional[float] = None  # None = uniform
    combiner: str = "sum"
    optimizer: str = "sgd"
    lr: float = 0.01
    eps: float = 1e-8
    seed: int = 0x5EED0000
    slot_table: List[int] = field(default_factory=list)
    keyspace: Optional[int] = None  # dynamic (hashed) table: keys drawn from [0, keyspace), rows on first touch

    @property
    def n_slots(self) -> int:
        return len(self.slot_table) if self.slot_table else len(self.cards)

    def slots(self) -> List[int]:
        return self.slot_table if self.slot_table else list(range(len(self.cards)))


def config1() -> Config:
    """26 slots x 1 hot over ONE 1M-key table, dim 16, batch 2048, sum, SGD."""
    return Config("cfg1-synthetic-1table-d16", [1_000_000], 16, 2048, seed=0x5EED0001, slot_table=[0] * 26)


def config2(batch_per_gpu: int = 6912) -> Config:
    """MLPerf DLRM shape: 26 Criteo-1TB tables (capped 40M), dim 128, one-hot, SGD."""
    return Config("cfg2-criteo1tb-26t-d128-sgd", list(CRITEO_1TB_CAPPED), 128, batch_per_gpu, seed=0x5EED0002)


def config3(batch_per_gpu: int = 6912) -> Config:
    """DCN/DeepFM multi-hot: 26 slots, 1..19 hots (mean 10), Zipf(1.1), dim 64, mean, AdaGrad."""
    return Config("cfg3-multihot-zipf1.1-d64-adagrad", list(CRITEO_1TB_CAPPED), 64, batch_per_gpu, hot=10,
                  zipf_s=1.1, combiner="mean", optimizer="adagrad", eps=1e-7, seed=0x5EED0003)


def config5(batch_per_gpu: int = 6912, capacity: int = 90_000_000) -> Config:
    """Large hashed table: 26 one-hot slots into ONE table over a 1e9-key space, dim 128,
    Adam, power-law (Zipf 1.05, continuous inverse) keys. fp32 Adam state for 1e9 rows does
    not fit 8 x 180 GB (SURVEY hard part 6), so rows materialise on first touch into a
    `capacity`-row pool per GPU (HPS_LOOKUP_INSERT)."""
    return Config("cfg5-hashed1e9-d128-adam", [capacity], 128, batch_per_gpu, zipf_s=1.05, optimizer="adam",
                  lr=0.001, seed=0x5EED0005, slot_table=[0] * 26, keyspace=1_000_000_000)


class PowerLaw:
    """Continuous-inverse Zipf(s) over ranks 1..n for n too large for a CDF table."""

    def __init__(self, n: int, s: float):
        self.n, self.s = n, s
        self.a = n ** (1.0 - s) - 1.0

    def ranks(self, r: np.ndarray) -> np.ndarray:
        u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        x = (self.a * u + 1.0) ** (1.0 / (1.0 - self.s))
        return np.minimum(np.floor(x).astype(np.int64) - 1, self.n - 1)


class BatchGen:
    """Deterministic batches: keys (sample-major bags), optional CSR offsets, and table-row indices."""

    def __init__(self, cfg: Config, cards: Optional[List[int]] = None):
        self.cfg = cfg
        self.cards = cards if cards is not None else cfg.cards
        self.slot_table = cfg.slots()
        self._zipf = {}
        # hashed tables draw indices from the logical key space, not from the row pool
        space = (lambda t: cfg.keyspace) if cfg.keyspace else (lambda t: self.cards[t])
        if cfg.zipf_s is not None:
            for t in set(self.slot_table):
                self._zipf[t] = (PowerLaw(space(t), cfg.zipf_s) if cfg.keyspace
                                 else Zipf(space(t), cfg.zipf_s))
        self._perm = {t: affine_perm(cfg.seed + 77 * t, space(t)) for t in set(self.slot_table)}
        self._space = space

    def batch(self, step: int, batch: Optional[int] = None, first_sample: int = 0):
        """Returns (keys u64[N], offsets u32[B*S+1] or None, table_idx i64[N], table_of i32[N])."""
        cfg = self.cfg
        B = batch if batch is not None else cfg.batch
        S = cfg.n_slots
        bag = np.arange(B * S, dtype=np.uint64) + np.uint64(first_sample * S)
        sseed = mix64((cfg.seed ^ (step * 0xA24BAED4963EE407)) & MASK64)
        if cfg.hot == 1:
            lens = np.ones(B * S, dtype=np.int64)
        else:
            lens = 1 + (rng(sseed ^ 0x1EAF, bag) % np.uint64(2 * cfg.hot - 1)).astype(np.int64)
        offsets = np.zeros(B * S + 1, dtype=np.int64)
        np.cumsum(lens, out=offsets[1:])
        N = int(offsets[-1])
        bag_of = np.repeat(np.arange(B * S, dtype=np.int64), lens)
        pos = np.arange(N, dtype=np.int64) - offsets[bag_of]
        slot_of = bag_of % S
        ctr = (bag[bag_of] * np.uint64(64) + pos.astype(np.uint64))
        r = rng(sseed, ctr)
        table_of = np.asarray(self.slot_table, dtype=np.int64)[slot_of]
        idx = np.empty(N, dtype=np.int64)
        keys = np.empty(N, dtype=np.uint64)
        for t in np.unique(table_of):
            m = table_of == t
            card = self._space(t)
            if cfg.zipf_s is None:
                ix = uniform_index(r[m], card)
            else:
                ix = np.asarray(self._perm[t](self._zipf[t].ranks(r[m])), dtype=np.int64)
            idx[m] = ix
            keys[m] = table_keys(cfg.seed, int(t), ix)
        offs = None if cfg.hot == 1 else offsets.astype(np.uint32)
        return keys, offs, idx, table_of.astype(np.int32)
