"""GPU parity for K1 (key_hash / partition_of / finiteness) against the reference's golden vectors."""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_vectors.json")))


def _keys():
    k = np.array([int(x) for x in G["key_hash"]["keys"]], dtype=np.uint64)
    return k, torch.from_numpy(k.view(np.int64)).cuda()


def test_key_hash_bit_exact(ctx):
    k, kt = _keys()
    want = np.array([int(h) for h in G["key_hash"]["hash"]], dtype=np.uint64)
    got = ctx.key_hash(kt).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(got, want)


def test_partition_of_bit_exact(ctx):
    k, kt = _keys()
    table = np.array(G["partition_of"]["table"], dtype=np.uint32)
    for j, n in enumerate(G["partition_of"]["shards"]):
        got = ctx.partition_of(kt, n).cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got, table[:, j], err_msg=f"n={n}")


def test_partition_of_rejects_zero_shards(ctx):
    from paper_2210_08803_b200 import HpsError
    _, kt = _keys()
    with pytest.raises(HpsError) as e:
        ctx.partition_of(kt, 0)
    assert e.value.code == 1


def test_partition_of_large_random_vs_oracle(ctx):
    from tests import oracle_lib as O
    keys = np.random.default_rng(3).integers(-2**63, 2**63 - 1, 3_000_001, dtype=np.int64)
    kt = torch.from_numpy(keys).cuda()
    for n in [8, 1_250_000, 2**32 - 1]:
        want = np.empty(len(keys), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(keys.view(np.uint64)), len(keys), n, O.P(want))
        got = ctx.partition_of(kt, n).cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got, want)


def test_has_non_finite(ctx):
    for name, rec in G["has_non_finite_f32"].items():
        v = np.array(rec["values_bits"], dtype=np.uint32).view(np.float32)
        t = torch.from_numpy(v.copy()).cuda() if len(v) else torch.empty(0, device="cuda")
        assert ctx.has_non_finite(t) == bool(rec["non_finite"]), name
    x = torch.randn(1 << 20, device="cuda")
    assert not ctx.has_non_finite(x)
    for pos in [0, 1, 3, 4, 12345, (1 << 20) - 1]:
        y = x.clone()
        y[pos] = float("inf")
        assert ctx.has_non_finite(y)
        assert ctx.has_non_finite(y[1:]) == (pos >= 1)  # misaligned start


def test_gen_keys_matches_workload(ctx):
    from paper_2210_08803_b200 import workload as W
    got = ctx.gen_keys(1234, 10, 1000).cpu().numpy().view(np.uint64)
    want = W.mix64(np.uint64(1234) ^ (np.arange(1000, dtype=np.uint64) + np.uint64(10)))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("group", [2, 4, 8])
def test_warp_cooperative_probe_matches_per_thread(ctx, group):
    """hps_gpu_debug_find_variant: the warp-cooperative window probe returns exactly the rows
    of the per-thread linear probe (hps_gpu_table_find), present and absent keys, at the
    index's full load (capacity rows inserted: load 0.5) and with wrap-around windows."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2210_08803_b200 import EmbeddingTableGroup
    from paper_2210_08803_b200 import _lib as L
    rs = np.random.default_rng(group)
    cap = 50_000
    g = EmbeddingTableGroup(ctx, [cap, 64], 4, [0, 1], "sgd", 1 << 16, 1 << 16, 1)
    ks = rs.integers(0, 2**63, cap).astype(np.uint64)
    g.insert(0, torch.from_numpy(ks.view(np.int64)).cuda(), return_rows=False)
    q = np.concatenate([ks, rs.integers(0, 2**63, 20_000).astype(np.uint64)])
    rs.shuffle(q)
    qt = torch.from_numpy(q.view(np.int64)).cuda()
    a = torch.empty(len(q), dtype=torch.int64, device="cuda")
    b = torch.empty_like(a)
    L.check(ctx.lib.hps_gpu_table_find(g.h, 0, C.c_void_p(qt.data_ptr()), len(q), C.c_void_p(a.data_ptr())), "find")
    L.check(ctx.lib.hps_gpu_debug_find_variant(g.h, 0, C.c_void_p(qt.data_ptr()), len(q), C.c_void_p(b.data_ptr()),
                                               group), "find_variant")
    ctx.sync()
    assert torch.equal(a, b)
    assert int((a >= 0).sum()) == cap
