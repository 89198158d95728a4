"""The miss path's lower tiers on the host (csrc/tiers.cpp through the C-ABI): the VDB (L2,
SPEC.md:192-250) and the PDB (L3), checked against the spec's examples and
against flat reference maps replaying the same policies (test infrastructure, below). No GPU
is touched: these tiers live in host memory and on disk."""
import os
import struct

import numpy as np
import pytest

from paper_2210_08803_b200 import _lib as L
from paper_2210_08803_b200 import tiers as T
from tests import oracle_lib as O


def vecs(rs, n, dim):
    return rs.standard_normal((n, dim)).astype(np.float32)


def partition_of(keys, n):
    import ctypes as C
    k = np.ascontiguousarray(keys, np.uint64)
    out = np.zeros(len(k), np.uint32)
    L.load().hps_shard_of(k.ctypes.data_as(C.POINTER(C.c_uint64)), len(k), n, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


# ---- VDB ----------------------------------------------------------------------------------
def test_vdb_spec_examples():
    v = T.Vdb(4, 100, 8)
    assert not v.get_batch([1, 2, 3])[0].any()                     # empty store -> all missing
    assert v.put_batch([1, 2, 3], np.ones((3, 8)), [1, 1, 1]) == 3  # 3 fresh entries
    x = np.arange(8, dtype=np.float32)
    assert v.put_batch([9], [x], [2]) == 1
    assert v.put_batch([9], [x + 1], [1]) == 0                      # versions 2 then 1 -> 2 stays
    f, got, ver = v.get_batch([9])
    assert f[0] and ver[0] == 2 and np.array_equal(got[0], x)
    with pytest.raises(L.HpsError) as e:
        v.shard_snapshot(4)
    assert e.value.code == L.E_BAD_SHARD


def test_vdb_reject_new_at_capacity():
    v = T.Vdb(1, 2, 4)
    assert v.put_batch([1, 2, 3], np.ones((3, 4)), [1, 1, 1]) == 2
    f, _, _ = v.get_batch([1, 2, 3])
    assert f.tolist() == [True, True, False]
    assert v.put_batch([1], [np.zeros(4)], [5]) == 1  # an update of a resident key is not an insert


def test_vdb_evict_oldest_version():
    v = T.Vdb(1, 2, 4, "evict_oldest_version")
    v.put_batch([1, 2], np.ones((2, 4)), [7, 3])
    assert v.put_batch([3], [np.full(4, 3.0)], [5]) == 1  # evicts key 2 (version 3)
    f, got, ver = v.get_batch([1, 2, 3])
    assert f.tolist() == [True, False, True] and ver[2] == 5 and got[2][0] == 3.0


def reference_vdb(shards, cap, policy, batches):
    """A flat map per shard replaying the VDB's rules in input order."""
    m = [dict() for _ in range(shards)]
    for keys, vs, vers in batches:
        sh = partition_of(keys, shards)
        for k, x, ver, s in zip(keys.tolist(), vs, vers.tolist(), sh.tolist()):
            d = m[s]
            if k in d:
                if ver > d[k][1]:
                    d[k] = (x.copy(), ver)
                continue
            if len(d) >= cap:
                if policy == "reject_new":
                    continue
                old = min(d.items(), key=lambda kv: (kv[1][1], kv[0]))[0]
                del d[old]
            d[k] = (x.copy(), ver)
    return m


@pytest.mark.parametrize("policy", ["reject_new", "evict_oldest_version"])
def test_vdb_randomized_matches_reference_map(policy):
    rs = np.random.default_rng(3)
    shards, cap, dim = 4, 40, 6
    v = T.Vdb(shards, cap, dim, policy)
    batches = []
    for _ in range(12):
        n = int(rs.integers(1, 60))
        keys = rs.integers(0, 300, n).astype(np.uint64)
        vers = rs.permutation(10_000)[:n].astype(np.uint64)  # distinct: the evicted entry is unambiguous
        x = vecs(rs, n, dim)
        v.put_batch(keys, x, vers)
        batches.append((keys, x, vers))
    ref = reference_vdb(shards, cap, policy, batches)
    total = 0
    for s in range(shards):
        k, x, ver = v.shard_snapshot(s)
        assert sorted(ref[s]) == k.tolist(), f"shard {s} keys"
        for j, key in enumerate(k.tolist()):
            assert ver[j] == ref[s][key][1] and np.array_equal(x[j], ref[s][key][0])
        assert len(k) <= cap
        assert (partition_of(k, shards) == s).all()  # routing invariant
        total += len(k)
    assert total == v.size()
    probe = np.arange(300, dtype=np.uint64)
    f, _, _ = v.get_batch(probe)
    assert f.sum() == total


def test_vdb_balance_one_million_keys():
    keys = np.random.default_rng(1).integers(0, 2**63, 1_000_000).astype(np.uint64)
    c = np.bincount(partition_of(keys, 8), minlength=8)
    assert c.max() <= 1.05 * c.mean()


# ---- PDB ----------------------------------------------------------------------------------
def test_pdb_empty_root_and_durability(tmp_path):
    root = str(tmp_path / "pdb")
    p = T.Pdb(root)
    assert p.table_count() == 0
    rs = np.random.default_rng(5)
    keys = np.unique(rs.integers(0, 2**63, 10_000).astype(np.uint64))
    x = vecs(rs, len(keys), 16)
    p.create_table("emb", 16)
    assert p.put_batch("emb", keys, x, np.ones(len(keys), np.uint64)) == len(keys)
    p.close()
    p = T.Pdb(root)
    assert p.table_count() == 1 and p.dropped_tail == 0
    f, got, ver = p.get_batch("emb", keys)
    assert f.all() and (ver == 1).all() and np.array_equal(got, x)  # bit-exact round trip


def test_pdb_versions_and_namespaces(tmp_path):
    root = str(tmp_path / "pdb")
    p = T.Pdb(root)
    p.create_table("a", 4)
    p.create_table("b", 4, default=np.full(4, 0.5))
    assert p.put_batch("a", [7], [np.full(4, 1.0)], [1]) == 1
    assert p.put_batch("a", [7], [np.full(4, 2.0)], [2]) == 1
    assert p.put_batch("a", [7], [np.full(4, 9.0)], [1]) == 0  # stale
    assert p.put_batch("b", [7], [np.full(4, 5.0)], [1]) == 1
    p.close()
    p = T.Pdb(root)
    fa, va, vera = p.get_batch("a", [7])
    fb, vb, _ = p.get_batch("b", [7])
    assert vera[0] == 2 and va[0][0] == 2.0 and vb[0][0] == 5.0  # version 2 wins; table-local
    assert np.array_equal(p.default("b"), np.full(4, 0.5, np.float32)) and not p.default("a").any()
    with pytest.raises(L.HpsError) as e:
        p.get_batch("nope", [1])
    assert e.value.code == L.E_UNKNOWN_TABLE
    with pytest.raises(L.HpsError) as e:
        p.create_table("a", 8)
    assert e.value.code == L.E_DIM_MISMATCH


def test_pdb_scan_and_compact(tmp_path):
    root = str(tmp_path / "pdb")
    p = T.Pdb(root)
    p.create_table("t", 8)
    rs = np.random.default_rng(9)
    keys = np.arange(500, dtype=np.uint64) * 977
    p.put_batch("t", keys, vecs(rs, 500, 8), np.ones(500, np.uint64))
    assert p.compact("t") == 0  # no overwrites: nothing reclaimed
    x2 = vecs(rs, 500, 8)
    p.put_batch("t", keys, x2, np.full(500, 2, np.uint64))  # overwrite every key once
    before = p.get_batch("t", keys)
    k, x, ver = p.scan("t")
    assert k.tolist() == sorted(keys.tolist()) and (ver == 2).all()
    rec = 8 + 8 + 2 + 1 + 8 * 4 + 4
    assert p.compact("t") == 500 * rec
    after = p.get_batch("t", keys)
    assert all(np.array_equal(a, b) for a, b in zip(before, after))
    p.close()
    p = T.Pdb(root)
    k2, x3, _ = p.scan("t")
    assert len(k2) == 500 and np.array_equal(x3[np.argsort(k2)], x2[np.argsort(keys)])


def segment_files(root, table):
    d = os.path.join(root, table)
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.startswith("seg_"))


def test_pdb_record_layout_and_checksum(tmp_path):
    """LogRecord = key | version | dim u16 | dtype u8 | payload | CRC-32C of the preceding bytes;
    the checksum is the reference's crc32c (pinned by its golden cases below)."""
    root = str(tmp_path / "pdb")
    p = T.Pdb(root)
    p.create_table("t", 3)
    p.put_batch("t", [0x1122334455667788], [np.array([1.5, -2.0, 3.25], np.float32)], [42])
    p.close()
    raw = open(segment_files(root, "t")[0], "rb").read()
    assert len(raw) == 19 + 12 + 4
    key, ver, dim, dtype = struct.unpack_from("<QQHB", raw, 0)
    assert (key, ver, dim, dtype) == (0x1122334455667788, 42, 3, 0)
    assert struct.unpack_from("<3f", raw, 19) == (1.5, -2.0, 3.25)
    (crc,) = struct.unpack_from("<I", raw, 31)
    assert T.crc32c(b"123456789") == 0xE3069283
    assert crc == T.crc32c(raw[:31])


def test_host_crc32c_matches_reference_goldens():
    """The PDB's host CRC-32C against the golden cases recorded from the reference's own
    compiled crc32c (tests/golden/ref_vectors.json, oracle/gen_golden.py), continuing values
    included."""
    import json
    from paper_2210_08803_b200 import workload as W
    G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.json")))
    g = G["crc32c"]
    blob = bytes((W.rng(g["blob_seed"], np.arange(g["blob_len"], dtype=np.uint64)) & np.uint64(0xFF)).astype(np.uint8))
    for c in g["cases"]:
        assert T.crc32c(blob[:c["len"]], c["crc_in"]) == c["crc"], c
    o = g["batch_offsets"]
    assert [T.crc32c(blob[a:b]) for a, b in zip(o[:-1], o[1:])] == g["batch_crc"]


def test_pdb_torn_tail_dropped_interior_corruption_fatal(tmp_path, monkeypatch):
    root = str(tmp_path / "pdb")
    rec = 19 + 4 * 4 + 4
    monkeypatch.setenv("HPS_PDB_SEGMENT_BYTES", str(10 * rec))  # 10 records per segment
    p = T.Pdb(root)
    p.create_table("t", 4)
    keys = np.arange(25, dtype=np.uint64)
    x = np.arange(100, dtype=np.float32).reshape(25, 4)
    p.put_batch("t", keys, x, np.ones(25, np.uint64))
    p.close()
    segs = segment_files(root, "t")
    assert len(segs) == 3
    with open(segs[-1], "r+b") as f:  # a torn tail: the last record half-written
        f.truncate(os.path.getsize(segs[-1]) - rec // 2)
    p = T.Pdb(root)
    assert p.dropped_tail == 1
    f, got, _ = p.get_batch("t", keys)
    assert f[:24].all() and not f[24] and np.array_equal(got[:24], x[:24])
    assert p.put_batch("t", [24], [x[24]], [1]) == 1  # appends after the truncated tail
    p.close()
    p = T.Pdb(root)
    assert p.dropped_tail == 0 and p.get_batch("t", keys)[0].all()
    p.close()
    with open(segs[0], "r+b") as f:  # a flipped payload byte inside an older segment
        f.seek(rec * 3 + 20)
        b = f.read(1)
        f.seek(rec * 3 + 20)
        f.write(bytes([b[0] ^ 0x40]))
    with pytest.raises(L.HpsError) as e:
        T.Pdb(root)
    assert e.value.code == L.E_CORRUPTION
