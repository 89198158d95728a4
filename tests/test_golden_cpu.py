"""CPU tests: the oracle and the product's host code against the REFERENCE's golden vectors.

tests/golden/ref_vectors.json was produced by oracle/gen_golden.py from the reference's
own sources compiled unmodified (oracle/_ref/libhps_ref.so). No GPU is needed here.
"""
import ctypes as C
import json
import os
import struct

import numpy as np
import pytest

from tests import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_vectors.json")))
KEYS = np.array([int(k) for k in G["key_hash"]["keys"]], dtype=np.uint64)
HASHES = np.array([int(h) for h in G["key_hash"]["hash"]], dtype=np.uint64)


def product():
    from paper_2210_08803_b200 import _lib
    return _lib.load()


def test_survey_appendix_a_known_answers():
    # SURVEY.md Appendix A.1 (computed from the compiled reference) and SPEC.md:57
    assert G["fnv1a64"][0]["hash"] == str(0xCBF29CE484222325)
    table = {0: 0xA8C7F832281A39C5, 1: 0x89CD31291D2AEFA4, 2: 0xE6BD86443DF8CE07, 3: 0xC7C2BF3B330983E6,
             2**64 - 1: 0x8CF51A8BFCA3883D, 123456789: 0xDF604AC5D726CE19}
    for k, h in table.items():
        i = int(np.nonzero(KEYS == np.uint64(k))[0][0])
        assert int(HASHES[i]) == h
    assert G["crc32c_123456789"] == 0xE3069283


def test_oracle_key_hash_matches_reference():
    L = O.lib()
    out = np.empty_like(KEYS)
    L.orc_key_hash_n(O.P(KEYS), len(KEYS), O.P(out))
    np.testing.assert_array_equal(out, HASHES)


def test_oracle_partition_of_matches_reference():
    L = O.lib()
    shards = G["partition_of"]["shards"]
    want = np.array(G["partition_of"]["table"], dtype=np.uint32)
    for j, n in enumerate(shards):
        out = np.empty(len(KEYS), dtype=np.uint32)
        L.orc_partition_of_n(O.P(KEYS), len(KEYS), n, O.P(out))
        np.testing.assert_array_equal(out, want[:, j])


def test_oracle_fnv1a64_matches_reference():
    L = O.lib()
    for rec in G["fnv1a64"]:
        b = bytes.fromhex(rec["hex"])
        assert L.orc_fnv1a64(b, len(b)) == int(rec["hash"])


def test_oracle_non_finite_matches_reference():
    L = O.lib()
    for name, rec in G["has_non_finite_f32"].items():
        v = np.array(rec["values_bits"], dtype=np.uint32).view(np.float32)
        assert L.orc_has_non_finite_f32(O.P(v) if len(v) else None, len(v)) == rec["non_finite"], name


def test_product_host_hash_header_matches_reference():
    lib = product()
    for k, h in zip(KEYS[:300], HASHES[:300]):
        assert lib.hps_key_hash_host(int(k)) == int(h)


def test_fastmod_is_exact():
    lib = product()
    rs = np.random.default_rng(1)
    divs = [1, 2, 3, 7, 8, 10, 26, 1000, 1250000, 12500000, 2**31 - 1, 2**32 - 1, 2**32 + 15, 2**63 + 5, 2**64 - 1]
    nums = [0, 1, 2**64 - 1, 2**63, 2**32 - 1] + [int(x) for x in rs.integers(0, 2**63, 200, dtype=np.int64)] + \
           [int(x) * 2 + 1 for x in rs.integers(0, 2**63, 200, dtype=np.int64)]
    for d in divs + [int(x) for x in rs.integers(1, 2**40, 50, dtype=np.int64)]:
        for a in nums:
            assert lib.hps_fastmod_u64_host(a, d) == a % d, (a, d)


def test_product_error_names_match_reference():
    lib = product()
    for code, name in G["error_code_name"].items():
        assert lib.hps_error_code_name(int(code)).decode() == name


def test_product_validation_matches_reference():
    lib = product()
    for dim, code in G["validate_dim"].items():
        assert lib.hps_validate_dim(int(dim)) == code
    cases = {"finite": [1.0, -2.0, 0.0, 3.4e38], "nan": [1.0, float("nan")], "inf": [float("inf")],
             "neg_inf": [0.0] * 8 + [-float("inf")], "long_tail_nan": [0.5] * 37 + [float("nan")]}
    for name, vals in cases.items():
        arr = (C.c_float * len(vals))(*vals)
        assert lib.hps_embedding_vector_f32_status(arr, len(vals)) == G["embedding_vector_f32_status"][name], name
    tm = G["table_meta_make"]
    assert lib.hps_table_meta_make_status(b"ads", 16, 16) == tm["ok"]
    assert lib.hps_table_meta_make_status(b"ads", 16, 8) == tm["dim_mismatch"]
    assert lib.hps_table_meta_make_status(b"", 16, 16) == tm["empty_name"]
    assert lib.hps_table_meta_make_status(b"x" * 256, 16, 16) == tm["long_name"]


def test_partition_balance_spec_examples():
    # n=1 -> 0; 1M random keys over 8 shards, max/mean <= 1.05
    L = O.lib()
    keys = np.random.default_rng(7).integers(0, 2**63, 1_000_000, dtype=np.int64).astype(np.uint64)
    out = np.empty(len(keys), dtype=np.uint32)
    L.orc_partition_of_n(O.P(keys), len(keys), 1, O.P(out))
    assert not out.any()
    L.orc_partition_of_n(O.P(keys), len(keys), 8, O.P(out))
    counts = np.bincount(out, minlength=8)
    assert counts.max() / counts.mean() <= 1.05
    seq = np.arange(1_000_000, dtype=np.uint64)
    L.orc_partition_of_n(O.P(seq), len(seq), 8, O.P(out))
    assert (np.bincount(out, minlength=8) == 125_000).all()


def test_oracle_f16_matches_reference():
    """The oracle's binary16 restatement (the F16 cache storage checker) against the
    reference's own f32_to_f16 / f16_to_f32 (kernels_scalar.cpp:25-57, golden vectors),
    and against IEEE binary16 (numpy) exhaustively for widening and on random narrowing."""
    L = O.lib()
    src = np.array(G["f16"]["f32_bits"], dtype=np.uint32).view(np.float32)
    out = np.empty(len(src), dtype=np.uint16)
    L.orc_f32_to_f16(O.P(src), O.P(out), len(src))
    np.testing.assert_array_equal(out, np.array(G["f16"]["f16_bits"], dtype=np.uint16))
    back = np.empty(len(src), dtype=np.float32)
    L.orc_f16_to_f32(O.P(out), O.P(back), len(out))
    np.testing.assert_array_equal(back.view(np.uint32), np.array(G["f16"]["roundtrip_f32_bits"], dtype=np.uint32))
    allh = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    wide = np.empty(65536, dtype=np.float32)
    L.orc_f16_to_f32(O.P(allh), O.P(wide), 65536)
    ref = allh.view(np.float16).astype(np.float32)
    fin = np.isfinite(ref)
    np.testing.assert_array_equal(wide[fin].view(np.uint32), ref[fin].view(np.uint32))
    rs = np.random.default_rng(5)
    x = rs.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    x = x[np.isfinite(x)]
    nar = np.empty(len(x), dtype=np.uint16)
    L.orc_f32_to_f16(O.P(x), O.P(nar), len(x))
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(nar, x.astype(np.float16).view(np.uint16))


def test_crc32c_golden_cases_restated():
    """The golden CRC-32C cases (recorded from the reference) against a table-driven
    restatement of kernels_scalar.cpp:89-108 — pins the fixture the GPU test reads."""
    from paper_2210_08803_b200 import workload as W
    tbl = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (0x82F63B78 ^ (c >> 1)) if c & 1 else c >> 1
        tbl.append(c)

    def crc(c, data):
        c ^= 0xFFFFFFFF
        for b in data:
            c = tbl[(c ^ b) & 0xFF] ^ (c >> 8)
        return c ^ 0xFFFFFFFF
    g = G["crc32c"]
    blob = bytes((W.rng(g["blob_seed"], np.arange(g["blob_len"], dtype=np.uint64)) & np.uint64(0xFF)).astype(np.uint8))
    for c in g["cases"]:
        if c["len"] <= 70000:
            assert crc(c["crc_in"], blob[:c["len"]]) == c["crc"]
    o = g["batch_offsets"]
    assert [crc(0, blob[a:b]) for a, b in zip(o[:20], o[1:21])] == g["batch_crc"][:20]
