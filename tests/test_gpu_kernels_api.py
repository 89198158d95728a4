"""The reference's kernel API (proj/include/hps/kernels.hpp:33-43) on the GPU, against the
golden vectors oracle/gen_golden.py recorded from the reference's own compiled scalar path
(tests/golden/ref_vectors.json): CRC-32C of seeded buffers (plain, continuing from a running
value, per record), binary16 widening over all 65,536 patterns and narrowing over 2^20
seeded f32 patterns (sha256 of the outputs), and the binary16 NaN/Inf scan."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import workload as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_vectors.json")))


def stream(seed, n):
    return W.rng(seed, np.arange(n, dtype=np.uint64))  # = gen_golden.splitmix_stream


def test_crc32c_matches_reference(ctx):
    g = G["crc32c"]
    blob = (stream(g["blob_seed"], g["blob_len"]) & np.uint64(0xFF)).astype(np.uint8)
    d = torch.from_numpy(blob).cuda()
    for c in g["cases"]:
        assert ctx.crc32c(d[:c["len"]], c["crc_in"]) == c["crc"], c
    assert ctx.crc32c(torch.tensor(list(b"123456789"), dtype=torch.uint8, device="cuda")) == 0xE3069283
    offs = torch.tensor(g["batch_offsets"], dtype=torch.int64, device="cuda")
    got = ctx.crc32c_batch(d, offs).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, np.array(g["batch_crc"], dtype=np.uint32))


def test_f16_conversions_match_reference(ctx):
    allh = torch.arange(65536, dtype=torch.int32).to(torch.int16).cuda()
    wide = ctx.f16_to_f32(allh).cpu().numpy()
    assert hashlib.sha256(wide.tobytes()).hexdigest() == G["f16_to_f32_all_sha256"]
    s = G["f32_to_f16_sample"]
    bits = (stream(s["seed"], s["n"]) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    nar = ctx.f32_to_f16(torch.from_numpy(bits.view(np.float32)).cuda()).cpu().numpy()
    assert hashlib.sha256(nar.tobytes()).hexdigest() == s["sha256"]
    # the small named cases too (65519 -> 0x7bff, 65520 -> inf, 1/3 -> 0x3555, ...)
    f = G["f16"]
    src = torch.from_numpy(np.array(f["f32_bits"], dtype=np.uint32).view(np.float32)).cuda()
    np.testing.assert_array_equal(ctx.f32_to_f16(src).cpu().numpy().view(np.uint16), np.array(f["f16_bits"], np.uint16))


def test_non_finite_f16_matches_reference(ctx):
    for k, case in G["has_non_finite_f16"].items():
        v = torch.from_numpy(np.array(case["bits"], dtype=np.uint16).view(np.int16)).cuda()
        assert ctx.has_non_finite_f16(v) == bool(case["non_finite"]), k
