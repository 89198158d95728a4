"""CPU tests: UpdateBatch frames — the product codec (update.cu host side,
via the C-ABI) against golden frames made by a codec over the REFERENCE's own
ByteWriter / ByteReader (oracle/gen_update_golden.py -> tests/golden/update_frames.json)."""
import json
import os

import numpy as np
import pytest

from paper_2210_08803_b200 import updates as U
from paper_2210_08803_b200._lib import HpsError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "update_frames.json")))


def test_spec_frame_sizes():
    # "ads", seq 1, 0 entries, dim 4, F32 -> 25 bytes; one entry -> 49 bytes
    assert len(U.encode_update_batch("ads", 1, np.zeros(0, np.uint64), np.zeros((0, 4), np.float32))) == 25
    assert len(U.encode_update_batch("ads", 1, np.array([7], np.uint64), np.ones((1, 4), np.float32))) == 49


@pytest.mark.parametrize("i", range(len(G["valid"])))
def test_encode_parse_decode_match_reference_frames(i):
    v = G["valid"][i]
    frame = bytes.fromhex(v["frame"])
    h = U.parse_update_batch(frame)
    assert (h["table"], h["seq"], h["count"], h["dim"], h["dtype"]) == (v["table"], int(v["seq"]), v["count"],
                                                                        v["dim"], v["dtype"])
    table, seq, keys, vals = U.decode_update_batch(frame)
    assert [int(k) for k in keys] == [int(k) for k in v["keys"]]
    # re-encoding the decoded batch reproduces the reference frame byte for byte
    again = U.encode_update_batch(table, seq, keys, vals.reshape(v["count"], v["dim"]))
    assert again == frame


@pytest.mark.parametrize("i", range(len(G["malformed"])))
def test_malformed_frames_raise_reference_codes(i):
    b = G["malformed"][i]
    with pytest.raises(HpsError) as e:
        U.parse_update_batch(bytes.fromhex(b["frame"]))
    assert e.value.code == b["code"], b["case"]


def test_round_trip_random_batches():
    rs = np.random.default_rng(17)
    for trial in range(20):
        count, dim = int(rs.integers(0, 50)), int(rs.integers(1, 300))
        keys = np.unique(rs.integers(0, 2**63 - 1, count + 5, dtype=np.int64))[:count].astype(np.uint64)
        if trial % 2:
            vals = rs.standard_normal((len(keys), dim)).astype(np.float16).view(np.uint16)
        else:
            vals = rs.standard_normal((len(keys), dim)).astype(np.float32)
        f = U.encode_update_batch(f"t{trial}", trial + 1, keys, vals)
        t, s, k, v = U.decode_update_batch(f)
        assert t == f"t{trial}" and s == trial + 1
        np.testing.assert_array_equal(k, keys)
        np.testing.assert_array_equal(v.reshape(vals.shape).view(np.uint8), vals.view(np.uint8))


def test_encode_rejects_long_names():
    with pytest.raises(HpsError) as e:
        U.encode_update_batch("x" * 256, 1, np.array([1], np.uint64), np.ones((1, 4), np.float32))
    assert e.value.code == 1
