"""Generate tests/golden/update_frames.json: UpdateBatch frames encoded and
decoded by oracle/_ref/libhps_ref.so — a codec written over the REFERENCE's own
ByteWriter / ByteReader (proj/include/hps/bytes.hpp:33-133; oracle/ref_shim.cpp
ref_update_encode / ref_update_decode). TEST INFRASTRUCTURE ONLY; run in the build
container: `make -C oracle && python oracle/gen_update_golden.py`.

Records: valid frames (hex) with their fields, and malformed frames with the ErrorCode
the reference primitives raise (BadMagic 2, BadFormatVersion 3, Truncated 4,
TrailingBytes 5, DuplicateKey 6, InvalidArgument 1 for an unknown dtype byte).
"""
import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
lib = C.CDLL(os.path.join(HERE, "_ref", "libhps_ref.so"))
vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
lib.ref_update_encode.restype = C.c_int
lib.ref_update_encode.argtypes = [C.c_char_p, u32, u64, u32, u32, C.c_int, vp, vp, vp, u64, C.POINTER(u64)]
lib.ref_update_decode.restype = C.c_int
lib.ref_update_decode.argtypes = [vp, u64, C.c_char_p, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32),
                                  C.POINTER(C.c_int), vp, vp, u64]


def encode(name, seq, keys, values, dtype):
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    v = np.ascontiguousarray(values)
    dim = v.shape[1]
    n = u64()
    st = lib.ref_update_encode(name.encode(), len(name.encode()), seq, len(k), dim, dtype, k.ctypes.data,
                               v.ctypes.data, None, 0, C.byref(n))
    assert st == 0, st
    out = np.empty(n.value, dtype=np.uint8)
    st = lib.ref_update_encode(name.encode(), len(name.encode()), seq, len(k), dim, dtype, k.ctypes.data,
                               v.ctypes.data, out.ctypes.data, n.value, C.byref(n))
    assert st == 0, st
    return out.tobytes()


def decode_status(frame):
    buf = np.frombuffer(frame, dtype=np.uint8) if frame else np.zeros(1, np.uint8)
    name = C.create_string_buffer(300)
    seq, count, dim, dt = u64(), u32(), u32(), C.c_int()
    keys = np.empty(4096, dtype=np.uint64)
    vals = np.empty(4096 * 256 * 4, dtype=np.uint8)
    st = lib.ref_update_decode(buf.ctypes.data, len(frame), name, C.byref(seq), C.byref(count), C.byref(dim),
                               C.byref(dt), keys.ctypes.data, vals.ctypes.data, 4096)
    return st, (name.value.decode(), seq.value, count.value, dim.value, dt.value)


def main():
    rs = np.random.default_rng(2210)
    valid, bad = [], []
    cases = [("ads", 1, 0, 4, 0), ("ads", 1, 1, 4, 0), ("t", 7, 5, 8, 1), ("clicks_v2", 2**40 + 3, 33, 16, 0),
             ("", 9, 3, 3, 1), ("x" * 255, 12, 2, 128, 0), ("emb", 2**64 - 1, 64, 128, 1)]
    for name, seq, count, dim, dtype in cases:
        keys = np.unique(rs.integers(0, 2**63 - 1, size=count + 8, dtype=np.int64))[:count].astype(np.uint64)
        rs.shuffle(keys)
        if count:
            keys[0] = 2**64 - 1
        if dtype == 0:
            vals = rs.standard_normal((count, dim)).astype(np.float32)
        else:
            vals = (rs.standard_normal((count, dim)).astype(np.float16)).view(np.uint16)
        f = encode(name, seq, keys, vals, dtype)
        st, fields = decode_status(f)
        assert st == 0 and fields == (name, seq, count, dim, dtype), (st, fields)
        valid.append({"table": name, "seq": str(seq), "count": count, "dim": dim, "dtype": dtype,
                      "keys": [str(int(k)) for k in keys], "frame": f.hex()})
    base = bytes.fromhex(valid[3]["frame"])
    dup_keys = np.array([5, 6, 5], dtype=np.uint64)
    dup = encode("dup", 3, dup_keys, np.zeros((3, 4), np.float32), 0)
    mutations = {
        "first_byte_flipped": bytes([base[0] ^ 0xFF]) + base[1:],
        "version_2": base[:4] + bytes([2]) + base[5:],
        "truncated_by_1": base[:-1],
        "truncated_in_header": base[:10],
        "empty": b"",
        "trailing_byte": base + b"\x00",
        "duplicate_key": dup,
        "dtype_byte_7": None,
    }
    name_len = 9
    dt_off = 4 + 1 + 2 + name_len + 8 + 4 + 2
    mutations["dtype_byte_7"] = base[:dt_off] + bytes([7]) + base[dt_off + 1:]
    for what, f in mutations.items():
        st, _ = decode_status(f)
        bad.append({"case": what, "frame": f.hex(), "code": st})
    json.dump({"valid": valid, "malformed": bad,
               "generator": "oracle/gen_update_golden.py over oracle/_ref/libhps_ref.so (reference ByteWriter/ByteReader)"},
              open(os.path.join(ROOT, "tests", "golden", "update_frames.json"), "w"), indent=1)
    print({b["case"]: b["code"] for b in bad})


if __name__ == "__main__":
    main()
