"""Generate tests/golden/ref_vectors.json from the REFERENCE's own compiled code.

TEST INFRASTRUCTURE ONLY. Runs in the build container (where /root/reference exists):
`make -C oracle && python oracle/gen_golden.py`. It loads oracle/_ref/libhps_ref.so
(built by oracle/Makefile from /root/reference/proj, sources untouched) and records
known answers for every reference function on the path:
  key_hash / partition_of / fnv1a64      proj/include/hps/hash.hpp:30-54
  f32_to_f16 / f16_to_f32                proj/src/kernels/kernels_scalar.cpp:25-77
  has_non_finite_f32/_f16                proj/src/kernels/kernels_scalar.cpp:110-123
  crc32c                                 proj/src/kernels/kernels_scalar.cpp:89-108
  error_code_name                        proj/src/core/types.cpp:28-49
  validate_dim / EmbeddingVector::f32 / TableMeta::make   proj/src/core/types.cpp:57-152
The JSON is committed; the GPU box never needs /root/reference.
"""
import ctypes as C
import json
import os
import struct

HERE = os.path.dirname(os.path.abspath(__file__))
lib = C.CDLL(os.path.join(HERE, "_ref", "libhps_ref.so"))
u64, u32 = C.c_uint64, C.c_uint32
lib.ref_key_hash.restype = u64
lib.ref_key_hash.argtypes = [u64]
lib.ref_partition_of.restype = u32
lib.ref_partition_of.argtypes = [u64, u32]
lib.ref_fnv1a64.restype = u64
lib.ref_fnv1a64.argtypes = [C.c_char_p, u64]
lib.ref_crc32c.restype = u32
lib.ref_crc32c.argtypes = [u32, C.c_char_p, u64]
lib.ref_error_code_name.restype = C.c_char_p
lib.ref_active_backend.restype = C.c_char_p


def splitmix_stream(seed, n):
    out, s = [], seed & (2**64 - 1)
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        out.append(z ^ (z >> 31))
    return out


def main():
    keys = [0, 1, 2, 3, 2**64 - 1, 123456789, 2**63, 2**32 - 1, 2**32, 255, 256]
    keys += [1 << i for i in range(64)]
    keys += splitmix_stream(0x5EED0001, 2000)
    shards = [1, 2, 3, 4, 7, 8, 10, 26, 1000, 1250000, 4294967295]
    g = {"generator": "oracle/gen_golden.py", "source": "oracle/_ref/libhps_ref.so (reference sources compiled unmodified)"}
    g["key_hash"] = {"keys": [str(k) for k in keys], "hash": [str(lib.ref_key_hash(k)) for k in keys]}
    g["partition_of"] = {
        "shards": shards,
        "table": [[lib.ref_partition_of(k, n) for n in shards] for k in keys],
    }
    blobs = [b"", b"a", b"foobar", bytes(range(256)), b"\x00" * 8]
    g["fnv1a64"] = [{"hex": b.hex(), "hash": str(lib.ref_fnv1a64(b, len(b)))} for b in blobs]
    # f16 conversion (scalar reference path forced, then the AVX2 path: both recorded)
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 1.0 / 3.0, 65504.0, 65519.0, 65520.0, 1e6, -1e6, 6e-8, 3e-8,
            2.98e-8, 1e-10, 0.1, -2.5, 1024.75, 6.103515625e-05, 6.1e-05]
    vals += [struct.unpack("<f", struct.pack("<I", b))[0] for b in splitmix_stream(7, 500) for b in [b & 0xFFFFFFFF] if (b & 0x7F800000) != 0x7F800000]
    n = len(vals)
    src = (C.c_float * n)(*vals)
    dst = (C.c_uint16 * n)()
    lib.ref_force_scalar(1)
    lib.ref_f32_to_f16(src, dst, n)
    f16 = list(dst)
    back = (C.c_float * n)()
    lib.ref_f16_to_f32(dst, back, n)
    f32bits = [struct.unpack("<I", struct.pack("<f", x))[0] for x in back]
    g["f16"] = {"f32_bits": [struct.unpack("<I", struct.pack("<f", x))[0] for x in vals], "f16_bits": f16, "roundtrip_f32_bits": f32bits}
    lib.ref_force_scalar(0)
    g["active_backend_default"] = lib.ref_active_backend().decode()
    # finiteness
    cases = {
        "finite": [1.0, -2.0, 0.0, 3.4e38],
        "nan": [1.0, float("nan")],
        "inf": [float("inf")],
        "neg_inf": [0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -float("inf")],
        "empty": [],
        "long_tail_nan": [0.5] * 37 + [float("nan")],
    }
    nf = {}
    for k, v in cases.items():
        arr = (C.c_float * max(1, len(v)))(*v)
        nf[k] = {"values_bits": [struct.unpack("<I", struct.pack("<f", x))[0] for x in v], "non_finite": int(lib.ref_has_non_finite_f32(arr, len(v)))}
    g["has_non_finite_f32"] = nf
    h16 = {"finite": [0x3C00, 0x7BFF], "inf": [0x7C00], "nan": [0x3C00, 0x7E01]}
    g["has_non_finite_f16"] = {k: {"bits": v, "non_finite": int(lib.ref_has_non_finite_f16((C.c_uint16 * len(v))(*v), len(v)))} for k, v in h16.items()}
    g["crc32c_123456789"] = lib.ref_crc32c(0, b"123456789", 9)
    # CRC-32C of seeded buffers (bytes = low byte of a splitmix64 stream), lengths across the
    # GPU kernel's chunk edges, plain and continuing from a running value; and per-record CRCs
    blob = bytes(x & 0xFF for x in splitmix_stream(0xC5C, 1 << 18))
    lens = [0, 1, 2, 3, 7, 8, 9, 63, 64, 65, 255, 256, 511, 512, 513, 1000, 4096, 4109, 65537, 1 << 18]
    g["crc32c"] = {"blob_seed": 0xC5C, "blob_len": len(blob),
                   "cases": [{"len": n, "crc_in": 0, "crc": lib.ref_crc32c(0, blob[:n], n)} for n in lens] +
                            [{"len": n, "crc_in": 0xDEADBEEF, "crc": lib.ref_crc32c(0xDEADBEEF, blob[:n], n)}
                             for n in (5, 777, 1 << 18)]}
    offs = [0]
    for x in splitmix_stream(0x0FF5, 300):
        offs.append(min(len(blob), offs[-1] + int(x % 3000)))
    g["crc32c"]["batch_offsets"] = offs
    g["crc32c"]["batch_crc"] = [lib.ref_crc32c(0, blob[a:b], b - a) for a, b in zip(offs[:-1], offs[1:])]
    # binary16 widening over all 65,536 patterns, narrowing over 2^20 seeded f32 patterns
    # (NaN payloads, infinities, subnormals included): sha256 of the reference's outputs
    import hashlib
    allh = (C.c_uint16 * 65536)(*range(65536))
    wide = (C.c_float * 65536)()
    lib.ref_force_scalar(1)
    lib.ref_f16_to_f32(allh, wide, 65536)
    g["f16_to_f32_all_sha256"] = hashlib.sha256(bytes(wide)).hexdigest()
    bits = [x & 0xFFFFFFFF for x in splitmix_stream(0xF16, 1 << 20)]
    src = (C.c_uint32 * len(bits))(*bits)
    nar = (C.c_uint16 * len(bits))()
    lib.ref_f32_to_f16(C.cast(src, C.POINTER(C.c_float)), nar, len(bits))
    lib.ref_force_scalar(0)
    g["f32_to_f16_sample"] = {"seed": 0xF16, "n": len(bits), "sha256": hashlib.sha256(bytes(nar)).hexdigest()}
    g["error_code_name"] = {str(c): lib.ref_error_code_name(c).decode() for c in range(0, 19)}
    g["validate_dim"] = {str(d): lib.ref_validate_dim(d) for d in [0, 1, 16, 4096, 4097, 65535]}
    ev = {}
    for k, v in cases.items():
        if not v:
            continue
        arr = (C.c_float * len(v))(*v)
        ev[k] = lib.ref_embedding_vector_f32(arr, len(v))
    g["embedding_vector_f32_status"] = ev
    g["table_meta_make"] = {
        "ok": lib.ref_table_meta_make(b"ads", 16, 16),
        "dim_mismatch": lib.ref_table_meta_make(b"ads", 16, 8),
        "empty_name": lib.ref_table_meta_make(b"", 16, 16),
        "long_name": lib.ref_table_meta_make(b"x" * 256, 16, 16),
        "bad_dim": lib.ref_table_meta_make(b"ads", 0, 1),
    }
    out = os.path.join(HERE, "..", "tests", "golden", "ref_vectors.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", os.path.normpath(out), len(keys), "keys")


if __name__ == "__main__":
    main()
