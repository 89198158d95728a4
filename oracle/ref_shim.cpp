// oracle/ref_shim.cpp — C entry points over the REFERENCE's own code, for pinning the oracle.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against the untouched sources
// under /root/reference/proj (include/hps/*.hpp, src/core/types.cpp,
// src/kernels/*.cpp); nothing here is copied from them. The result,
// oracle/_ref/libhps_ref.so, is what tests/golden/ref_vectors.json was generated
// from (oracle/gen_golden.py) and what the CPU baseline may call for key_hash.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include <hps/bytes.hpp>
#include <hps/error.hpp>
#include <hps/hash.hpp>
#include <hps/kernels.hpp>
#include <hps/types.hpp>

extern "C" {

uint64_t ref_key_hash(uint64_t key) { return hps::key_hash(key); }                    // hash.hpp:42
uint32_t ref_partition_of(uint64_t key, uint32_t n) { return hps::partition_of(key, n); }  // hash.hpp:52
uint64_t ref_fnv1a64(const uint8_t* p, uint64_t n) {                                  // hash.hpp:30
  return hps::fnv1a64(std::span<const std::byte>(reinterpret_cast<const std::byte*>(p), n));
}
void ref_key_hash_n(const uint64_t* keys, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = hps::key_hash(keys[i]);
}
void ref_f32_to_f16(const float* src, uint16_t* dst, uint64_t n) { hps::kernels::f32_to_f16(src, dst, n); }
void ref_f16_to_f32(const uint16_t* src, float* dst, uint64_t n) { hps::kernels::f16_to_f32(src, dst, n); }
uint32_t ref_crc32c(uint32_t crc, const void* p, uint64_t n) { return hps::kernels::crc32c(crc, p, n); }
int ref_has_non_finite_f32(const float* v, uint64_t n) { return hps::kernels::has_non_finite_f32(v, n); }
int ref_has_non_finite_f16(const uint16_t* v, uint64_t n) { return hps::kernels::has_non_finite_f16(v, n); }
const char* ref_active_backend() { return hps::kernels::active_backend(); }
void ref_force_scalar(int on) { hps::kernels::force_scalar(on != 0); }
const char* ref_error_code_name(int code) { return hps::error_code_name(static_cast<hps::ErrorCode>(code)); }

// EmbeddingVector::f32 (types.cpp:67-77): 0 on success, else the ErrorCode it raised.
int ref_embedding_vector_f32(const float* v, uint64_t n) {
  try {
    auto ev = hps::EmbeddingVector::f32(std::span<const float>(v, n));
    return ev.dim() == n ? 0 : -1;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}
int ref_validate_dim(uint32_t dim) {
  try {
    hps::validate_dim(dim);
    return 0;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}
// TableMeta::make with a default vector of `dv_dim` zeros (types.cpp:136-152).
int ref_table_meta_make(const char* name, uint32_t dim, uint32_t dv_dim) {
  try {
    auto dv = hps::EmbeddingVector::zeros(static_cast<uint16_t>(dv_dim));
    auto m = hps::TableMeta::make(name, static_cast<uint16_t>(dim), hps::Dtype::F32, dv);
    return m.dim == dim ? 0 : -1;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}


// UpdateBatch codec built on the reference's OWN ByteWriter / ByteReader
// (bytes.hpp:33-133): the reference ships the primitives but no codec, so this restates
// the SPEC layout over them. encode: 0 or an ErrorCode; *out_len = frame size.
int ref_update_encode(const char* name, uint32_t name_len, uint64_t seq, uint32_t count, uint32_t dim, int dtype,
                      const uint64_t* keys, const void* values, uint8_t* out, uint64_t cap, uint64_t* out_len) {
  try {
    if (name_len > 255) hps::raise(hps::ErrorCode::InvalidArgument, "name length > 255");
    hps::ByteWriter w;
    w.bytes(std::string_view("HPSU", 4));
    w.u8(1);
    w.u16(static_cast<uint16_t>(name_len));
    w.bytes(std::string_view(name, name_len));
    w.u64(seq);
    w.u32(count);
    w.u16(static_cast<uint16_t>(dim));
    w.u8(static_cast<uint8_t>(dtype));
    const size_t esz = dtype == 0 ? 4 : 2;
    for (uint32_t e = 0; e < count; ++e) {
      w.u64(keys[e]);
      for (uint32_t j = 0; j < dim; ++j) {
        if (dtype == 0) {
          uint32_t b;
          std::memcpy(&b, static_cast<const uint8_t*>(values) + (size_t(e) * dim + j) * esz, 4);
          w.u32(b);
        } else {
          uint16_t b;
          std::memcpy(&b, static_cast<const uint8_t*>(values) + (size_t(e) * dim + j) * esz, 2);
          w.u16(b);
        }
      }
    }
    *out_len = w.size();
    if (out) {
      if (cap < w.size()) return 1;
      std::memcpy(out, w.view().data(), w.size());
    }
    return 0;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}

// decode: 0 or the ErrorCode (BadMagic 2, BadFormatVersion 3, Truncated 4 — from
// ByteReader::need —, TrailingBytes 5, DuplicateKey 6). Outputs: header fields, keys,
// values as raw scalars (count x dim x esz bytes).
int ref_update_decode(const uint8_t* frame, uint64_t n, char* name_out, uint64_t* seq, uint32_t* count, uint32_t* dim,
                      int* dtype, uint64_t* keys_out, uint8_t* values_out, uint64_t max_count) {
  try {
    hps::ByteReader r(std::span<const std::byte>(reinterpret_cast<const std::byte*>(frame), n));
    if (r.str(4) != "HPSU") hps::raise(hps::ErrorCode::BadMagic, "bad magic");
    if (r.u8() != 1) hps::raise(hps::ErrorCode::BadFormatVersion, "format version");
    const uint16_t nl = r.u16();
    const std::string name = r.str(nl);
    std::memcpy(name_out, name.data(), nl);
    name_out[nl] = 0;
    *seq = r.u64();
    *count = r.u32();
    *dim = r.u16();
    const uint8_t dt = r.u8();
    *dtype = static_cast<int>(hps::dtype_from_byte(dt));
    const size_t esz = hps::scalar_size(static_cast<hps::Dtype>(*dtype));
    std::vector<uint64_t> seen;
    for (uint32_t e = 0; e < *count; ++e) {
      const uint64_t k = r.u64();
      auto v = r.bytes(size_t(*dim) * esz);
      seen.push_back(k);
      if (e < max_count) {
        keys_out[e] = k;
        std::memcpy(values_out + size_t(e) * *dim * esz, v.data(), v.size());
      }
    }
    if (!r.done()) hps::raise(hps::ErrorCode::TrailingBytes, "trailing bytes");
    std::sort(seen.begin(), seen.end());
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end()) hps::raise(hps::ErrorCode::DuplicateKey, "dup");
    return 0;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}

}  // extern "C"
