// oracle/ref_shim.cpp — C entry points over the REFERENCE's own code, for pinning the oracle.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against the untouched sources
// under /root/reference/proj (include/hps/*.hpp, src/core/types.cpp,
// src/kernels/*.cpp); nothing here is copied from them. The result,
// oracle/_ref/libhps_ref.so, is what tests/golden/ref_vectors.json was generated
// from (oracle/gen_golden.py) and what the CPU baseline may call for key_hash.
#include <cstdint>
#include <cstring>
#include <span>

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

}  // extern "C"
