// API conformance: this translation unit uses only declarations the reference exports
// (proj/include/hps/{types,hash,error}.hpp). tests/test_api_conformance.py compiles it
// against BOTH header trees — the reference's and include/hps — so any drift in names,
// signatures, enum values or constants breaks the build.
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include <hps/error.hpp>
#include <hps/hash.hpp>
#include <hps/types.hpp>

static_assert(static_cast<int>(hps::ErrorCode::InvalidArgument) == 1);
static_assert(static_cast<int>(hps::ErrorCode::NonFinite) == 10);
static_assert(static_cast<int>(hps::ErrorCode::Infeasible) == 16);
static_assert(static_cast<int>(hps::ErrorCode::Protocol) == 17);
static_assert(static_cast<int>(hps::Dtype::F32) == 0 && static_cast<int>(hps::Dtype::F16) == 1);
static_assert(hps::kMaxDim == 4096 && hps::kMaxTableNameBytes == 255 && hps::kBulkLoadVersion == 0);
static_assert(hps::kFnv1a64OffsetBasis == 0xcbf29ce484222325ull && hps::kFnv1a64Prime == 0x100000001b3ull);
static_assert(hps::key_hash(0) == 0xa8c7f832281a39c5ull);
static_assert(hps::partition_of(0, 8) == 5);
static_assert(hps::fnv1a64(std::span<const std::byte>{}) == 0xcbf29ce484222325ull);

int conformance_uses() {
  hps::EmbeddingKey k = 42;
  std::uint32_t (*part)(hps::EmbeddingKey, std::uint32_t) = &hps::partition_of;
  std::uint64_t (*kh)(hps::EmbeddingKey) = &hps::key_hash;
  (void)part;
  (void)kh;
  const char* (*name)(hps::ErrorCode) = &hps::error_code_name;
  (void)name;
  void (*vd)(std::uint32_t) = &hps::validate_dim;
  void (*vt)(const hps::TableName&) = &hps::validate_table_name;
  hps::Dtype (*db)(std::uint8_t) = &hps::dtype_from_byte;
  (void)vd;
  (void)vt;
  (void)db;
  std::size_t ss = hps::scalar_size(hps::Dtype::F16);
  std::vector<float> v(4, 1.0f);
  hps::EmbeddingVector ev = hps::EmbeddingVector::f32(std::span<const float>(v));
  hps::EmbeddingVector z = hps::EmbeddingVector::zeros(4, hps::Dtype::F32);
  std::vector<std::byte> raw(16);
  hps::EmbeddingVector fb = hps::EmbeddingVector::from_bytes(4, hps::Dtype::F32, std::span<const std::byte>(raw));
  hps::EmbeddingVector fu = hps::EmbeddingVector::from_bytes_unchecked(4, hps::Dtype::F32, raw);
  std::vector<std::uint16_t> h(4, 0x3c00);
  hps::EmbeddingVector e16 = hps::EmbeddingVector::f16(std::span<const std::uint16_t>(h));
  std::span<const float> fv = ev.f32_values();
  std::span<const std::uint16_t> hv = e16.f16_bits();
  std::span<const std::byte> bytes = ev.bytes();
  bool same = (ev == fu) && z.dim() == 4 && !z.empty() && z.byte_size() == 16 && z.dtype() == hps::Dtype::F32;
  hps::VersionedEntry ve{k, ev, hps::kBulkLoadVersion};
  hps::TableMeta m = hps::TableMeta::make("ads", 4);
  hps::TableMeta m2 = hps::TableMeta::make("ads", 4, hps::Dtype::F32, z);
  m.validate();
  try {
    hps::raise(hps::ErrorCode::Io, "x");
  } catch (const hps::Error& e) {
    same = same && e.code() == hps::ErrorCode::Io;
  }
  return static_cast<int>(ss + fv.size() + hv.size() + bytes.size() + fb.dim() + (ve == ve) + (m == m2) + same);
}
