// core_types.cpp — definitions behind include/hps/types.hpp and include/hps/error.hpp.
//
// Behaviour follows the reference's core model (proj/src/core/types.cpp:28-152):
// the same validation rules, the same ErrorCode for each failure, the same
// enumerator names. The finiteness scan is a plain host loop over the exponent
// bits (proj/src/kernels/kernels_scalar.cpp:110-123 semantics); bulk payloads take
// the GPU path instead (hps_gpu_has_non_finite_f32, fused into cache insert/refresh).
#include <bit>
#include <cstring>
#include <string>

#include <hps/error.hpp>
#include <hps/types.hpp>

static_assert(std::endian::native == std::endian::little,
              "payloads are little-endian wire bytes; big-endian hosts are not supported");

namespace hps {
namespace {

constexpr const char* kNames[] = {"InvalidArgument", "BadMagic",     "BadFormatVersion", "Truncated",
                                  "TrailingBytes",   "DuplicateKey", "DimMismatch",      "DtypeMismatch",
                                  "F16Range",        "NonFinite",    "UnknownTable",     "TableExists",
                                  "BadShard",        "Io",           "Corruption",       "Infeasible",
                                  "Protocol"};

template <typename Word, Word kExpMask>
bool any_all_ones_exponent(const Word* v, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if ((v[i] & kExpMask) == kExpMask) return true;
  return false;
}

bool f32_non_finite(const float* v, std::size_t n) {
  static_assert(sizeof(float) == sizeof(std::uint32_t));
  for (std::size_t i = 0; i < n; ++i)
    if ((std::bit_cast<std::uint32_t>(v[i]) & 0x7f800000u) == 0x7f800000u) return true;
  return false;
}

bool f16_non_finite(const std::uint16_t* v, std::size_t n) {
  return any_all_ones_exponent<std::uint16_t, 0x7c00u>(v, n);
}

EmbeddingVector make_vector(std::uint16_t dim, Dtype dtype, const void* src, std::size_t bytes) {
  std::vector<std::byte> data(bytes);
  if (bytes) std::memcpy(data.data(), src, bytes);
  return EmbeddingVector::from_bytes_unchecked(dim, dtype, std::move(data));
}

}  // namespace

const char* error_code_name(ErrorCode code) {
  const int c = static_cast<int>(code);
  return (c >= 1 && c <= 17) ? kNames[c - 1] : "Unknown";
}

void validate_table_name(const TableName& name) {
  if (name.empty()) raise(ErrorCode::InvalidArgument, "table name must not be empty");
  if (name.size() > kMaxTableNameBytes)
    raise(ErrorCode::InvalidArgument, "table name longer than 255 bytes: " + name.substr(0, 32));
}

void validate_dim(std::uint32_t dim) {
  if (dim < 1 || dim > kMaxDim)
    raise(ErrorCode::InvalidArgument, "dim must be in [1, 4096], got " + std::to_string(dim));
}

Dtype dtype_from_byte(std::uint8_t b) {
  switch (b) {
    case 0: return Dtype::F32;
    case 1: return Dtype::F16;
    default: raise(ErrorCode::InvalidArgument, "unknown dtype byte " + std::to_string(b));
  }
}

EmbeddingVector EmbeddingVector::f32(std::span<const float> values) {
  validate_dim(static_cast<std::uint32_t>(values.size()));
  if (f32_non_finite(values.data(), values.size())) raise(ErrorCode::NonFinite, "embedding vector has NaN/Inf");
  return make_vector(static_cast<std::uint16_t>(values.size()), Dtype::F32, values.data(), values.size_bytes());
}

EmbeddingVector EmbeddingVector::f16(std::span<const std::uint16_t> bits) {
  validate_dim(static_cast<std::uint32_t>(bits.size()));
  if (f16_non_finite(bits.data(), bits.size())) raise(ErrorCode::NonFinite, "embedding vector has NaN/Inf");
  return make_vector(static_cast<std::uint16_t>(bits.size()), Dtype::F16, bits.data(), bits.size_bytes());
}

EmbeddingVector EmbeddingVector::zeros(std::uint16_t dim, Dtype dtype) {
  validate_dim(dim);
  return EmbeddingVector::from_bytes_unchecked(dim, dtype, std::vector<std::byte>(dim * scalar_size(dtype)));
}

EmbeddingVector EmbeddingVector::from_bytes(std::uint16_t dim, Dtype dtype, std::span<const std::byte> data) {
  validate_dim(dim);
  if (data.size() != dim * scalar_size(dtype))
    raise(ErrorCode::DimMismatch, "payload is " + std::to_string(data.size()) + " bytes, expected dim*scalar_size");
  std::vector<std::byte> copy(data.begin(), data.end());
  const bool bad = dtype == Dtype::F32
                       ? f32_non_finite(reinterpret_cast<const float*>(copy.data()), dim)
                       : f16_non_finite(reinterpret_cast<const std::uint16_t*>(copy.data()), dim);
  if (bad) raise(ErrorCode::NonFinite, "embedding vector has NaN/Inf");
  return EmbeddingVector::from_bytes_unchecked(dim, dtype, std::move(copy));
}

EmbeddingVector EmbeddingVector::from_bytes_unchecked(std::uint16_t dim, Dtype dtype, std::vector<std::byte> data) {
  EmbeddingVector v;
  v.dim_ = dim;
  v.dtype_ = dtype;
  v.data_ = std::move(data);
  return v;
}

std::span<const float> EmbeddingVector::f32_values() const {
  if (dtype_ != Dtype::F32) raise(ErrorCode::DtypeMismatch, "vector dtype is not F32");
  return {reinterpret_cast<const float*>(data_.data()), dim_};
}

std::span<const std::uint16_t> EmbeddingVector::f16_bits() const {
  if (dtype_ != Dtype::F16) raise(ErrorCode::DtypeMismatch, "vector dtype is not F16");
  return {reinterpret_cast<const std::uint16_t*>(data_.data()), dim_};
}

TableMeta TableMeta::make(TableName table, std::uint16_t dim, Dtype dtype) {
  validate_dim(dim);
  return make(std::move(table), dim, dtype, EmbeddingVector::zeros(dim, dtype));
}

TableMeta TableMeta::make(TableName table, std::uint16_t dim, Dtype dtype, EmbeddingVector default_vector) {
  TableMeta m;
  m.table = std::move(table);
  m.dim = dim;
  m.dtype = dtype;
  m.default_vector = std::move(default_vector);
  m.validate();
  return m;
}

void TableMeta::validate() const {
  validate_table_name(table);
  validate_dim(dim);
  if (default_vector.dim() != dim || default_vector.dtype() != dtype)
    raise(ErrorCode::DimMismatch, "default vector does not match the table's dim/dtype");
}

}  // namespace hps

// C entry points used by the Python conformance tests (no exceptions cross the ABI).
extern "C" {
const char* hps_error_code_name(int code) { return hps::error_code_name(static_cast<hps::ErrorCode>(code)); }
int hps_validate_dim(unsigned dim) {
  try {
    hps::validate_dim(dim);
    return 0;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}
int hps_embedding_vector_f32_status(const float* v, unsigned long long n) {
  try {
    auto ev = hps::EmbeddingVector::f32(std::span<const float>(v, n));
    return ev.dim() == n ? 0 : -1;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}
int hps_table_meta_make_status(const char* name, unsigned dim, unsigned default_dim) {
  try {
    auto m = hps::TableMeta::make(name, static_cast<std::uint16_t>(dim), hps::Dtype::F32,
                                  hps::EmbeddingVector::zeros(static_cast<std::uint16_t>(default_dim)));
    return m.dim == dim ? 0 : -1;
  } catch (const hps::Error& e) {
    return static_cast<int>(e.code());
  }
}
}
