// hps/gpu.hpp — C++ host API over the C-ABI (include/hps_gpu.h), in the reference's vocabulary.
//
// The reference's core model (proj/include/hps/types.hpp:29-107) speaks in EmbeddingKey,
// EmbeddingVector, VersionedEntry and TableMeta, and raises hps::Error(ErrorCode, msg) on
// failure (error.hpp:46-56). These wrappers keep that contract for the B200 path:
//   * hps::gpu::HotCache   — SPEC.md:112-190 query / insert / refresh / stats over host spans
//   * hps::gpu::EmbeddingTable — insert / find / export by key; the training hot path
//     (lookup_pooled, backward_update) takes DEVICE pointers and is stream-ordered
// Every C-ABI status != 0 becomes hps::Error with the matching ErrorCode.
// Header-only; link with libhps_gpu.so and cudart.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include <hps/error.hpp>
#include <hps/types.hpp>
#include "hps_gpu.h"

namespace hps::gpu {

inline void check(int status, const char* what) {
  if (status != HPS_GPU_OK)
    raise(error_code_from_status(status), std::string(what) + ": " + hps_gpu_status_string(status) + " " +
                                              hps_gpu_last_error_message());
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(ErrorCode::Io, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer owned by the wrappers (staging for host spans).
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) { resize(n); }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void resize(size_t n) {
    if (n <= n_) return;
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
    cuda_check(cudaMalloc(&p_, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    n_ = n;
  }
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

class Context {
 public:
  explicit Context(int device = 0, cudaStream_t stream = nullptr) : stream_(stream) {
    check(hps_gpu_ctx_create(device, stream, &h_), "hps_gpu_ctx_create");
  }
  ~Context() { hps_gpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  hps_gpu_ctx handle() const { return h_; }
  cudaStream_t stream() const { return stream_; }
  /// Waits for the stream; raises the first data error a kernel latched (NonFinite, Infeasible, ...).
  void sync() { check(hps_gpu_ctx_sync(h_), "hps_gpu_ctx_sync"); }

 private:
  hps_gpu_ctx h_ = nullptr;
  cudaStream_t stream_ = nullptr;
};

namespace detail {
// binary16 <-> fp32 on the host for F16 tables: the device stores binary16; rows travel as
// fp32. Widening is exact, and so is narrowing a widened binary16 value.
inline float f16_bits_to_float(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  uint32_t b;
  if (e == 31) {
    b = sign | 0x7f800000u | (m << 13);
  } else if (e) {
    b = sign | ((e + 112u) << 23) | (m << 13);
  } else if (!m) {
    b = sign;
  } else {
    int k = 0;
    uint32_t mm = m;
    while (!(mm & 0x400u)) mm <<= 1, ++k;
    b = sign | (static_cast<uint32_t>(113 - k) << 23) | ((mm & 0x3ffu) << 13);
  }
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}
inline uint16_t float_to_f16_bits(float f) {  // round to nearest even; |f| beyond range -> inf
  uint32_t b;
  std::memcpy(&b, &f, 4);
  const uint32_t sign = (b >> 16) & 0x8000u, a = b & 0x7fffffffu;
  if (a >= 0x7f800000u) return static_cast<uint16_t>(sign | 0x7c00u | (a > 0x7f800000u ? 0x200u : 0u));
  const int e = static_cast<int>(a >> 23) - 112;
  if (e >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return static_cast<uint16_t>(sign);
    const uint32_t m = (a & 0x7fffffu) | 0x800000u, sh = static_cast<uint32_t>(14 - e);
    uint32_t q = m >> sh;
    const uint32_t r = m & ((1u << sh) - 1u), half = 1u << (sh - 1u);
    if (r > half || (r == half && (q & 1u))) ++q;
    return static_cast<uint16_t>(sign | q);
  }
  uint32_t q = (static_cast<uint32_t>(e) << 10) | ((a >> 13) & 0x3ffu);
  const uint32_t r = a & 0x1fffu;
  if (r > 0x1000u || (r == 0x1000u && (q & 1u))) ++q;
  return static_cast<uint16_t>(sign | q);
}

// fp32 rows of the entries; their vectors must have the table's dtype (F16 rows widen).
inline std::vector<float> rows_of(std::span<const VersionedEntry> entries, uint16_t dim, Dtype dtype = Dtype::F32) {
  std::vector<float> rows(entries.size() * dim);
  for (size_t i = 0; i < entries.size(); ++i) {
    const EmbeddingVector& v = entries[i].vector;
    if (v.dtype() != dtype) raise(ErrorCode::DtypeMismatch, "entry dtype does not match the table");
    if (v.dim() != dim) raise(ErrorCode::DimMismatch, "entry dim does not match the table");
    if (dtype == Dtype::F32) {
      std::memcpy(rows.data() + i * dim, v.bytes().data(), dim * sizeof(float));
    } else {
      const auto bits = v.f16_bits();
      for (uint16_t j = 0; j < dim; ++j) rows[i * dim + j] = f16_bits_to_float(bits[j]);
    }
  }
  return rows;
}
}  // namespace detail

/// HPS GPU embedding cache for one table.
class HotCache {
 public:
  struct QueryResult {
    std::vector<std::pair<EmbeddingKey, EmbeddingVector>> found;  // input order
    std::vector<EmbeddingKey> missing;                            // input order
  };

  HotCache(Context& ctx, TableMeta meta, uint64_t capacity, uint32_t ways = 8, uint64_t aging_interval = 0,
           uint64_t max_batch = 1 << 17)
      : ctx_(ctx), meta_(std::move(meta)), max_batch_(max_batch) {
    meta_.validate();
    // F16 tables: rows held as binary16 on the device (hps_cache_config.dtype)
    const hps_cache_config cfg{capacity, ways, aging_interval, meta_.dim, max_batch,
                               meta_.dtype == Dtype::F16 ? uint32_t(HPS_DTYPE_F16) : uint32_t(HPS_DTYPE_F32)};
    check(hps_gpu_cache_create(ctx.handle(), &cfg, &h_), "hps_gpu_cache_create");
  }
  ~HotCache() { hps_gpu_cache_destroy(h_); }
  hps_gpu_cache handle() const { return h_; }  // for C-ABI entries that take the cache (e.g. hps_gpu_tiered_create)
  HotCache(const HotCache&) = delete;
  HotCache& operator=(const HotCache&) = delete;

  const TableMeta& meta() const { return meta_; }

  QueryResult query(std::span<const EmbeddingKey> keys) {
    QueryResult r;
    for (size_t b = 0; b < keys.size(); b += max_batch_) {
      const size_t n = std::min<size_t>(max_batch_, keys.size() - b);
      keys_.resize(n);
      vecs_.resize(n * meta_.dim);
      fidx_.resize(n);
      midx_.resize(n);
      counts_.resize(2);
      cuda_check(cudaMemcpyAsync(keys_.get(), keys.data() + b, n * 8, cudaMemcpyHostToDevice, ctx_.stream()), "H2D");
      check(hps_gpu_cache_query(h_, keys_.get(), n, vecs_.get(), fidx_.get(), midx_.get(), counts_.get()),
            "hps_gpu_cache_query");
      uint64_t c[2];
      cuda_check(cudaMemcpyAsync(c, counts_.get(), 16, cudaMemcpyDeviceToHost, ctx_.stream()), "D2H");
      ctx_.sync();
      std::vector<uint32_t> fi(c[0]), mi(c[1]);
      std::vector<float> fv(c[0] * meta_.dim);
      if (c[0]) {
        cuda_check(cudaMemcpy(fi.data(), fidx_.get(), c[0] * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(fv.data(), vecs_.get(), fv.size() * 4, cudaMemcpyDeviceToHost), "D2H");
      }
      if (c[1]) cuda_check(cudaMemcpy(mi.data(), midx_.get(), c[1] * 4, cudaMemcpyDeviceToHost), "D2H");
      for (uint64_t j = 0; j < c[0]; ++j) {
        if (meta_.dtype == Dtype::F16) {  // exact: the device holds binary16
          std::vector<uint16_t> bits(meta_.dim);
          for (uint16_t q = 0; q < meta_.dim; ++q) bits[q] = detail::float_to_f16_bits(fv[j * meta_.dim + q]);
          r.found.emplace_back(keys[b + fi[j]], EmbeddingVector::f16(bits));
          continue;
        }
        std::vector<std::byte> bytes(meta_.dim * sizeof(float));
        std::memcpy(bytes.data(), fv.data() + j * meta_.dim, bytes.size());
        r.found.emplace_back(keys[b + fi[j]],
                             EmbeddingVector::from_bytes_unchecked(meta_.dim, Dtype::F32, std::move(bytes)));
      }
      for (uint64_t j = 0; j < c[1]; ++j) r.missing.push_back(keys[b + mi[j]]);
    }
    return r;
  }

  /// Admitted (newly inserted) entries. Resident keys take refresh semantics.
  uint64_t insert(std::span<const VersionedEntry> entries) { return apply(entries, true); }
  /// Replacements (resident keys with a newer version); never inserts.
  uint64_t refresh(std::span<const VersionedEntry> entries) { return apply(entries, false); }

  /// Refresh from one encoded UpdateBatch frame: resident keys with an
  /// older version take the frame's vectors at version = seq. Returns replacements.
  uint64_t apply_update(std::span<const std::byte> frame) {
    counts_.resize(2);
    check(hps_gpu_cache_apply_update(h_, reinterpret_cast<const uint8_t*>(frame.data()), frame.size(), counts_.get()),
          "hps_gpu_cache_apply_update");
    uint64_t n = 0;
    cuda_check(cudaMemcpy(&n, counts_.get(), 8, cudaMemcpyDeviceToHost), "D2H");
    return n;
  }

  hps_cache_stats stats() {
    hps_cache_stats s{};
    check(hps_gpu_cache_stats(h_, &s), "hps_gpu_cache_stats");
    return s;
  }
  void reset_stats() { check(hps_gpu_cache_reset_stats(h_), "hps_gpu_cache_reset_stats"); }
  uint64_t size() {
    uint64_t n = 0;
    check(hps_gpu_cache_size(h_, &n), "hps_gpu_cache_size");
    return n;
  }

 private:
  uint64_t apply(std::span<const VersionedEntry> entries, bool insert) {
    uint64_t total = 0;
    for (size_t b = 0; b < entries.size(); b += max_batch_) {
      const size_t n = std::min<size_t>(max_batch_, entries.size() - b);
      auto part = entries.subspan(b, n);
      std::vector<float> rows = detail::rows_of(part, meta_.dim, meta_.dtype);
      std::vector<uint64_t> k(n), v(n);
      for (size_t i = 0; i < n; ++i) k[i] = part[i].key, v[i] = part[i].version;
      keys_.resize(n);
      vecs_.resize(n * meta_.dim);
      vers_.resize(n);
      counts_.resize(2);
      cuda_check(cudaMemcpyAsync(keys_.get(), k.data(), n * 8, cudaMemcpyHostToDevice, ctx_.stream()), "H2D");
      cuda_check(cudaMemcpyAsync(vers_.get(), v.data(), n * 8, cudaMemcpyHostToDevice, ctx_.stream()), "H2D");
      cuda_check(cudaMemcpyAsync(vecs_.get(), rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, ctx_.stream()),
                 "H2D");
      if (insert)
        check(hps_gpu_cache_insert(h_, keys_.get(), vecs_.get(), vers_.get(), n, counts_.get()), "cache_insert");
      else
        check(hps_gpu_cache_refresh(h_, keys_.get(), vecs_.get(), vers_.get(), n, counts_.get()), "cache_refresh");
      uint64_t c = 0;
      cuda_check(cudaMemcpyAsync(&c, counts_.get(), 8, cudaMemcpyDeviceToHost, ctx_.stream()), "D2H");
      ctx_.sync();
      total += c;
    }
    return total;
  }

  Context& ctx_;
  TableMeta meta_;
  uint64_t max_batch_;
  hps_gpu_cache h_ = nullptr;
  DeviceBuffer<uint64_t> keys_, vers_, counts_;
  DeviceBuffer<float> vecs_;
  DeviceBuffer<uint32_t> fidx_, midx_;
};

enum class Optimizer : int { SGD = HPS_OPT_SGD, AdaGrad = HPS_OPT_ADAGRAD, Adam = HPS_OPT_ADAM };

/// A group of embedding tables (one TableMeta each, same dim) trained together.
class EmbeddingTable {
 public:
  EmbeddingTable(Context& ctx, std::vector<TableMeta> metas, std::vector<uint64_t> row_capacity,
                 std::vector<uint32_t> slot_table, Optimizer opt = Optimizer::SGD, uint64_t max_batch_keys = 1 << 20,
                 uint64_t max_batch_bags = 1 << 20, uint64_t init_seed = 0, float adagrad_a0 = 0.f)
      : ctx_(ctx), metas_(std::move(metas)) {
    if (metas_.empty() || metas_.size() != row_capacity.size())
      raise(ErrorCode::InvalidArgument, "one TableMeta and one capacity per table");
    for (auto& m : metas_) {
      m.validate();
      if (m.dim != metas_[0].dim) raise(ErrorCode::DimMismatch, "tables of one group share a dim");
      if (m.dtype != Dtype::F32) raise(ErrorCode::DtypeMismatch, "the B200 path stores F32 rows");
    }
    const hps_table_config cfg{static_cast<uint32_t>(metas_.size()), metas_[0].dim, row_capacity.data(),
                               static_cast<uint32_t>(slot_table.size()), slot_table.data(), static_cast<int>(opt),
                               max_batch_keys, max_batch_bags, init_seed, adagrad_a0};
    check(hps_gpu_table_create(ctx.handle(), &cfg, &h_), "hps_gpu_table_create");
    for (uint32_t t = 0; t < metas_.size(); ++t) {
      auto v = metas_[t].default_vector.f32_values();
      check(hps_gpu_table_set_default_vector(h_, t, v.data()), "set_default_vector");
    }
  }
  ~EmbeddingTable() { hps_gpu_table_destroy(h_); }
  EmbeddingTable(const EmbeddingTable&) = delete;
  EmbeddingTable& operator=(const EmbeddingTable&) = delete;

  hps_gpu_table handle() const { return h_; }
  uint16_t dim() const { return metas_[0].dim; }

  /// Insert keys (rows initialised deterministically); returns each key's row id.
  std::vector<uint64_t> insert(uint32_t table, std::span<const EmbeddingKey> keys) { return insert_impl(table, keys, nullptr); }

  /// Insert entries with their vectors (the first occurrence of a key wins).
  std::vector<uint64_t> insert(uint32_t table, std::span<const VersionedEntry> entries) {
    std::vector<float> rows = detail::rows_of(entries, dim());
    std::vector<EmbeddingKey> keys(entries.size());
    for (size_t i = 0; i < entries.size(); ++i) keys[i] = entries[i].key;
    return insert_impl(table, keys, &rows);
  }

  /// Vector of each key, or nullopt when absent.
  std::vector<std::optional<EmbeddingVector>> find(uint32_t table, std::span<const EmbeddingKey> keys) {
    const size_t n = keys.size();
    std::vector<std::optional<EmbeddingVector>> out(n);
    if (!n) return out;
    DeviceBuffer<uint64_t> dk(n), dr(n);
    cuda_check(cudaMemcpyAsync(dk.get(), keys.data(), n * 8, cudaMemcpyHostToDevice, ctx_.stream()), "H2D");
    check(hps_gpu_table_find(h_, table, dk.get(), n, dr.get()), "hps_gpu_table_find");
    std::vector<uint64_t> rows(n);
    cuda_check(cudaMemcpyAsync(rows.data(), dr.get(), n * 8, cudaMemcpyDeviceToHost, ctx_.stream()), "D2H");
    ctx_.sync();
    DeviceBuffer<float> w(dim());
    for (size_t i = 0; i < n; ++i) {
      if (rows[i] == ~0ull) continue;
      check(hps_gpu_table_export(h_, table, rows[i], 1, w.get(), nullptr, nullptr), "export");
      std::vector<std::byte> bytes(dim() * sizeof(float));
      cuda_check(cudaMemcpyAsync(bytes.data(), w.get(), bytes.size(), cudaMemcpyDeviceToHost, ctx_.stream()), "D2H");
      ctx_.sync();
      out[i] = EmbeddingVector::from_bytes_unchecked(dim(), Dtype::F32, std::move(bytes));
    }
    return out;
  }

  uint64_t size(uint32_t table) {
    uint64_t n = 0;
    check(hps_gpu_table_size(h_, table, &n), "hps_gpu_table_size");
    return n;
  }

  // ---- training hot path: device pointers, stream-ordered, graph-capturable ----
  void lookup_pooled(const uint64_t* d_keys, const uint32_t* d_offsets, uint32_t n_samples, int combiner, float* d_out,
                     bool train) {
    check(hps_gpu_lookup_pooled(h_, d_keys, d_offsets, n_samples, combiner, d_out, train ? HPS_LOOKUP_TRAIN : 0),
          "hps_gpu_lookup_pooled");
  }
  void backward_update(const float* d_dout, const hps_opt_params& p) {
    check(hps_gpu_backward_update(h_, d_dout, &p), "hps_gpu_backward_update");
  }

 private:
  std::vector<uint64_t> insert_impl(uint32_t table, std::span<const EmbeddingKey> keys, const std::vector<float>* rows) {
    const size_t n = keys.size();
    std::vector<uint64_t> out(n);
    if (!n) return out;
    DeviceBuffer<uint64_t> dk(n), dr(n);
    DeviceBuffer<float> dv;
    cuda_check(cudaMemcpyAsync(dk.get(), keys.data(), n * 8, cudaMemcpyHostToDevice, ctx_.stream()), "H2D");
    if (rows) {
      dv.resize(rows->size());
      cuda_check(cudaMemcpyAsync(dv.get(), rows->data(), rows->size() * 4, cudaMemcpyHostToDevice, ctx_.stream()),
                 "H2D");
    }
    check(hps_gpu_table_insert(h_, table, dk.get(), n, rows ? dv.get() : nullptr, dr.get()), "hps_gpu_table_insert");
    cuda_check(cudaMemcpyAsync(out.data(), dr.get(), n * 8, cudaMemcpyDeviceToHost, ctx_.stream()), "D2H");
    ctx_.sync();  // surfaces NonFinite / Infeasible as hps::Error
    return out;
  }

  Context& ctx_;
  std::vector<TableMeta> metas_;
  hps_gpu_table h_ = nullptr;
};

}  // namespace hps::gpu
