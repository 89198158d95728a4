// exchange.cu — device-side halves of the model-parallel embedding exchange
// (distributed and localized slot placement).
//
// Distributed slot (key -> owner = partition_of(key, G), hash.hpp:52-54), per step:
//   requester  hps_gpu_xplan_bucketize   stable counting sort of the occurrences by owner
//                                         (1-pass radix over log2(G) bits) -> send buffers,
//                                         per-owner counts, and perm[i] = send position
//   (NCCL all-to-all: keys, tables)       -- torch.distributed, paper_2210_08803_b200/exchange.py
//   owner      hps_gpu_gather_rows        rows of the received keys (table.cu), training state
//   (NCCL all-to-all: rows back)
//   requester  hps_gpu_pool_rows          bag pooling straight from the received row buffer
//   requester  hps_gpu_scatter_grads      per-occurrence gradients laid out in send order
//   (NCCL all-to-all: gradients)
//   owner      hps_gpu_backward_update    dedup + reduction + optimizer (backward.cu)
// Stability everywhere keeps every key's occurrences in global canonical order (ranks in
// order, then each rank's own order), so the sharded step is bit-identical to one table.
//
// Localized slot (slot -> owner by the LPT plan), per step:
//   requester  hps_gpu_regroup_bags       the bags of the slots one owner holds, as CSR
//   owner      hps_gpu_lookup_pooled / hps_gpu_backward_update on its tables
//   both       hps_gpu_place_pooled       [B x S_o x D] <-> [B x S x D] slot placement
#include <algorithm>

#include "common.cuh"
#include "primitives.cuh"

using namespace hpsg;

struct hps_gpu_xplan_s {
  hps_gpu_ctx ctx = nullptr;
  uint64_t max_keys = 0;
  uint32_t n_shards = 0;
  int bits = 1;
  uint32_t *owners = nullptr, *owners_b = nullptr, *idx_a = nullptr, *idx_b = nullptr, *sort_ws = nullptr;
  uint64_t* d_n = nullptr;
  size_t sort_words = 0;
};

namespace {

__global__ void k_owner(const uint64_t* __restrict__ keys, uint64_t n, uint32_t n_shards, hps::FastMod64 fm,
                        uint32_t* __restrict__ owners, uint64_t* d_n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_n = n;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    owners[i] = n_shards == 1 ? 0u : static_cast<uint32_t>(fm.mod(hps::key_hash(keys[i])));
}

__global__ void k_pack(const uint64_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ sorted_idx,
                       const uint32_t* __restrict__ occ_bag, uint32_t n_slots, const uint32_t* __restrict__ slot_table,
                       uint64_t* __restrict__ send_keys, uint32_t* __restrict__ send_tables,
                       uint32_t* __restrict__ perm) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t i = sorted_idx ? sorted_idx[p] : static_cast<uint32_t>(p);  // (one owner: identity)
    const uint32_t bag = occ_bag ? occ_bag[i] : i;
    send_keys[p] = keys[i];
    send_tables[p] = slot_table[bag % n_slots];
    perm[i] = static_cast<uint32_t>(p);
  }
}

__global__ void k_count_all(uint32_t* counts, uint32_t n) {
  if (threadIdx.x == 0) counts[0] = n;
}

__global__ void k_counts(const uint32_t* __restrict__ hist, uint32_t n_shards, uint32_t* __restrict__ counts) {
  for (uint32_t g = threadIdx.x; g < n_shards; g += blockDim.x) counts[g] = hist[g];
}

__global__ void k_occ_bags(const uint32_t* __restrict__ offsets, uint64_t n_bags, uint32_t* __restrict__ occ_bag) {
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < n_bags; b += uint64_t(gridDim.x) * blockDim.x)
    for (uint32_t i = offsets[b]; i < offsets[b + 1]; ++i) occ_bag[i] = static_cast<uint32_t>(b);
}

// out[bag] = combiner over rows[perm[i]] for the bag's occurrences, in bag order.
template <int LPR>
__global__ void __launch_bounds__(256) k_pool_rows(const float* __restrict__ rows, const uint32_t* __restrict__ perm,
                                                   const uint32_t* __restrict__ offsets, uint64_t n_bags, uint32_t dim,
                                                   int mean, float* __restrict__ out) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t b = gid; b < n_bags; b += ng) {
    const uint32_t lo = offsets ? offsets[b] : static_cast<uint32_t>(b);
    const uint32_t hi = offsets ? offsets[b + 1] : static_cast<uint32_t>(b + 1);
    float4* o = reinterpret_cast<float4*>(out + b * dim);
    for (uint32_t v = gl; v < nvec; v += LPR) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t i = lo; i < hi; ++i)
        acc = f4_add(acc, __ldg(reinterpret_cast<const float4*>(rows + uint64_t(perm[i]) * dim) + v));
      if (mean && hi > lo) acc = f4_div(acc, static_cast<float>(hi - lo));
      o[v] = acc;
    }
  }
}

// grads[perm[i]] = d_out[bag(i)] (/ len for mean), for every occurrence i.
template <int LPR>
__global__ void __launch_bounds__(256) k_scatter_grads(const float* __restrict__ dout, const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ offsets, uint64_t n_bags,
                                                       uint32_t dim, int mean, float* __restrict__ grads) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t b = gid; b < n_bags; b += ng) {
    const uint32_t lo = offsets ? offsets[b] : static_cast<uint32_t>(b);
    const uint32_t hi = offsets ? offsets[b + 1] : static_cast<uint32_t>(b + 1);
    const float fl = static_cast<float>(hi - lo);
    const float4* d = reinterpret_cast<const float4*>(dout + b * dim);
    for (uint32_t v = gl; v < nvec; v += LPR) {
      float4 x = __ldg(d + v);
      if (mean) x = f4_div(x, fl);
      for (uint32_t i = lo; i < hi; ++i) reinterpret_cast<float4*>(grads + uint64_t(perm[i]) * dim)[v] = x;
    }
  }
}

// Localized: the bags of the selected slots, sample-major, as CSR (lengths then a scan).
__global__ void k_sel_lengths(const uint32_t* __restrict__ offsets, uint32_t n_samples, uint32_t n_slots,
                              const uint32_t* __restrict__ sel, uint32_t n_sel, uint32_t* __restrict__ lens) {
  const uint64_t n = uint64_t(n_samples) * n_sel;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = (k / n_sel) * n_slots + sel[k % n_sel];
    lens[k] = offsets ? offsets[b + 1] - offsets[b] : 1u;
  }
}

struct OffsetsOp {
  const uint32_t* lens;
  uint32_t* out_offsets;
  uint64_t n;
  __device__ uint64_t size() const { return n; }
  __device__ uint32_t count(uint64_t k) const { return lens[k]; }
  __device__ void emit(uint64_t k, uint64_t excl, uint64_t) const { out_offsets[k] = static_cast<uint32_t>(excl); }
  __device__ void total(uint64_t t) const { out_offsets[n] = static_cast<uint32_t>(t); }
};

__global__ void k_sel_keys(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ offsets, uint32_t n_samples,
                           uint32_t n_slots, const uint32_t* __restrict__ sel, uint32_t n_sel,
                           const uint32_t* __restrict__ out_offsets, uint64_t* __restrict__ out_keys) {
  const uint64_t n = uint64_t(n_samples) * n_sel;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = (k / n_sel) * n_slots + sel[k % n_sel];
    const uint32_t lo = offsets ? offsets[b] : static_cast<uint32_t>(b);
    const uint32_t hi = offsets ? offsets[b + 1] : static_cast<uint32_t>(b + 1);
    const uint32_t o = out_offsets[k];
    for (uint32_t i = lo; i < hi; ++i) out_keys[o + (i - lo)] = keys[i];
  }
}

// direction 0: dst[b*S + sel[j]] = src[b*n_sel + j]; 1: dst[b*n_sel + j] = src[b*S + sel[j]].
template <int LPR>
__global__ void __launch_bounds__(256) k_place(const float* __restrict__ src, const uint32_t* __restrict__ sel,
                                               uint32_t n_sel, uint32_t n_samples, uint32_t n_slots, uint32_t dim,
                                               int direction, float* __restrict__ dst) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t n = uint64_t(n_samples) * n_sel;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t k = gid; k < n; k += ng) {
    const uint64_t full = (k / n_sel) * n_slots + sel[k % n_sel];
    const uint64_t s = direction == 0 ? k : full, d = direction == 0 ? full : k;
    const float4* sp = reinterpret_cast<const float4*>(src + s * dim);
    float4* dp = reinterpret_cast<float4*>(dst + d * dim);
    for (uint32_t v = gl; v < nvec; v += LPR) dp[v] = __ldg(sp + v);
  }
}

// Hybrid: per-cold-occurrence gradient rows in send order: out[perm[c]] = d_out[bag_c] (/len).
template <int LPR>
__global__ void __launch_bounds__(256) k_cold_grads(const float* __restrict__ dout, const uint32_t* __restrict__ bags,
                                                    const uint32_t* __restrict__ perm,
                                                    const uint32_t* __restrict__ offsets, uint64_t n, uint32_t dim,
                                                    int mean, float* __restrict__ out) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t c = gid; c < n; c += ng) {
    const uint32_t b = bags[c];
    const float len = (mean && offsets) ? static_cast<float>(offsets[b + 1] - offsets[b]) : 1.f;
    const float4* src = reinterpret_cast<const float4*>(dout + uint64_t(b) * dim);
    float4* dst = reinterpret_cast<float4*>(out + uint64_t(perm[c]) * dim);
    for (uint32_t v = gl; v < nvec; v += LPR) {
      float4 x = __ldg(src + v);
      if (mean) x = f4_div(x, len);
      dst[v] = x;
    }
  }
}

// Hybrid hot-row all-reduce, deterministic: out[r] = sum over parts p in order of the parts
// that touched r (the first such part starts the sum), touched_out[r] = any.
__global__ void k_sum_partials(const float* __restrict__ parts, const uint32_t* __restrict__ touched,
                               uint32_t n_parts, uint64_t rows, uint32_t dim, float* __restrict__ out,
                               uint32_t* __restrict__ touched_out) {
  const uint64_t total = rows * dim;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / dim;
    float acc = 0.f;
    bool any = false;
    for (uint32_t p = 0; p < n_parts; ++p) {
      if (!touched[uint64_t(p) * rows + r]) continue;
      const float x = parts[uint64_t(p) * total + i];
      acc = any ? __fadd_rn(acc, x) : x;
      any = true;
    }
    out[i] = acc;
    if (i % dim == 0) touched_out[r] = any ? 1u : 0u;
  }
}

int lpr_of(uint32_t dim) {
  const uint32_t nvec = dim / 4;
  return nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
}

#define HPSG_LPR_LAUNCH(KERNEL, LPR, GRID, ...)                                     \
  do {                                                                              \
    switch (LPR) {                                                                  \
      case 32: KERNEL<32><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                \
      case 16: KERNEL<16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                \
      case 8: KERNEL<8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                  \
      case 4: KERNEL<4><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                  \
      case 2: KERNEL<2><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                  \
      default: KERNEL<1><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;                 \
    }                                                                               \
  } while (0)

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

}  // namespace

extern "C" {

int hps_gpu_xplan_create(hps_gpu_ctx ctx, uint64_t max_keys, uint32_t n_shards, hps_gpu_xplan* out) {
  if (!ctx || !out || n_shards == 0 || n_shards > 256 || max_keys == 0 || max_keys >= (1ull << 31))
    return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaSetDevice(ctx->device));
  auto p = new hps_gpu_xplan_s;
  p->ctx = ctx;
  p->max_keys = max_keys;
  p->n_shards = n_shards;
  p->bits = std::max(1, bits_for(n_shards - 1));
  p->sort_words = sort_ws_words(max_keys, 1);
  bool ok = cudaMalloc(&p->owners, max_keys * 4) == cudaSuccess && cudaMalloc(&p->owners_b, max_keys * 4) == cudaSuccess &&
            cudaMalloc(&p->idx_a, max_keys * 4) == cudaSuccess && cudaMalloc(&p->idx_b, max_keys * 4) == cudaSuccess &&
            cudaMalloc(&p->sort_ws, p->sort_words * 4) == cudaSuccess && cudaMalloc(&p->d_n, 8) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    hps_gpu_xplan_destroy(p);
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  *out = p;
  return HPS_GPU_OK;
}

int hps_gpu_xplan_destroy(hps_gpu_xplan p) {
  if (!p) return HPS_GPU_OK;
  for (void* q : {static_cast<void*>(p->owners), static_cast<void*>(p->owners_b), static_cast<void*>(p->idx_a),
                  static_cast<void*>(p->idx_b), static_cast<void*>(p->sort_ws), static_cast<void*>(p->d_n)})
    if (q) cudaFree(q);
  delete p;
  return HPS_GPU_OK;
}

int hps_gpu_occurrence_bags(hps_gpu_ctx ctx, const uint32_t* offsets, uint64_t n_bags, uint32_t* occ_bag_out) {
  if (!ctx || !offsets || !occ_bag_out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n_bags == 0) return HPS_GPU_OK;
  k_occ_bags<<<grid_for(n_bags, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(offsets, n_bags, occ_bag_out);
  HPSG_CHECK_LAUNCH("k_occ_bags");
  return HPS_GPU_OK;
}

int hps_gpu_xplan_bucketize(hps_gpu_xplan p, const uint64_t* keys, uint64_t n, const uint32_t* occ_bag,
                            uint32_t n_slots, const uint32_t* slot_table, uint64_t* send_keys, uint32_t* send_tables,
                            uint32_t* perm, uint32_t* counts) {
  if (!p) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n > p->max_keys || n_slots == 0) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = p->ctx->stream;
  if (n == 0) {
    HPSG_CUDA(cudaMemsetAsync(counts, 0, p->n_shards * 4, st));
    return HPS_GPU_OK;
  }
  if (!keys || !slot_table || !send_keys || !send_tables || !perm || !counts) return HPS_GPU_E_INVALID_ARGUMENT;
  if (p->n_shards == 1) {  // one owner: the stable order is the input order (no sort)
    k_pack<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(keys, n, nullptr, occ_bag, n_slots, slot_table, send_keys,
                                                           send_tables, perm);
    k_count_all<<<1, 32, 0, st>>>(counts, static_cast<uint32_t>(n));
    HPSG_CHECK_LAUNCH("bucketize");
    return HPS_GPU_OK;
  }
  k_owner<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(keys, n, p->n_shards, hps::FastMod64(p->n_shards), p->owners,
                                                          p->d_n);
  cudaError_t err;
  const bool in_b = radix_sort_pairs(st, p->owners, nullptr, p->idx_a, p->owners_b, p->idx_b, p->d_n, n, p->bits,
                                     p->sort_ws, &err);
  if (err != cudaSuccess) return cuda_status(err, "bucketize sort");
  k_pack<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(keys, n, in_b ? p->idx_b : p->idx_a, occ_bag, n_slots,
                                                         slot_table, send_keys, send_tables, perm);
  k_counts<<<1, 256, 0, st>>>(p->sort_ws, p->n_shards, counts);  // pass-0 histogram = per-owner counts
  HPSG_CHECK_LAUNCH("bucketize");
  return HPS_GPU_OK;
}

int hps_gpu_pool_rows(hps_gpu_ctx ctx, const float* rows, const uint32_t* perm, const uint32_t* offsets,
                      uint64_t n_bags, uint32_t dim, int combiner, float* out) {
  if (!ctx || dim == 0 || dim % 4) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n_bags == 0) return HPS_GPU_OK;
  if (!rows || !perm || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  const int lpr = lpr_of(dim);
  const int grid = grid_for(n_bags * lpr, 256, kNumSMs * 32);
  HPSG_LPR_LAUNCH(k_pool_rows, lpr, grid, rows, perm, offsets, n_bags, dim, combiner == HPS_COMBINER_MEAN, out);
  HPSG_CHECK_LAUNCH("k_pool_rows");
  return HPS_GPU_OK;
}

int hps_gpu_scatter_grads(hps_gpu_ctx ctx, const float* d_out, const uint32_t* perm, const uint32_t* offsets,
                          uint64_t n_bags, uint32_t dim, int combiner, float* grads_out) {
  if (!ctx || dim == 0 || dim % 4) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n_bags == 0) return HPS_GPU_OK;
  if (!d_out || !perm || !grads_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  const int lpr = lpr_of(dim);
  const int grid = grid_for(n_bags * lpr, 256, kNumSMs * 32);
  HPSG_LPR_LAUNCH(k_scatter_grads, lpr, grid, d_out, perm, offsets, n_bags, dim, combiner == HPS_COMBINER_MEAN,
                  grads_out);
  HPSG_CHECK_LAUNCH("k_scatter_grads");
  return HPS_GPU_OK;
}

int hps_gpu_regroup_bags(hps_gpu_ctx ctx, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         uint32_t n_slots, const uint32_t* sel, uint32_t n_sel, uint32_t* lens_ws,
                         uint64_t* out_keys, uint32_t* out_offsets, uint64_t* scan_ws) {
  if (!ctx || !sel || !lens_ws || !out_keys || !out_offsets || !scan_ws) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  const uint64_t n = uint64_t(n_samples) * n_sel;
  const uint64_t tiles = scan_tiles(n);
  HPSG_CUDA(cudaMemsetAsync(scan_ws, 0, (tiles + 1) * 8, st));
  if (n == 0) {
    HPSG_CUDA(cudaMemsetAsync(out_offsets, 0, 4, st));
    return HPS_GPU_OK;
  }
  k_sel_lengths<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(offsets, n_samples, n_slots, sel, n_sel, lens_ws);
  OffsetsOp op{lens_ws, out_offsets, n};
  k_scan<OffsetsOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, scan_ws,
                                                                         reinterpret_cast<uint32_t*>(scan_ws + tiles));
  k_sel_keys<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(keys, offsets, n_samples, n_slots, sel, n_sel, out_offsets,
                                                             out_keys);
  HPSG_CHECK_LAUNCH("regroup_bags");
  return HPS_GPU_OK;
}

int hps_gpu_lengths_to_offsets(hps_gpu_ctx ctx, const uint32_t* lens, uint64_t n, uint32_t* offsets_out,
                               uint64_t* scan_ws) {
  if (!ctx || !offsets_out || !scan_ws || (n && !lens)) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  const uint64_t tiles = scan_tiles(n);
  if (n == 0) {
    HPSG_CUDA(cudaMemsetAsync(offsets_out, 0, 4, st));
    return HPS_GPU_OK;
  }
  HPSG_CUDA(cudaMemsetAsync(scan_ws, 0, (tiles + 1) * sizeof(uint64_t), st));
  OffsetsOp op{lens, offsets_out, n};
  k_scan<OffsetsOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(
      op, scan_ws, reinterpret_cast<uint32_t*>(scan_ws + tiles));
  HPSG_CHECK_LAUNCH("lengths_to_offsets");
  return HPS_GPU_OK;
}

int hps_gpu_place_pooled(hps_gpu_ctx ctx, const float* src, const uint32_t* sel, uint32_t n_sel, uint32_t n_samples,
                         uint32_t n_slots, uint32_t dim, int direction, float* dst) {
  if (!ctx || !src || !sel || !dst || dim == 0 || dim % 4) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint64_t n = uint64_t(n_samples) * n_sel;
  if (n == 0) return HPS_GPU_OK;
  cudaStream_t st = ctx->stream;
  const int lpr = lpr_of(dim);
  const int grid = grid_for(n * lpr, 256, kNumSMs * 32);
  HPSG_LPR_LAUNCH(k_place, lpr, grid, src, sel, n_sel, n_samples, n_slots, dim, direction, dst);
  HPSG_CHECK_LAUNCH("k_place");
  return HPS_GPU_OK;
}

int hps_gpu_cold_grads(hps_gpu_ctx ctx, const float* d_out, const uint32_t* bags, const uint32_t* perm,
                       const uint32_t* offsets, uint64_t n, uint32_t dim, int combiner, float* grads_out) {
  if (!ctx || dim == 0 || dim % 4) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n == 0) return HPS_GPU_OK;
  if (!d_out || !bags || !perm || !grads_out) return HPS_GPU_E_INVALID_ARGUMENT;
  const int lpr = lpr_of(dim);
  const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
  cudaStream_t st = ctx->stream;
  const int mean = combiner == HPS_COMBINER_MEAN;
  HPSG_LPR_LAUNCH(k_cold_grads, lpr, grid, d_out, bags, perm, offsets, n, dim, mean, grads_out);
  HPSG_CHECK_LAUNCH("k_cold_grads");
  return HPS_GPU_OK;
}

int hps_gpu_sum_partials(hps_gpu_ctx ctx, const float* parts, const uint32_t* touched, uint32_t n_parts, uint64_t rows,
                         uint32_t dim, float* out, uint32_t* touched_out) {
  if (!ctx || dim == 0) return HPS_GPU_E_INVALID_ARGUMENT;
  if (rows == 0) return HPS_GPU_OK;
  if (!parts || !touched || !out || !touched_out || n_parts == 0) return HPS_GPU_E_INVALID_ARGUMENT;
  k_sum_partials<<<grid_for(rows * dim, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(parts, touched, n_parts, rows, dim,
                                                                                  out, touched_out);
  HPSG_CHECK_LAUNCH("k_sum_partials");
  return HPS_GPU_OK;
}

}  // extern "C"
