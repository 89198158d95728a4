// backward.cu — K4 dedup + blocked segmented reduction and K5 fused sparse optimizers.
//
// Semantics (oracle/oracle.cpp reduce_and_update): every key
// occurrence receives d_out[bag] (or d_out[bag]/len for mean); occurrences of one key
// are taken in canonical (occurrence) order, summed in chunks of 32 from the first
// element, the chunk partials summed in order; then SGD / AdaGrad / Adam update the row.
//
// Pipeline (no global sort on the hot path):
//   forward (table.cu) : every found occurrence is registered in an L2-resident dedup
//                        table keyed by row (CAS claim / atomicAdd), which returns its
//                        ARRIVAL rank among the key's occurrences
//   K1 k_scan<DedupScanOp>: compacts the dedup table into unique segments
//                        (row, len, offset) with one packed (unique, occurrence) prefix
//                        scan, resets the table, lists segments longer than 32
//   K2 k_dedup_scatter : occurrence i -> occ_list[offset(u) + arrival rank]
//   K3 k_reduce_short  : one warp per segment of <= 32 occurrences: warp bitonic sort
//                        of the occurrence ids (restores canonical order; only for >= 3),
//                        ordered sum of d_out rows (8 rows in flight), fused optimizer
//   K4 k_long_sort     : one CTA per long segment: stable smem radix sort (<= 4096 ids)
//                        or an occurrence bitmap walk (longer), ids written back in order
//   K5 k_long_chunks   : one warp per 32-occurrence chunk of a long segment -> partial
//   K6 k_long_combine  : one CTA per long segment: partials summed in order (smem
//                        staged), fused optimizer
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "primitives.cuh"
#include "table_internal.cuh"

using namespace hpsg;

namespace {

// ---- K1 --------------------------------------------------------------------------
struct DedupScanOp {
  uint64_t* scr;
  uint64_t cap;
  uint32_t* slot_u;
  uint32_t* seg_row;
  uint32_t* seg_len;
  uint32_t* seg_off;
  uint32_t* long_seg;
  uint32_t* long_base;
  unsigned long long* long_packed;  // (n_long << 32) | total long chunks
  uint64_t* counts;
  __device__ uint64_t size() const { return cap; }
  __device__ uint64_t count(uint64_t s) const {
    const uint64_t v = scr[s];
    return static_cast<uint32_t>(v) == 0xffffffffu ? 0ull : ((1ull << 32) | (v >> 32));
  }
  __device__ void emit(uint64_t s, uint64_t excl, uint64_t c) const {
    if (!c) return;
    const uint64_t v = scr[s];
    const uint32_t u = static_cast<uint32_t>(excl >> 32), off = static_cast<uint32_t>(excl);
    const uint32_t len = static_cast<uint32_t>(v >> 32);
    seg_row[u] = static_cast<uint32_t>(v);
    seg_len[u] = len;
    seg_off[u] = off;
    slot_u[s] = u;
    if (len > kChunk) {
      const uint32_t m = (len + kChunk - 1) / kChunk;
      const unsigned long long p = atomicAdd(long_packed, (1ull << 32) | m);
      long_seg[p >> 32] = u;
      long_base[p >> 32] = static_cast<uint32_t>(p);
    }
    scr[s] = kScrEmpty;  // the table is empty again for the next step
  }
  __device__ void total(uint64_t t) const {
    counts[1] = t >> 32;
    counts[2] = static_cast<uint32_t>(t);
  }
};

// ---- K2 --------------------------------------------------------------------------
__global__ void k_dedup_scatter(const uint64_t* counts, const uint32_t* __restrict__ occ_scr,
                                const uint32_t* __restrict__ occ_rank, const uint32_t* __restrict__ slot_u,
                                const uint32_t* __restrict__ seg_off, uint32_t* __restrict__ occ_list) {
  const uint64_t n = counts[0];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = occ_scr[i];
    if (s == kNoScr) continue;
    occ_list[seg_off[slot_u[s]] + occ_rank[i]] = static_cast<uint32_t>(i);
  }
}

// ---- shared reduction helpers ------------------------------------------------------
struct BwdArgs {
  const uint64_t* counts;
  const uint32_t* seg_row;
  const uint32_t* seg_len;
  const uint32_t* seg_off;
  uint32_t* occ_list;
  const uint32_t* occ_bag;  // nullptr: the bag of occurrence i is i (one key per bag)
  const uint32_t* bag_len;  // mean combiner: bag lengths (nullptr: sum)
  const float* dout;
  uint32_t dim;
  const uint32_t* long_seg;
  const uint32_t* long_base;
  uint32_t* task_long;
  const unsigned long long* long_packed;
  unsigned long long* long_ticket;
  float* partial;
  uint32_t combine_batch;  // partials staged in smem per round of K6
  uint32_t* bitmap;
  uint64_t bitmap_words;
  float* W;
  float* S0;
  float* S1;
  int optimizer;
  hps_opt_params opt;
};

__device__ __forceinline__ uint32_t warp_bitonic_sort(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t p = __shfl_xor_sync(0xffffffffu, v, j);
      const bool asc = (lane & k) == 0, low = (lane & j) == 0;
      v = (asc == low) ? min(v, p) : max(v, p);
    }
  }
  return v;
}

// Ordered sum over n <= 32 occurrences whose bags are spread one per lane (lane q holds
// occurrence q): acc = g_0 + g_1 + ... in exactly that order, 8 rows in flight.
template <int VPL>
__device__ __forceinline__ void ordered_sum(const BwdArgs& a, uint32_t bag, float fl, uint32_t n, float4 (&acc)[VPL]) {
  constexpr int RB = VPL >= 8 ? 1 : 8 / VPL;  // rows in flight per lane (register budget)
  const uint32_t lane = lane_id(), nvec = a.dim / 4;
  for (uint32_t q0 = 0; q0 < n; q0 += RB) {
    float4 x[RB][VPL];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const uint32_t q = q0 + j;
      const uint32_t b = __shfl_sync(0xffffffffu, bag, q & 31);
      const float f = __shfl_sync(0xffffffffu, fl, q & 31);
      const float4* d = reinterpret_cast<const float4*>(a.dout + uint64_t(b) * a.dim);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const uint32_t v = lane + 32 * k;
        float4 t = (q < n && v < nvec) ? __ldg(d + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.bag_len) t = f4_div(t, f);
        x[j][k] = t;
      }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      if (q0 + j < n) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) acc[k] = (q0 + j == 0) ? x[j][k] : f4_add(acc[k], x[j][k]);
      }
    }
  }
}

// Fused optimizer on one row (operation order identical to the oracle).
template <int VPL>
__device__ __forceinline__ void update_row(const BwdArgs& a, uint32_t row, const float4 (&g)[VPL]) {
  const uint32_t lane = lane_id(), nvec = a.dim / 4;
  const uint64_t base = uint64_t(row) * a.dim;
  float4* w = reinterpret_cast<float4*>(a.W + base);
  float4* s0 = reinterpret_cast<float4*>(a.S0 ? a.S0 + base : nullptr);
  float4* s1 = reinterpret_cast<float4*>(a.S1 ? a.S1 + base : nullptr);
  const float lr = a.opt.lr, eps = a.opt.eps;
  float4 wv[VPL], sv[VPL], qv[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {  // issue every load of the row before any math
    const uint32_t v = lane + 32 * k;
    if (v < nvec) {
      wv[k] = w[v];
      if (a.optimizer >= HPS_OPT_ADAGRAD) sv[k] = s0[v];
      if (a.optimizer == HPS_OPT_ADAM) qv[k] = s1[v];
    }
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = lane + 32 * k;
    if (v >= nvec) continue;
    float* wf = reinterpret_cast<float*>(&wv[k]);
    float* sf = reinterpret_cast<float*>(&sv[k]);
    float* qf = reinterpret_cast<float*>(&qv[k]);
    const float* gf = reinterpret_cast<const float*>(&g[k]);
    if (a.optimizer == HPS_OPT_SGD) {
#pragma unroll
      for (int c = 0; c < 4; ++c) wf[c] = __fsub_rn(wf[c], __fmul_rn(lr, gf[c]));
    } else if (a.optimizer == HPS_OPT_ADAGRAD) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(sf[c], __fmul_rn(gf[c], gf[c]));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(lr, gf[c]), __fadd_rn(__fsqrt_rn(sf[c]), eps)));
      }
      s0[v] = sv[k];
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(__fmul_rn(a.opt.beta1, sf[c]), __fmul_rn(a.opt.one_minus_beta1, gf[c]));
        qf[c] = __fadd_rn(__fmul_rn(a.opt.beta2, qf[c]), __fmul_rn(a.opt.one_minus_beta2, __fmul_rn(gf[c], gf[c])));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(a.opt.lr_t, sf[c]), __fadd_rn(__fsqrt_rn(qf[c]), eps)));
      }
      s0[v] = sv[k];
      s1[v] = qv[k];
    }
    w[v] = wv[k];
  }
}

// Load the bag (and mean divisor) of sorted occurrence id `id` (0xffffffff = none).
__device__ __forceinline__ void bag_of(const BwdArgs& a, uint32_t id, uint32_t* bag, float* fl) {
  *bag = 0;
  *fl = 1.0f;
  if (id == 0xffffffffu) return;
  *bag = a.occ_bag ? a.occ_bag[id] : id;
  if (a.bag_len) *fl = static_cast<float>(a.bag_len[*bag]);
}

// ---- K3: segments of <= 32 occurrences ---------------------------------------------
template <int VPL>
__global__ void __launch_bounds__(256) k_reduce_short(BwdArgs a) {
  const uint32_t lane = lane_id();
  const uint64_t U = a.counts[1];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = warp; u < U; u += n_warps) {
    const uint32_t len = a.seg_len[u];
    if (len > kChunk) continue;
    const uint32_t off = a.seg_off[u], row = a.seg_row[u];
    uint32_t id = lane < len ? a.occ_list[off + lane] : 0xffffffffu;
    if (len >= 3) id = warp_bitonic_sort(id);  // arrival order -> canonical order
    uint32_t bag;
    float fl;
    bag_of(a, id, &bag, &fl);
    float4 acc[VPL];
    ordered_sum<VPL>(a, bag, fl, len, acc);
    update_row<VPL>(a, row, acc);
  }
}

// ---- K4: canonical order for long segments ----------------------------------------
// Stable ascending LSD radix sort (8-bit digits) of n <= kSortSmemMax keys in smem,
// blockDim == 256. Returns the buffer holding the result.
__device__ uint32_t* block_sort_ids(uint32_t* keys, uint32_t* tmp, uint32_t n, int bits, uint32_t* s_cnt,
                                    uint32_t* s_hist, uint32_t* s_scr) {
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31, lt = lanemask_lt();
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    s_hist[tid] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += 256) atomicAdd(&s_hist[(keys[i] >> shift) & 255u], 1u);
    __syncthreads();
    uint32_t total;
    uint32_t running = block_excl_scan<256>(s_hist[tid], s_scr, &total);  // thread d: start of digit d
    for (uint32_t r0 = 0; r0 < n; r0 += 256) {
      const uint32_t i = r0 + tid;
      const bool ok = i < n;
      const uint32_t k = ok ? keys[i] : 0u;
      const uint32_t d = ok ? ((k >> shift) & 255u) : 256u + lane;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s_cnt[ww * 256 + tid] = 0;
      __syncthreads();
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & lt);
      if (ok && (__ffs(peers) - 1) == static_cast<int>(lane)) s_cnt[w * 256 + d] = __popc(peers);
      __syncthreads();
      uint32_t acc = running;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) {
        const uint32_t c = s_cnt[ww * 256 + tid];
        s_cnt[ww * 256 + tid] = acc;
        acc += c;
      }
      running = acc;
      __syncthreads();
      if (ok) tmp[s_cnt[w * 256 + d] + rank] = k;
      __syncthreads();
    }
    uint32_t* t = keys;
    keys = tmp;
    tmp = t;
  }
  return keys;
}

__global__ void __launch_bounds__(256) k_long_sort(BwdArgs a, int id_bits) {
  __shared__ uint32_t s_keys[kSortSmemMax];
  __shared__ uint32_t s_tmp[kSortSmemMax];
  __shared__ uint32_t s_cnt[8 * 256];
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_scr[40];
  __shared__ uint32_t s_j;
  const uint32_t tid = threadIdx.x;
  const uint32_t n_long = static_cast<uint32_t>(*a.long_packed >> 32);
  uint32_t* bm = a.bitmap + uint64_t(blockIdx.x) * a.bitmap_words;
  const uint64_t n_occ = a.counts[0];
  while (true) {
    if (tid == 0) s_j = static_cast<uint32_t>(atomicAdd(a.long_ticket, 1ull));
    __syncthreads();
    const uint32_t j = s_j;
    __syncthreads();
    if (j >= n_long) break;
    const uint32_t u = a.long_seg[j];
    const uint32_t len = a.seg_len[u], off = a.seg_off[u];
    uint32_t* seg = a.occ_list + off;
    if (len <= kSortSmemMax) {
      for (uint32_t i = tid; i < len; i += 256) s_keys[i] = seg[i];
      __syncthreads();
      const uint32_t* sorted = block_sort_ids(s_keys, s_tmp, len, id_bits, s_cnt, s_hist, s_scr);
      for (uint32_t i = tid; i < len; i += 256) seg[i] = sorted[i];
    } else {
      // Dense segment: mark its occurrences in a bitmap over [0, n_occ), then walk the
      // bitmap in order (block-wide popcount prefix) — an O(n_occ/32) ordered compaction.
      for (uint32_t i = tid; i < len; i += 256) {
        const uint32_t id = seg[i];
        atomicOr(&bm[id >> 5], 1u << (id & 31));
      }
      __syncthreads();
      const uint64_t words = (n_occ + 31) / 32;
      uint32_t written = 0;
      for (uint64_t w0 = 0; w0 < words; w0 += 256) {
        const uint64_t wi = w0 + tid;
        uint32_t word = wi < words ? __ldcg(bm + wi) : 0u;  // L2: the bits were set by atomics
        uint32_t tot;
        uint32_t pos = written + block_excl_scan<256>(static_cast<uint32_t>(__popc(word)), s_scr, &tot);
        if (word) bm[wi] = 0;  // leave the bitmap clean for the next segment
        while (word) {
          const int b = __ffs(word) - 1;
          word &= word - 1;
          seg[pos++] = static_cast<uint32_t>(wi * 32 + b);
        }
        written += tot;
      }
    }
    const uint32_t m = (len + kChunk - 1) / kChunk, base = a.long_base[j];
    for (uint32_t c = tid; c < m; c += 256) a.task_long[base + c] = j;
    __syncthreads();
  }
}

// ---- K5: chunk partials of long segments --------------------------------------------
template <int VPL>
__global__ void __launch_bounds__(256) k_long_chunks(BwdArgs a) {
  const uint32_t lane = lane_id(), nvec = a.dim / 4;
  const uint64_t T = static_cast<uint32_t>(*a.long_packed);
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t t = warp; t < T; t += n_warps) {
    const uint32_t j = a.task_long[t];
    const uint32_t u = a.long_seg[j];
    const uint32_t c = static_cast<uint32_t>(t) - a.long_base[j];
    const uint32_t off = a.seg_off[u], len = a.seg_len[u];
    const uint32_t lo = c * kChunk, n = min(kChunk, len - lo);
    const uint32_t id = lane < n ? a.occ_list[off + lo + lane] : 0xffffffffu;
    uint32_t bag;
    float fl;
    bag_of(a, id, &bag, &fl);
    float4 acc[VPL];
    ordered_sum<VPL>(a, bag, fl, n, acc);
    float4* p = reinterpret_cast<float4*>(a.partial + t * a.dim);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t v = lane + 32 * k;
      if (v < nvec) __stcg(p + v, acc[k]);
    }
  }
}

// ---- K6: ordered combine of the partials + optimizer --------------------------------
template <int VPL>
__global__ void __launch_bounds__(256) k_long_combine(BwdArgs a) {
  extern __shared__ float4 s_part[];  // combine_batch partials of dim floats
  const uint32_t kCombineBatch = a.combine_batch;
  const uint32_t tid = threadIdx.x, lane = tid & 31, nvec = a.dim / 4;
  const uint32_t n_long = static_cast<uint32_t>(*a.long_packed >> 32);
  for (uint32_t j = blockIdx.x; j < n_long; j += gridDim.x) {
    const uint32_t u = a.long_seg[j];
    const uint32_t m = (a.seg_len[u] + kChunk - 1) / kChunk, base = a.long_base[j];
    float4 acc[VPL];
    for (uint32_t b0 = 0; b0 < m; b0 += kCombineBatch) {
      const uint32_t nb = min(kCombineBatch, m - b0);
      const float4* src = reinterpret_cast<const float4*>(a.partial + uint64_t(base + b0) * a.dim);
      for (uint32_t e = tid; e < nb * nvec; e += 256) s_part[e] = __ldcg(src + e);
      __syncthreads();
      if (tid < 32) {
        for (uint32_t q = 0; q < nb; ++q) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const uint32_t v = lane + 32 * k;
            if (v < nvec) {
              const float4 x = s_part[q * nvec + v];
              acc[k] = (b0 + q == 0) ? x : f4_add(acc[k], x);
            }
          }
        }
      }
      __syncthreads();
    }
    if (tid < 32) update_row<VPL>(a, a.seg_row[u], acc);
  }
}

__global__ void k_copy_u64(const uint64_t* src, uint64_t* dst) { *dst = *src; }

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

#define HPSG_DISPATCH_VPL(KERNEL, GRID, SMEM, ...)                                \
  do {                                                                            \
    if (nvec > 128) KERNEL<8><<<GRID, 256, SMEM, st>>>(__VA_ARGS__);              \
    else if (nvec > 64) KERNEL<4><<<GRID, 256, SMEM, st>>>(__VA_ARGS__);          \
    else if (nvec > 32) KERNEL<2><<<GRID, 256, SMEM, st>>>(__VA_ARGS__);          \
    else KERNEL<1><<<GRID, 256, SMEM, st>>>(__VA_ARGS__);                         \
  } while (0)

}  // namespace

extern "C" {

int hps_gpu_backward_update(hps_gpu_table t, const float* d_out, const hps_opt_params* opt) {
  if (!t || !opt) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!t->have_train) {
    set_last_error("backward_update: no preceding lookup_pooled with HPS_LOOKUP_TRAIN");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!d_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const uint64_t nk = t->last_n_keys_host;
  const uint64_t cap = 1ull << t->scr_bits;
  const uint64_t tiles = scan_tiles(cap);
  uint64_t* status = t->ws_scan;
  uint32_t* ticket = reinterpret_cast<uint32_t*>(t->ws_scan + tiles);
  auto* long_packed = reinterpret_cast<unsigned long long*>(t->ws_scan + tiles + 1);
  auto* long_ticket = reinterpret_cast<unsigned long long*>(t->ws_scan + tiles + 2);
  HPSG_CUDA(cudaMemsetAsync(t->ws_scan, 0, t->scan_words * sizeof(uint64_t), st));

  DedupScanOp op{t->ws_scr,      cap,          t->ws_slot_u,  t->ws_seg_row, t->ws_seg_len,
                 t->ws_seg_off,  t->ws_long_seg, t->ws_long_base, long_packed, t->ws_counts};
  k_scan<DedupScanOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, status, ticket);
  k_dedup_scatter<<<grid_for(nk, 256, kNumSMs * 8), 256, 0, st>>>(t->ws_counts, t->ws_occ_scr, t->ws_occ_rank,
                                                                 t->ws_slot_u, t->ws_seg_off, t->ws_occ_list);
  BwdArgs a{};
  a.counts = t->ws_counts;
  a.seg_row = t->ws_seg_row;
  a.seg_len = t->ws_seg_len;
  a.seg_off = t->ws_seg_off;
  a.occ_list = t->ws_occ_list;
  a.occ_bag = t->last_multi ? t->ws_occ_bag : nullptr;
  a.bag_len = (t->last_multi && t->last_combiner == HPS_COMBINER_MEAN) ? t->ws_bag_len : nullptr;
  a.dout = d_out;
  a.dim = t->dim;
  a.long_seg = t->ws_long_seg;
  a.long_base = t->ws_long_base;
  a.task_long = t->ws_task_long;
  a.long_packed = long_packed;
  a.long_ticket = long_ticket;
  a.partial = t->ws_partial;
  a.bitmap = t->ws_bitmap;
  a.bitmap_words = t->bitmap_words;
  a.W = t->d_w;
  a.S0 = t->d_s0;
  a.S1 = t->d_s1;
  a.optimizer = t->optimizer;
  a.opt = *opt;
  const uint32_t nvec = t->dim / 4;
  const int warps_grid = grid_for(nk * 32, 256, kNumSMs * 16);
  HPSG_DISPATCH_VPL(k_reduce_short, warps_grid, 0, a);
  k_long_sort<<<t->long_ctas, 256, 0, st>>>(a, std::max(1, bits_for(nk)));
  const int chunk_grid = grid_for(std::min<uint64_t>(t->max_chunks, nk / kChunk + 2) * 32, 256, kNumSMs * 16);
  HPSG_DISPATCH_VPL(k_long_chunks, chunk_grid, 0, a);
  a.combine_batch = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(32, (48 * 1024) / (t->dim * 4))));
  const size_t smem = a.combine_batch * size_t(t->dim) * sizeof(float);
  HPSG_DISPATCH_VPL(k_long_combine, t->long_ctas, smem, a);
  HPSG_CHECK_LAUNCH("backward");
  t->scr_dirty = false;
  return HPS_GPU_OK;
}

int hps_gpu_table_last_unique(hps_gpu_table t, uint64_t* count_out, uint32_t* unique_rows_out) {
  if (!t || !count_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  k_copy_u64<<<1, 1, 0, st>>>(t->ws_counts + 1, count_out);
  HPSG_CHECK_LAUNCH("k_copy_u64");
  if (!unique_rows_out) return HPS_GPU_OK;
  // Ascending row order (reporting only, syncs; not on the training hot path).
  uint64_t n = 0;
  HPSG_CUDA(cudaMemcpyAsync(&n, t->ws_counts + 1, 8, cudaMemcpyDeviceToHost, st));
  HPSG_CUDA(cudaStreamSynchronize(st));
  if (n == 0) return HPS_GPU_OK;
  const int bits = std::max(1, bits_for(t->total_rows));
  const size_t words = sort_ws_words(n, (bits + 7) / 8);
  uint32_t *ka = nullptr, *va = nullptr, *kb = nullptr, *vb = nullptr, *ws = nullptr;
  HPSG_CUDA(cudaMallocAsync(&ka, n * 4, st));
  HPSG_CUDA(cudaMallocAsync(&va, n * 4, st));
  HPSG_CUDA(cudaMallocAsync(&kb, n * 4, st));
  HPSG_CUDA(cudaMallocAsync(&vb, n * 4, st));
  HPSG_CUDA(cudaMallocAsync(&ws, words * 4, st));
  HPSG_CUDA(cudaMemcpyAsync(ka, t->ws_seg_row, n * 4, cudaMemcpyDeviceToDevice, st));
  cudaError_t err;
  const bool in_b = radix_sort_pairs(st, ka, nullptr, va, kb, vb, t->ws_counts + 1, n, bits, ws, &err);
  if (err != cudaSuccess) return cuda_status(err, "last_unique sort");
  HPSG_CUDA(cudaMemcpyAsync(unique_rows_out, in_b ? kb : ka, n * 4, cudaMemcpyDeviceToDevice, st));
  for (uint32_t* p : {ka, va, kb, vb, ws}) HPSG_CUDA(cudaFreeAsync(p, st));
  return HPS_GPU_OK;
}

}  // extern "C"
