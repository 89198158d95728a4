// backward.cu — K4 dedup + blocked segmented reduction and K5 fused sparse optimizers.
//
// Semantics (oracle/oracle.cpp reduce_and_update): every key
// occurrence receives d_out[bag] (or d_out[bag]/len for mean); occurrences of one key
// are taken in canonical (occurrence) order, summed in chunks of 32 from the first
// element, the chunk partials summed in order; then SGD / AdaGrad / Adam update the row.
//
// Pipeline (sizes device-resident: one memset node + 6 + passes kernels, graph-capturable):
//   k_radix_hist/k_radix_pass : stable LSD sort of (row, bag) by row — the dedup, and the
//                               stability keeps each key's occurrences in canonical order
//   k_scan<SegOp>    : unique-row segments [start, end) + occurrence -> segment
//   k_list_long      : segments longer than kItemW (or absent keys) are cut into
//                      chunk-aligned pieces of kItemW occurrences; their occurrences are
//                      flagged so the short items skip them
//   k_stream         : persistent blocks take work items — kItemW-wide windows of the
//                      sorted list (short segments) or long pieces — stage d_out rows in
//                      shared memory with coalesced 128-bit loads, run the blocked ordered
//                      sums column-parallel from smem, and apply the optimizer to every
//                      finished segment in batched warp passes (long pieces emit chunk
//                      partials instead). Work is balanced by OCCURRENCES, so hot keys
//                      cannot serialise a warp.
//   k_long_combine   : one CTA per long segment: chunk partials in order + optimizer
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "primitives.cuh"
#include "table_internal.cuh"

using namespace hpsg;

namespace {

constexpr uint32_t kSkip = 0x80000000u;  // occ_seg flag: owned by a long piece / absent key
constexpr uint32_t kSegMask = 0x7fffffffu;
constexpr int kStreamBlock = 256;
constexpr uint32_t kMaxTile = 128;

struct BwdArgs {
  const uint64_t* counts;  // [0]=N occurrences [1]=U segments
  const uint32_t* rows;    // sorted global rows
  const uint32_t* bags;    // bag of each sorted occurrence
  uint32_t* seg_start;
  uint32_t* seg_end;
  uint32_t* occ_seg;
  uint32_t row_absent;
  const uint32_t* bag_len;  // mean combiner: bag lengths (nullptr: sum)
  const float* dout;
  uint32_t dim;
  uint32_t* long_seg;
  uint32_t* long_base;
  uint32_t* pieces;
  unsigned long long* long_packed;  // (n_long << 32) | total long chunks
  unsigned long long* piece_count;
  unsigned long long* item_ticket;
  uint64_t n_short_items;
  uint32_t tile;  // occurrences staged per smem tile
  float* partial;
  uint32_t combine_batch;
  float* W;
  float* S0;
  float* S1;
  int optimizer;
  hps_opt_params opt;
};

// ---- segments of the sorted list ----------------------------------------------------
struct SegOp {
  const uint32_t* rows;
  uint32_t* seg_start;
  uint32_t* seg_end;
  uint32_t* occ_seg;
  uint64_t* counts;
  __device__ uint64_t size() const { return counts[0]; }
  __device__ uint32_t count(uint64_t i) const { return (i == 0 || rows[i] != rows[i - 1]) ? 1u : 0u; }
  __device__ void emit(uint64_t i, uint64_t excl, uint64_t c) const {
    const uint32_t u = static_cast<uint32_t>(excl + c - 1);
    if (c) seg_start[u] = static_cast<uint32_t>(i);
    occ_seg[i] = u;
    if (i + 1 == counts[0] || rows[i + 1] != rows[i]) seg_end[u] = static_cast<uint32_t>(i + 1);
  }
  __device__ void total(uint64_t u) const { counts[1] = u; }
};

// ---- long segments -> pieces ----------------------------------------------------------
// A warp inspects 32 segments (one per lane); long or absent ones are handed out as
// pieces and their occurrences flagged by the whole warp (coalesced).
__global__ void __launch_bounds__(256) k_list_long(BwdArgs a) {
  const uint32_t lane = lane_id();
  const uint64_t U = a.counts[1];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u0 = warp * 32; u0 < U; u0 += n_warps * 32) {
    const uint64_t u = u0 + lane;
    uint32_t s = 0, e = 0;
    bool flag = false;
    if (u < U) {
      s = a.seg_start[u];
      e = a.seg_end[u];
      const bool absent = a.rows[s] == a.row_absent;
      const uint32_t len = e - s;
      flag = absent || len > kItemW;
      if (!absent && len > kItemW) {
        const uint32_t m = (len + kChunk - 1) / kChunk;
        const unsigned long long p = atomicAdd(a.long_packed, (1ull << 32) | m);
        const uint32_t j = static_cast<uint32_t>(p >> 32);
        a.long_seg[j] = static_cast<uint32_t>(u);
        a.long_base[j] = static_cast<uint32_t>(p);
        const uint32_t np = (len + kItemW - 1) / kItemW;
        const uint32_t p0 = static_cast<uint32_t>(atomicAdd(a.piece_count, static_cast<unsigned long long>(np)));
        for (uint32_t k = 0; k < np; ++k) {
          a.pieces[2 * (p0 + k)] = j;
          a.pieces[2 * (p0 + k) + 1] = k;
        }
      }
    }
    uint32_t todo = __ballot_sync(0xffffffffu, flag);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t ss = __shfl_sync(0xffffffffu, s, src), ee = __shfl_sync(0xffffffffu, e, src);
      for (uint32_t o = ss + lane; o < ee; o += 32) a.occ_seg[o] |= kSkip;
    }
  }
}

// ---- row math --------------------------------------------------------------------------
template <int VPL>
struct RowState {
  float4 w[VPL], s[VPL], q[VPL];
};

template <int VPL>
__device__ __forceinline__ void load_row(const BwdArgs& a, uint32_t row, uint32_t gl, uint32_t lpr, RowState<VPL>& r) {
  const uint32_t nvec = a.dim / 4;
  const uint64_t base = uint64_t(row) * a.dim;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = gl + k * lpr;
    if (v < nvec) {
      r.w[k] = reinterpret_cast<const float4*>(a.W + base)[v];
      if (a.optimizer >= HPS_OPT_ADAGRAD) r.s[k] = reinterpret_cast<const float4*>(a.S0 + base)[v];
      if (a.optimizer == HPS_OPT_ADAM) r.q[k] = reinterpret_cast<const float4*>(a.S1 + base)[v];
    }
  }
}

// Fused optimizer (operation order identical to the oracle), then store.
template <int VPL>
__device__ __forceinline__ void update_store(const BwdArgs& a, uint32_t row, uint32_t gl, uint32_t lpr,
                                             RowState<VPL>& r, const float4 (&g)[VPL]) {
  const uint32_t nvec = a.dim / 4;
  const uint64_t base = uint64_t(row) * a.dim;
  const float lr = a.opt.lr, eps = a.opt.eps;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = gl + k * lpr;
    if (v >= nvec) continue;
    float* wf = reinterpret_cast<float*>(&r.w[k]);
    float* sf = reinterpret_cast<float*>(&r.s[k]);
    float* qf = reinterpret_cast<float*>(&r.q[k]);
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
      reinterpret_cast<float4*>(a.S0 + base)[v] = r.s[k];
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(__fmul_rn(a.opt.beta1, sf[c]), __fmul_rn(a.opt.one_minus_beta1, gf[c]));
        qf[c] = __fadd_rn(__fmul_rn(a.opt.beta2, qf[c]), __fmul_rn(a.opt.one_minus_beta2, __fmul_rn(gf[c], gf[c])));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(a.opt.lr_t, sf[c]), __fadd_rn(__fsqrt_rn(qf[c]), eps)));
      }
      reinterpret_cast<float4*>(a.S0 + base)[v] = r.s[k];
      reinterpret_cast<float4*>(a.S1 + base)[v] = r.q[k];
    }
    reinterpret_cast<float4*>(a.W + base)[v] = r.w[k];
  }
}

// ---- the streaming reduction -----------------------------------------------------------
// CPT: columns (floats) per thread in the ordered-sum phase (dim <= 256 * CPT).
// VPL: float4 per lane in the optimizer phase (dim <= 128 * VPL).
template <int CPT, int VPL>
__global__ void __launch_bounds__(kStreamBlock) k_stream(BwdArgs a) {
  extern __shared__ float s_tile[];  // [tile][dim] gradient rows, then finished-segment totals
  __shared__ uint32_t s_row[kMaxTile], s_pos[kMaxTile], s_flag[kMaxTile], s_bag[kMaxTile];
  __shared__ float s_len[kMaxTile];
  __shared__ uint32_t s_done[kMaxTile];
  __shared__ uint32_t s_ndone;
  __shared__ uint32_t s_mode, s_A, s_B, s_seg_s, s_seg_e, s_cbase;  // item descriptor
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t D = a.dim, nvec = D / 4, T = a.tile;
  const uint64_t N = a.counts[0];
  const uint64_t n_items = a.n_short_items + *a.piece_count;
  constexpr uint32_t kLast = 1u, kValid = 2u;
  while (true) {
    if (tid == 0) {
      const uint64_t item = atomicAdd(a.item_ticket, 1ull);
      uint32_t mode = 0, A = 0, B = 0, ss = 0, se = 0, cb = 0;  // mode 0: nothing, 1: short, 2: long piece, 3: done
      if (item >= n_items) {
        mode = 3;
      } else if (item < a.n_short_items) {
        const uint64_t lo = item * kItemW;
        if (lo < N) {
          const uint64_t hi = std::min<uint64_t>(N, lo + kItemW);
          const uint32_t U = static_cast<uint32_t>(a.counts[1]);
          uint32_t s0 = a.occ_seg[lo] & kSegMask;
          if (a.seg_start[s0] < lo) ++s0;  // that segment belongs to an earlier item
          uint32_t s1;                     // last segment starting before hi
          if (hi >= N) {
            s1 = U - 1;
          } else {
            s1 = a.occ_seg[hi] & kSegMask;
            if (a.seg_start[s1] >= hi) --s1;
          }
          if (s0 < U && s0 <= s1) {
            mode = 1;
            A = a.seg_start[s0];
            B = a.seg_end[s1];
          }
        }
      } else {
        const uint64_t p = item - a.n_short_items;
        const uint32_t j = a.pieces[2 * p], k = a.pieces[2 * p + 1];
        const uint32_t u = a.long_seg[j];
        ss = a.seg_start[u];
        se = a.seg_end[u];
        A = ss + k * kItemW;
        B = min(se, A + kItemW);
        cb = a.long_base[j];
        mode = 2;
      }
      s_mode = mode;
      s_A = A;
      s_B = B;
      s_seg_s = ss;
      s_seg_e = se;
      s_cbase = cb;
    }
    __syncthreads();
    const uint32_t mode = s_mode, A = s_A, B = s_B;
    if (mode == 3) break;
    if (mode == 0) {
      __syncthreads();
      continue;
    }
    float part[CPT], total[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) part[i] = total[i] = 0.f;
    for (uint32_t t0 = A; t0 < B; t0 += T) {
      const uint32_t nt = min(T, B - t0);
      if (tid == 0) s_ndone = 0;
      // phase 1: per-occurrence metadata
      if (tid < nt) {
        const uint32_t o = t0 + tid;
        uint32_t flag = 0, pos = 0;
        const uint32_t bag = a.bags[o];
        s_row[tid] = a.rows[o];
        if (mode == 2) {
          pos = o - s_seg_s;
          flag = kValid | ((o + 1 == s_seg_e) ? kLast : 0u);
        } else {
          const uint32_t sg = a.occ_seg[o];
          if (!(sg & kSkip)) {
            const uint32_t ss = a.seg_start[sg], se = a.seg_end[sg];
            pos = o - ss;
            flag = kValid | ((o + 1 == se) ? kLast : 0u);
          }
        }
        s_bag[tid] = bag;
        s_pos[tid] = pos;
        s_flag[tid] = flag;
        s_len[tid] = (a.bag_len && flag) ? static_cast<float>(a.bag_len[bag]) : 1.0f;
      }
      __syncthreads();
      // phase 2: stage the gradient rows (warp w: rows w, w+8, ...; 128-bit coalesced)
      for (uint32_t q = w; q < nt; q += kStreamBlock / 32) {
        if (!s_flag[q]) continue;
        const float4* src = reinterpret_cast<const float4*>(a.dout + uint64_t(s_bag[q]) * D);
        float4* dst = reinterpret_cast<float4*>(s_tile + q * D);
        const float fl = s_len[q];
        for (uint32_t v = lane; v < nvec; v += 32) {
          float4 x = __ldg(src + v);
          if (a.bag_len) x = f4_div(x, fl);
          dst[v] = x;
        }
      }
      __syncthreads();
      // phase 3: ordered blocked sums, column-parallel
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const uint32_t c = tid + i * kStreamBlock;
        if (c >= D) continue;
        for (uint32_t q = 0; q < nt; ++q) {
          const uint32_t f = s_flag[q];
          if (!f) continue;
          const uint32_t pos = s_pos[q];
          const float g = s_tile[q * D + c];
          part[i] = (pos % kChunk == 0) ? g : __fadd_rn(part[i], g);
          if ((pos % kChunk) == kChunk - 1 || (f & kLast)) {
            if (mode == 2) {
              __stcg(a.partial + uint64_t(s_cbase + pos / kChunk) * D + c, part[i]);
            } else {
              total[i] = (pos < kChunk) ? part[i] : __fadd_rn(total[i], part[i]);
              if (f & kLast) s_tile[q * D + c] = total[i];
            }
          }
        }
      }
      if (mode == 1 && tid < nt && (s_flag[tid] & kLast)) s_done[atomicAdd(&s_ndone, 1u)] = tid;
      __syncthreads();
      // phase 4: optimizer on the segments finished in this tile (4 rows in flight / warp)
      if (mode == 1) {
        const uint32_t nd = s_ndone;
        for (uint32_t d0 = w * 4; d0 < nd; d0 += (kStreamBlock / 32) * 4) {
          RowState<VPL> rs[4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (d0 + r < nd) load_row<VPL>(a, s_row[s_done[d0 + r]], lane, 32, rs[r]);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (d0 + r >= nd) continue;
            const uint32_t q = s_done[d0 + r];
            float4 g[VPL];
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
              const uint32_t v = lane + 32 * k;
              g[k] = v < nvec ? reinterpret_cast<const float4*>(s_tile + q * D)[v] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            update_store<VPL>(a, s_row[q], lane, 32, rs[r], g);
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) k_long_combine(BwdArgs a) {
  extern __shared__ float4 s_part[];  // combine_batch partials of dim floats
  const uint32_t tid = threadIdx.x, lane = tid & 31, nvec = a.dim / 4;
  const uint32_t n_long = static_cast<uint32_t>(*a.long_packed >> 32);
  for (uint32_t j = blockIdx.x; j < n_long; j += gridDim.x) {
    const uint32_t u = a.long_seg[j];
    const uint32_t start = a.seg_start[u];
    const uint32_t m = (a.seg_end[u] - start + kChunk - 1) / kChunk, base = a.long_base[j];
    const uint32_t row = a.rows[start];
    RowState<VPL> rs;
    if (tid < 32) load_row<VPL>(a, row, lane, 32, rs);
    float4 acc[VPL];
    for (uint32_t b0 = 0; b0 < m; b0 += a.combine_batch) {
      const uint32_t nb = min(a.combine_batch, m - b0);
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
    if (tid < 32) update_store<VPL>(a, row, lane, 32, rs, acc);
  }
}

__global__ void k_unique_rows(const uint32_t* rows, const uint32_t* seg_start, const uint64_t* counts,
                              uint32_t row_absent, uint32_t* out, uint64_t* count_out) {
  const uint64_t U = counts[1];
  const bool has_absent = U > 0 && rows[seg_start[U - 1]] == row_absent;
  const uint64_t n = has_absent ? U - 1 : U;
  if (blockIdx.x == 0 && threadIdx.x == 0 && count_out) *count_out = n;
  if (!out) return;
  for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n; u += uint64_t(gridDim.x) * blockDim.x)
    out[u] = rows[seg_start[u]];
}

template <int CPT, int VPL>
int launch_stream(const BwdArgs& a, cudaStream_t st, size_t smem, int grid) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_stream<CPT, VPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
  k_stream<CPT, VPL><<<grid, kStreamBlock, smem, st>>>(a);
  return 0;
}

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
  const int passes = (t->sort_bits + 7) / 8;
  // zeroed region (table_internal.cuh bwd_zero_words)
  uint32_t* z = t->ws_zero;
  const size_t sort_words = bwd_sort_words(nk, passes);
  const uint64_t tiles = scan_tiles(nk);
  uint64_t* scan_status = reinterpret_cast<uint64_t*>(z + sort_words);
  uint32_t* scan_ticket = reinterpret_cast<uint32_t*>(scan_status + tiles);
  auto* long_packed = reinterpret_cast<unsigned long long*>(scan_status + tiles + 1);
  auto* piece_count = reinterpret_cast<unsigned long long*>(scan_status + tiles + 2);
  auto* item_ticket = reinterpret_cast<unsigned long long*>(scan_status + tiles + 3);
  const size_t used = sort_words + 2 * (tiles + 6);
  HPSG_CUDA(cudaMemsetAsync(z, 0, used * sizeof(uint32_t), st));

  // K4a: stable sort of (row, bag) by row. One key per bag: the bag IS the occurrence.
  {
    const uint64_t stiles = sort_tiles(nk);
    uint32_t* hist = z;
    uint32_t* stick = z + 4 * 256;
    uint32_t* status = stick + 4;
    k_radix_hist<<<grid_for(nk, 256, kNumSMs * 2), 256, 0, st>>>(t->ws_rows_a, t->ws_counts, passes, hist);
    const uint32_t* kin = t->ws_rows_a;
    const uint32_t* vin = t->last_multi ? t->ws_occ_bag : nullptr;
    bool in_b = false;
    for (int p = 0; p < passes; ++p) {
      uint32_t* kout = in_b ? t->ws_rows_a : t->ws_rows_b;
      uint32_t* vout = in_b ? t->ws_bags_a : t->ws_bags_b;
      k_radix_pass<<<static_cast<unsigned>(stiles), kSortBlock, 0, st>>>(
          kin, vin, kout, vout, t->ws_counts, 8 * p, hist + 256 * p, status + size_t(p) * stiles * 256, stick + p);
      kin = kout;
      vin = vout;
      in_b = !in_b;
    }
    t->sorted_in_b = in_b;
    HPSG_CHECK_LAUNCH("radix sort");
  }
  const uint32_t* rows = t->sorted_in_b ? t->ws_rows_b : t->ws_rows_a;
  const uint32_t* bags = t->sorted_in_b ? t->ws_bags_b : t->ws_bags_a;
  // K4b: unique-row segments.
  SegOp sop{rows, t->ws_seg_start, t->ws_seg_end, t->ws_occ_seg, t->ws_counts};
  k_scan<SegOp><<<static_cast<unsigned>(std::max<uint64_t>(1, tiles)), kScanBlock, 0, st>>>(sop, scan_status,
                                                                                            scan_ticket);
  BwdArgs a{};
  a.counts = t->ws_counts;
  a.rows = rows;
  a.bags = bags;
  a.seg_start = t->ws_seg_start;
  a.seg_end = t->ws_seg_end;
  a.occ_seg = t->ws_occ_seg;
  a.row_absent = t->row_absent;
  a.bag_len = (t->last_multi && t->last_combiner == HPS_COMBINER_MEAN) ? t->ws_bag_len : nullptr;
  a.dout = d_out;
  a.dim = t->dim;
  a.long_seg = t->ws_long_seg;
  a.long_base = t->ws_long_base;
  a.pieces = t->ws_pieces;
  a.long_packed = long_packed;
  a.piece_count = piece_count;
  a.item_ticket = item_ticket;
  a.n_short_items = (nk + kItemW - 1) / kItemW;
  a.tile = static_cast<uint32_t>(std::max<uint64_t>(16, std::min<uint64_t>(kMaxTile, 8192 / t->dim)));
  a.partial = t->ws_partial;
  a.W = t->d_w;
  a.S0 = t->d_s0;
  a.S1 = t->d_s1;
  a.optimizer = t->optimizer;
  a.opt = *opt;
  a.combine_batch = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(32, (48 * 1024) / (t->dim * 4))));
  k_list_long<<<grid_for((nk + 31) / 32 * 32, 256, kNumSMs * 8), 256, 0, st>>>(a);
  // K4c + K5: streaming reduction fused with the optimizer.
  const size_t tile_smem = size_t(a.tile) * t->dim * sizeof(float);
  const uint64_t max_items = a.n_short_items + t->max_pieces;
  const int sgrid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(max_items, kNumSMs * 4)));
  const uint32_t D = t->dim;
  if (D <= 128) launch_stream<1, 1>(a, st, tile_smem, sgrid);
  else if (D <= 256) launch_stream<1, 2>(a, st, tile_smem, sgrid);
  else if (D <= 512) launch_stream<2, 4>(a, st, tile_smem, sgrid);
  else launch_stream<4, 8>(a, st, tile_smem, sgrid);
  const size_t smem = a.combine_batch * size_t(t->dim) * sizeof(float);
  const int comb_grid = static_cast<int>(std::min<uint64_t>(t->max_long, 2 * kNumSMs));
  const uint32_t nvec = D / 4;
  if (nvec > 128) k_long_combine<8><<<comb_grid, 256, smem, st>>>(a);
  else if (nvec > 64) k_long_combine<4><<<comb_grid, 256, smem, st>>>(a);
  else if (nvec > 32) k_long_combine<2><<<comb_grid, 256, smem, st>>>(a);
  else k_long_combine<1><<<comb_grid, 256, smem, st>>>(a);
  HPSG_CHECK_LAUNCH("backward");
  return HPS_GPU_OK;
}

int hps_gpu_table_last_unique(hps_gpu_table t, uint64_t* count_out, uint32_t* unique_rows_out) {
  if (!t || !count_out) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint32_t* rows = t->sorted_in_b ? t->ws_rows_b : t->ws_rows_a;
  k_unique_rows<<<grid_for(t->last_n_keys_host, 256, kNumSMs * 8), 256, 0, t->ctx->stream>>>(
      rows, t->ws_seg_start, t->ws_counts, t->row_absent, unique_rows_out, count_out);
  HPSG_CHECK_LAUNCH("k_unique_rows");
  return HPS_GPU_OK;
}

}  // extern "C"
