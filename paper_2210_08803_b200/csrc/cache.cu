// cache.cu — HPS GPU embedding cache (K6 query, K7 insert/evict, K8 refresh).
//
// Semantics: SPEC.md:112-190 (set-associative LFU with aging and last-touch tie-break)
// with the resolutions of DESIGN.md §5, restated on the CPU in oracle/oracle.cpp
// (Cache). Placement: set = key_hash(key) mod num_sets (hash.hpp:42-49),
// computed with an exact 128-bit-magic modulo.
//
// Batch-parallel with exact sequential semantics:
//   * a query batch never changes residency, so every hit/miss is decided in parallel
//     against the state before the batch (K6a); found/missing are compacted in input
//     order by a decoupled look-back scan; hits are gathered with 128-bit loads;
//   * the metadata side effects (freq, last_touch, aging) depend on per-set ORDER only,
//     so accesses are stably radix-sorted by set and one warp per touched set replays
//     them 32 at a time in closed form (saturating adds between aging points);
//   * insert/refresh are sequential per set (eviction depends on the previous insert),
//     so the same sort feeds one warp per set that walks its entries in input order,
//     lanes = ways.
// HBM layout (set-major): keys/versions/last_touch [sets x ways] u64,
// freq [sets x ways] u8 (0 = empty way), vectors [sets x ways x dim] fp32 or binary16.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_fp16.h>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "primitives.cuh"

using namespace hpsg;

namespace hpsg {
int cache_query(hps_gpu_cache c, const uint64_t* keys, uint64_t n, const uint64_t* d_n, float* found_vecs,
                uint32_t* found_idx, uint32_t* missing_idx, uint64_t* counts, bool scatter_found = false);
}

struct hps_gpu_cache_s {
  hps_gpu_ctx ctx = nullptr;
  uint64_t capacity = 0, num_sets = 0, aging_period = 0, max_batch = 0;
  uint32_t ways = 0, dim = 0;
  uint32_t dim_io = 0;     // the caller's dim; `dim` = padded_dim(dim_io) is the row stride
  float* ws_io = nullptr;  // dim_io != dim: [max_batch x dim] staging of query / insert rows
  hps::FastMod64 set_mod;
  int set_bits = 0;
  uint64_t *d_keys = nullptr, *d_ver = nullptr, *d_touch = nullptr, *d_set_acc = nullptr;
  uint8_t* d_freq = nullptr;
  void* d_vec = nullptr;  // [capacity x dim] fp32, or binary16 when f16
  bool f16 = false;
  uint64_t* d_state = nullptr;  // [0]=clock [1]=clock snapshot of the running call [2..8]=stats [9]=scratch count
  // workspaces
  uint32_t *ws_set = nullptr, *ws_keys_b = nullptr, *ws_vals_a = nullptr, *ws_vals_b = nullptr;
  uint8_t* ws_hit = nullptr;
  uint32_t* ws_rank = nullptr;
  uint32_t* ws_seg = nullptr;
  uint32_t* ws_sort = nullptr;
  uint64_t* ws_scan = nullptr;
  uint64_t* ws_counts = nullptr;  // [0]=n [1]=U (segments) [2]=found [3]=valid
  size_t sort_words = 0;
  // the last query's set-sorted access list (cache_insert_after_query derives an insert's
  // set grouping from it) and that derivation's buffers
  const uint32_t* q_sets = nullptr;
  const uint32_t* q_idx = nullptr;
  uint32_t *ws_der_set = nullptr, *ws_der_idx = nullptr, *ws_der_pos = nullptr;
  uint32_t* ws_qmiss = nullptr;    // the last query's access -> miss rank (SplitOp)
  uint32_t* ws_setcnt = nullptr;   // counting grouping: per-set counters [num_sets + 1], zero at rest
  uint32_t* ws_ticket = nullptr;   // counting grouping: arrival rank of each access in its set
  bool count_group = false;        // distinct-key queries group by set with counters (no radix sort)
  bool query_distinct = false;     // the next cache_query's keys are distinct (the read-through sets it)
  // pre-zeroed scan regions (the read-through zeroes kScanRegions look-back regions with ONE
  // memset and each scan of the call takes the next one: no memset node per scan)
  uint64_t* ws_scan_multi = nullptr;
  int scan_slot = -1;              // >= 0: the next scan's region; -1: memset per scan
  uint64_t* ws_dcounts = nullptr;  // [0] entries of the derived list [1] its set segments
  bool no_small_sort = false;  // HPS_GPU_NO_SMALL_SORT=1: small batches take the multi-kernel sort too (tests)
};

namespace {

constexpr uint8_t kMiss = 0xff;
constexpr int kScanRegions = 8;

enum { kClock = 0, kSnap = 1, kStats = 2, kScratch = 9 };
enum { sQueries = 0, sHits, sMisses, sInsertions, sRejected, sRefresh, sEvictions };

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// ---- K6a: probe every query against the pre-batch state --------------------------
__global__ void k_probe(const uint64_t* __restrict__ keys, uint64_t n, hps::FastMod64 fm, uint32_t ways,
                        const uint64_t* __restrict__ ckeys, const uint8_t* __restrict__ cfreq,
                        uint32_t* __restrict__ set_out, uint8_t* __restrict__ hit_out, uint64_t* state,
                        uint64_t* counts, const uint64_t* d_n) {
  pdl_wait();
  pdl_launch_dependents();
  if (d_n) n = *d_n;  // key count produced on the device (the orchestrator's distinct keys); n was the bound
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[kSnap] = state[kClock];
    state[kClock] += n;
    counts[0] = n;
    counts[4] = 0;  // huge-set list count of this query's metadata replay (k_query_meta_lanes)
  }
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t s = fm.mod(hps::key_hash(k));
    const uint64_t* kr = ckeys + s * ways;
    const uint8_t* fr = cfreq + s * ways;
    uint8_t hit = kMiss;
    for (uint32_t w = 0; w < ways; ++w) {
      if (fr[w] != 0 && kr[w] == k) {
        hit = static_cast<uint8_t>(w);
        break;
      }
    }
    set_out[i] = static_cast<uint32_t>(s);
    hit_out[i] = hit;
  }
}

// ---- K6b: order-preserving found/missing split --------------------------------------
struct SplitOp {
  const uint8_t* hit;
  uint32_t* found_idx;
  uint32_t* missing_idx;
  uint64_t* counts_out;  // caller's [found, missing]
  uint64_t* counts;      // internal [.., .., found]
  uint64_t* stats;
  uint32_t* miss_rank;   // access -> its position in missing_idx (UINT32_MAX: a hit)
  __device__ uint64_t size() const { return counts[0]; }
  __device__ uint32_t count(uint64_t i) const { return hit[i] != kMiss ? 1u : 0u; }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    if (c) {
      found_idx[excl] = static_cast<uint32_t>(i);
      miss_rank[i] = 0xffffffffu;
    } else {
      missing_idx[i - excl] = static_cast<uint32_t>(i);
      miss_rank[i] = static_cast<uint32_t>(i - excl);
    }
  }
  __device__ void total(uint64_t f) const {
    const uint64_t n = counts[0];
    counts[2] = f;
    counts_out[0] = f;
    counts_out[1] = n - f;
    stats[sQueries] += n;
    stats[sHits] += f;
    stats[sMisses] += n - f;
  }
};

// ---- K6c: gather hit rows (LPR lanes per row, 128-bit loads) ------------------------
// Four cached scalars of entry e, widened to fp32 (binary16 -> fp32 is exact).
template <bool F16>
__device__ __forceinline__ float4 load_cached4(const void* cvec, uint64_t e, uint32_t dim, uint32_t q) {
  if constexpr (F16) {
    const uint2 h = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(cvec) + e * dim) + q);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(cvec) + e * dim) + q);
  }
}

template <int LPR, bool F16>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ found_idx, const uint64_t* counts,
                                                const uint32_t* __restrict__ set_of, const uint8_t* __restrict__ hit,
                                                uint32_t ways, const void* __restrict__ vec, uint32_t dim,
                                                float* __restrict__ out, int scatter) {
  pdl_wait();
  pdl_launch_dependents();
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR;
  const uint64_t nf = counts[2];
  const uint32_t nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  // R rows per group in flight: their positions, then their entries, then their rows are
  // loaded together (a lane group otherwise walks ~2 rows one dependent chain at a time)
  constexpr int R = 4;
  for (uint64_t j0 = gid; j0 < nf; j0 += ng * R) {
    uint32_t i[R];
    uint64_t e[R];
    bool ok[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ok[r] = j0 + uint64_t(r) * ng < nf;
      i[r] = ok[r] ? found_idx[j0 + uint64_t(r) * ng] : 0u;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) e[r] = ok[r] ? uint64_t(set_of[i[r]]) * ways + hit[i[r]] : 0ull;
    // scatter: the row lands at its access position (out[i]) instead of compacted (out[j])
    if (nvec <= LPR) {
      float4 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        x[r] = (ok[r] && gl < nvec) ? load_cached4<F16>(vec, e[r], dim, gl) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ok[r] && gl < nvec)
          reinterpret_cast<float4*>(out + (scatter ? uint64_t(i[r]) : j0 + uint64_t(r) * ng) * dim)[gl] = x[r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!ok[r]) continue;
        float4* dst = reinterpret_cast<float4*>(out + (scatter ? uint64_t(i[r]) : j0 + uint64_t(r) * ng) * dim);
        for (uint32_t v = gl; v < nvec; v += LPR) dst[v] = load_cached4<F16>(vec, e[r], dim, v);
      }
    }
  }
}

// ---- segments of a set-sorted access list -------------------------------------------
struct SetSegOp {
  const uint32_t* sets_sorted;
  uint32_t* seg_start;
  uint64_t* counts;  // [0]=n [1]=U
  __device__ uint64_t size() const { return counts[0]; }
  __device__ uint32_t count(uint64_t i) const {
    return (i == 0 || sets_sorted[i] != sets_sorted[i - 1]) ? 1u : 0u;
  }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    if (c) seg_start[excl] = static_cast<uint32_t>(i);
  }
  __device__ void total(uint64_t u) const {
    counts[1] = u;
    seg_start[u] = static_cast<uint32_t>(counts[0]);
  }
};

__device__ __forceinline__ uint32_t sat_add_freq(uint32_t f, uint32_t x) {
  return f == 0 ? 0u : min(255u, f + x);
}
__device__ __forceinline__ uint32_t age_freq(uint32_t f) { return f == 0 ? 0u : max(1u, f >> 1); }

// ---- K6d: replay the batch's metadata effects per touched set ---------------------------
// Warp-cooperative replay of set s's accesses [lo, hi) (32 at a time, closed form per way:
// saturating adds between aging points).
__device__ __forceinline__ void meta_set_warp(const uint32_t* __restrict__ idx_sorted, const uint8_t* __restrict__ hit,
                                              uint32_t ways, uint64_t aging_period, uint8_t* __restrict__ cfreq,
                                              uint64_t* __restrict__ ctouch, uint64_t* __restrict__ set_acc,
                                              uint64_t clock0, uint64_t s, uint32_t lo, uint32_t hi) {
  const uint32_t lane = lane_id();
  uint32_t f = lane < ways ? cfreq[s * ways + lane] : 0u;
  uint64_t touch = lane < ways ? ctouch[s * ways + lane] : 0ull;
  uint64_t acc = set_acc[s];
  for (uint32_t c = lo; c < hi; c += 32) {
    const uint32_t j = c + lane;
    const bool valid = j < hi;
    const uint32_t i = valid ? idx_sorted[j] : 0u;
    const uint32_t hw = valid ? hit[i] : kMiss;
    const uint32_t cnt = min(32u, hi - c);
    const bool fire = valid && ((acc + lane + 1) % aging_period == 0);
    const uint32_t F = __ballot_sync(0xffffffffu, fire);
    uint32_t H = 0;
    for (uint32_t w = 0; w < ways; ++w) {
      const uint32_t m = __ballot_sync(0xffffffffu, hw == w);
      if (lane == w) H = m;
    }
    uint32_t prev = 0, Fm = F;
    while (Fm) {
      const uint32_t b = __ffs(Fm) - 1;
      Fm &= Fm - 1;
      const uint32_t seg = H & (((b >= 32) ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << prev) - 1u));
      f = age_freq(sat_add_freq(f, __popc(seg)));
      prev = b;
    }
    const uint32_t tailmask = (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u)) & ~((prev >= 32) ? 0xffffffffu : ((1u << prev) - 1u));
    f = sat_add_freq(f, __popc(H & tailmask));
    const uint32_t lastp = H ? 31u - __clz(H) : 0u;
    const uint32_t ilast = __shfl_sync(0xffffffffu, i, lastp);
    if (H) touch = clock0 + ilast + 1;
    acc = (acc + cnt) % aging_period;
  }
  if (lane < ways) {
    cfreq[s * ways + lane] = static_cast<uint8_t>(f);
    ctouch[s * ways + lane] = touch;
  }
  if (lane == 0) set_acc[s] = acc;
}

// Any number of ways: one warp per touched set.
__global__ void __launch_bounds__(256) k_query_meta(const uint32_t* __restrict__ sets_sorted,
                                                    const uint32_t* __restrict__ idx_sorted,
                                                    const uint32_t* __restrict__ seg_start, const uint64_t* counts,
                                                    const uint8_t* __restrict__ hit, uint32_t ways,
                                                    uint64_t aging_period, uint8_t* __restrict__ cfreq,
                                                    uint64_t* __restrict__ ctouch, uint64_t* __restrict__ set_acc,
                                                    const uint64_t* state) {
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t U = counts[1];
  const uint64_t clock0 = state[kSnap];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = warp; u < U; u += n_warps)
    meta_set_warp(idx_sorted, hit, ways, aging_period, cfreq, ctouch, set_acc, clock0, sets_sorted[seg_start[u]],
                  seg_start[u], seg_start[u + 1]);
}

// ways <= 8: a lane replays one set (most sets see one or two accesses per batch), 32 sets
// per warp with every metadata load in flight together; a set with more than
// kLaneMetaMax accesses is replayed by the whole warp afterwards (closed form), and one
// with more than kHugeMeta by k_query_meta_huge.
constexpr uint32_t kLaneMetaMax = 8;
constexpr uint32_t kHugeMeta = 256;
constexpr uint32_t kHugeStage = 8192;
__global__ void __launch_bounds__(256) k_query_meta_lanes(const uint32_t* __restrict__ sets_sorted,
                                                          const uint32_t* __restrict__ idx_sorted,
                                                          const uint32_t* __restrict__ seg_start, const uint64_t* counts,
                                                          const uint8_t* __restrict__ hit, uint32_t ways,
                                                          uint64_t aging_period, uint8_t* __restrict__ cfreq,
                                                          uint64_t* __restrict__ ctouch, uint64_t* __restrict__ set_acc,
                                                          const uint64_t* state, uint32_t* huge_list,
                                                          unsigned long long* n_huge) {
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t lane = lane_id();
  const uint64_t U = counts[1];
  const uint64_t clock0 = state[kSnap];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u0 = warp * 32; u0 < U; u0 += n_warps * 32) {
    const uint64_t u = u0 + lane;
    const bool have = u < U;
    uint32_t lo = 0, hi = 0;
    uint64_t s = 0;
    if (have) {
      lo = seg_start[u];
      hi = seg_start[u + 1];
      s = sets_sorted[lo];
    }
    const bool mine = have && hi - lo <= kLaneMetaMax;
    if (mine) {
      uint32_t f[8];
      uint64_t t[8];
#pragma unroll
      for (uint32_t w = 0; w < 8; ++w) {
        f[w] = w < ways ? cfreq[s * ways + w] : 0u;
        t[w] = w < ways ? ctouch[s * ways + w] : 0ull;
      }
      uint64_t acc = set_acc[s];
      uint32_t ii[kLaneMetaMax], hw[kLaneMetaMax];
#pragma unroll
      for (uint32_t q = 0; q < kLaneMetaMax; ++q) ii[q] = lo + q < hi ? idx_sorted[lo + q] : 0u;
#pragma unroll
      for (uint32_t q = 0; q < kLaneMetaMax; ++q) hw[q] = lo + q < hi ? hit[ii[q]] : kMiss;
#pragma unroll
      for (uint32_t q = 0; q < kLaneMetaMax; ++q) {
        if (lo + q >= hi) break;
        if (++acc >= aging_period) {  // the access that completes an aging period ages first
          acc = 0;
#pragma unroll
          for (uint32_t w = 0; w < 8; ++w) f[w] = age_freq(f[w]);
        }
#pragma unroll
        for (uint32_t w = 0; w < 8; ++w) {
          if (hw[q] == w) {
            f[w] = sat_add_freq(f[w], 1u);
            t[w] = clock0 + ii[q] + 1;
          }
        }
      }
#pragma unroll
      for (uint32_t w = 0; w < 8; ++w) {
        if (w < ways) {
          cfreq[s * ways + w] = static_cast<uint8_t>(f[w]);
          ctouch[s * ways + w] = t[w];
        }
      }
      set_acc[s] = acc;
    }
    const bool huge = have && hi - lo > kHugeMeta;  // k_query_meta_huge replays these
    const uint32_t hm = __ballot_sync(0xffffffffu, huge);
    if (hm) {
      unsigned long long b = 0;
      if (lane == static_cast<uint32_t>(__ffs(hm) - 1)) b = atomicAdd(n_huge, static_cast<unsigned long long>(__popc(hm)));
      b = __shfl_sync(0xffffffffu, b, __ffs(hm) - 1);
      if (huge) huge_list[b + __popc(hm & lanemask_lt())] = static_cast<uint32_t>(u);
    }
    uint32_t longs = __ballot_sync(0xffffffffu, have && !mine && !huge);
    while (longs) {
      const int src = __ffs(longs) - 1;
      longs &= longs - 1;
      const uint32_t slo = __shfl_sync(0xffffffffu, lo, src), shi = __shfl_sync(0xffffffffu, hi, src);
      const uint64_t ss = __shfl_sync(0xffffffffu, s, src);
      meta_set_warp(idx_sorted, hit, ways, aging_period, cfreq, ctouch, set_acc, clock0, ss, slo, shi);
    }
  }
}

// Sets with more than kHugeMeta accesses in the batch (Zipf-head keys: thousands): one CTA
// per set gathers the accesses' hit ways and indices into shared memory with all its
// threads (kHugeStage at a time). Aging fires every P accesses, so (P >= 32) the whole CTA
// counts each way's hits per aging segment and its last hit (shared atomics) and the
// sequential part is one step per segment: f = sat(f + hits); f = age(f); ...
// (identical to the per-access semantics). Small P: the 32-access closed form, from smem.
constexpr uint32_t kHugeSegs = kHugeStage / 32 + 2;
__global__ void __launch_bounds__(256) k_query_meta_huge(const uint32_t* __restrict__ sets_sorted,
                                                         const uint32_t* __restrict__ idx_sorted,
                                                         const uint32_t* __restrict__ seg_start,
                                                         const uint32_t* __restrict__ huge_list, const uint64_t* n_huge,
                                                         const uint8_t* __restrict__ hit, uint32_t ways,
                                                         uint64_t aging_period, uint8_t* __restrict__ cfreq,
                                                         uint64_t* __restrict__ ctouch, uint64_t* __restrict__ set_acc,
                                                         const uint64_t* state) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ uint32_t s_idx[kHugeStage];
  __shared__ uint8_t s_hw[kHugeStage];
  __shared__ uint16_t s_cnt[kHugeSegs][8];  // hits per (aging segment, way)
  __shared__ uint32_t s_last[8];            // last hit position per way (+1; 0 = none)
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  const uint64_t clock0 = state[kSnap];
  const uint64_t nh = *n_huge;
  for (uint64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const uint32_t u = huge_list[h];
    const uint32_t lo = seg_start[u], hi = seg_start[u + 1];
    const uint64_t s = sets_sorted[lo];
    uint32_t f = 0, acc32 = 0;
    uint64_t touch = 0;
    if (w == 0) {
      f = lane < ways ? cfreq[s * ways + lane] : 0u;
      touch = lane < ways ? ctouch[s * ways + lane] : 0ull;
      acc32 = static_cast<uint32_t>(set_acc[s]);  // < aging_period < 2^32
    }
    const uint32_t P = static_cast<uint32_t>(aging_period);
    for (uint32_t b0 = lo; b0 < hi; b0 += kHugeStage) {
      const uint32_t nb = min(kHugeStage, hi - b0);
      __syncthreads();  // the previous stage is consumed
      const uint32_t P_acc = __shfl_sync(0xffffffffu, acc32, 0);  // (warp 0's; broadcast below)
      if (w == 0 && lane == 0) s_last[0] = P_acc;
      __syncthreads();
      const uint32_t acc_in = s_last[0];
      __syncthreads();
      const bool seg_mode = P >= 32 && ways <= 8;
      if (seg_mode) {
        for (uint32_t e = threadIdx.x; e < kHugeSegs * 8; e += blockDim.x) (&s_cnt[0][0])[e] = 0;
        if (threadIdx.x < 8) s_last[threadIdx.x] = 0;
        __syncthreads();
      }
      // first aging point of this stage: access q0 = P - 1 - acc_in (acc_in < P)
      const uint32_t q0 = P - 1 - acc_in;
      for (uint32_t q = threadIdx.x; q < nb; q += blockDim.x) {
        const uint32_t i = idx_sorted[b0 + q];
        const uint32_t hw = hit[i];
        s_idx[q] = i;
        s_hw[q] = static_cast<uint8_t>(hw);
        if (seg_mode && hw < ways) {
          const uint32_t k = q < q0 ? 0u : 1u + (q - q0) / P;  // segment k >= 1 starts at an aging point
          atomicAdd(reinterpret_cast<unsigned int*>(&s_cnt[0][0]) + ((k * 8 + hw) >> 1), 1u << (16 * ((k * 8 + hw) & 1)));
          atomicMax(&s_last[hw], q + 1);
        }
      }
      __syncthreads();
      if (seg_mode) {
        if (w == 0) {
          const uint32_t n_seg = nb <= q0 ? 1u : 2u + (nb - 1 - q0) / P;
          if (lane < ways) {
            f = sat_add_freq(f, s_cnt[0][lane]);
            for (uint32_t k = 1; k < n_seg; ++k) f = sat_add_freq(age_freq(f), s_cnt[k][lane]);
            if (s_last[lane]) touch = clock0 + s_idx[s_last[lane] - 1] + 1;
          }
          acc32 = (acc32 + nb) % P;
        }
        continue;
      }
      if (w == 0) {
        for (uint32_t c = 0; c < nb; c += 32) {
          const uint32_t q = c + lane;
          const bool valid = q < nb;
          const uint32_t hw = valid ? s_hw[q] : kMiss;
          const uint32_t cnt = min(32u, nb - c);
          const bool fire = valid && (acc32 + lane + 1) % P == 0;
          const uint32_t F = __ballot_sync(0xffffffffu, fire);
          uint32_t H = 0;
          for (uint32_t ww = 0; ww < ways; ++ww) {
            const uint32_t m = __ballot_sync(0xffffffffu, hw == ww);
            if (lane == ww) H = m;
          }
          uint32_t prev = 0, Fm = F;
          while (Fm) {
            const uint32_t b = __ffs(Fm) - 1;
            Fm &= Fm - 1;
            const uint32_t seg = H & (((b >= 32) ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << prev) - 1u));
            f = age_freq(sat_add_freq(f, __popc(seg)));
            prev = b;
          }
          const uint32_t tailmask =
              (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u)) & ~((prev >= 32) ? 0xffffffffu : ((1u << prev) - 1u));
          f = sat_add_freq(f, __popc(H & tailmask));
          if (H) touch = clock0 + s_idx[c + 31u - __clz(H)] + 1;
          acc32 = (acc32 + cnt) % P;
        }
      }
    }
    if (w == 0) {
      if (lane < ways) {
        cfreq[s * ways + lane] = static_cast<uint8_t>(f);
        ctouch[s * ways + lane] = touch;
      }
      if (lane == 0) set_acc[s] = acc32;
    }
  }
}

// ---- K7/K8 prep: validate rows (NaN/Inf -> NonFinite; binary16 storage: out of range ->
// F16Range), set id, validity ----------------------------------------------------------
__device__ __forceinline__ bool f16_overflows(uint32_t bits) { return (bits & 0x7fffffffu) >= 0x477ff000u; }

template <int LPR>
__global__ void __launch_bounds__(256) k_entry_prep(const uint64_t* __restrict__ keys, const float* __restrict__ vecs,
                                                    uint64_t n, uint32_t dim, hps::FastMod64 fm, uint32_t invalid_set,
                                                    uint32_t* __restrict__ set_out, uint8_t* __restrict__ valid_out,
                                                    uint32_t* status, uint64_t* counts, const uint64_t* d_n,
                                                    const uint8_t* __restrict__ skip, int f16, uint64_t* zero_out) {
  pdl_wait();
  pdl_launch_dependents();
  if (zero_out && blockIdx.x == 0 && threadIdx.x == 0) *zero_out = 0;  // the call's admitted count
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR;
  const uint32_t gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const uint32_t nvec = dim / 4;
  if (d_n) n = min(n, *d_n);  // entry count produced on the device (read-through path)
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = n;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t i = gid; i < n; i += ng) {
    const uint4* v = reinterpret_cast<const uint4*>(vecs + i * dim);
    bool bad = false, range = false;
    for (uint32_t q = gl; q < nvec; q += LPR) {
      const uint4 x = __ldg(v + q);
      bad |= non_finite_bits(x.x) | non_finite_bits(x.y) | non_finite_bits(x.z) | non_finite_bits(x.w);
      // binary16 storage: |x| >= 65520 rounds to infinity (the largest finite is 65504)
      if (f16) range |= f16_overflows(x.x) | f16_overflows(x.y) | f16_overflows(x.z) | f16_overflows(x.w);
    }
    bad = __any_sync(gmask, bad);
    range = __any_sync(gmask, range) && !bad;
    if (gl == 0) {
      if (bad) latch_status(status, HPS_GPU_E_NON_FINITE);
      if (range) latch_status(status, HPS_GPU_E_F16_RANGE);
      const bool skipped = bad || range || (skip && skip[i]);  // skip: absent from the backing store
      set_out[i] = skipped ? invalid_set : static_cast<uint32_t>(fm.mod(hps::key_hash(keys[i])));
      valid_out[i] = skipped ? 0 : 1;
    }
  }
}

// rank among valid entries (the access clock of an insert), and the clock reservation
struct RankOp {
  const uint8_t* valid;
  uint32_t* rank;
  uint64_t* counts;
  uint64_t* state;
  __device__ uint64_t size() const { return counts[0]; }
  __device__ uint32_t count(uint64_t i) const { return valid[i]; }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t) const { rank[i] = static_cast<uint32_t>(excl); }
  __device__ void total(uint64_t nv) const {
    counts[3] = nv;
    state[kSnap] = state[kClock];
    state[kClock] += nv;
  }
};

// One fp32 row into cached entry e (warp-wide); binary16 storage rounds to nearest even
// (cvt.rn.f16x2.f32, the reference's f32_to_f16: kernels_scalar.cpp:25-57).
template <bool F16>
__device__ __forceinline__ void warp_store_row(void* cvec, uint64_t e, const float* src, uint32_t dim) {
  const uint32_t nvec = dim / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  if constexpr (F16) {
    uint2* d = reinterpret_cast<uint2*>(static_cast<__half*>(cvec) + e * dim);
    for (uint32_t q = lane_id(); q < nvec; q += 32) {
      const float4 x = __ldg(s4 + q);
      const __half2 lo = __floats2half2_rn(x.x, x.y), hi = __floats2half2_rn(x.z, x.w);
      d[q] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  } else {
    float4* d4 = reinterpret_cast<float4*>(static_cast<float*>(cvec) + e * dim);
    for (uint32_t q = lane_id(); q < nvec; q += 32) d4[q] = __ldg(s4 + q);
  }
}

// ---- K7: insert, one warp per touched set, entries in input order --------------------
template <bool F16>
__global__ void __launch_bounds__(256) k_insert_sets(const uint32_t* __restrict__ sets_sorted,
                                                     const uint32_t* __restrict__ idx_sorted,
                                                     const uint32_t* __restrict__ seg_start, const uint64_t* counts,
                                                     const uint64_t* __restrict__ keys, const float* __restrict__ vecs,
                                                     const uint64_t* __restrict__ versions,
                                                     const uint32_t* __restrict__ rank, uint32_t ways, uint32_t dim,
                                                     uint64_t aging_period, uint32_t invalid_set, uint64_t* ckeys,
                                                     uint64_t* cver, uint8_t* cfreq, uint64_t* ctouch, uint64_t* set_acc,
                                                     void* cvec, uint64_t* state, uint64_t* admitted_out) {
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t lane = lane_id();
  const uint64_t U = counts[1];
  const uint64_t clock0 = state[kSnap];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t n_ins = 0, n_evict = 0, n_refresh = 0;
  for (uint64_t u = warp; u < U; u += n_warps) {
    const uint32_t lo = seg_start[u], hi = seg_start[u + 1];
    const uint32_t s32 = sets_sorted[lo];
    if (s32 == invalid_set) continue;
    const uint64_t s = s32, e0 = s * ways;
    const bool way = lane < ways;
    uint64_t k_w = way ? ckeys[e0 + lane] : 0, v_w = way ? cver[e0 + lane] : 0, t_w = way ? ctouch[e0 + lane] : 0;
    uint32_t f_w = way ? cfreq[e0 + lane] : 0;
    uint64_t acc = set_acc[s];
    for (uint32_t j = lo; j < hi; ++j) {
      const uint32_t i = idx_sorted[j];
      const uint64_t k = keys[i], ver = versions ? versions[i] : hps::kBulkLoadVersion;
      const uint64_t t = clock0 + rank[i] + 1;
      if (++acc >= aging_period) {
        acc = 0;
        f_w = age_freq(f_w);
      }
      const uint32_t res = __ballot_sync(0xffffffffu, way && f_w != 0 && k_w == k);
      if (res) {  // resident: refresh semantics (version-gated replace, no freq/touch change)
        const int w = __ffs(res) - 1;
        const uint64_t vw = __shfl_sync(0xffffffffu, v_w, w);
        if (ver > vw) {
          warp_store_row<F16>(cvec, e0 + w, vecs + uint64_t(i) * dim, dim);
          if (lane == static_cast<uint32_t>(w)) v_w = ver;
          ++n_refresh;
        }
        continue;
      }
      const uint32_t free_ways = __ballot_sync(0xffffffffu, way && f_w == 0);
      int w;
      if (free_ways) {
        w = __ffs(free_ways) - 1;
      } else {  // victim = min (freq, last_touch)
        uint32_t bf = way ? f_w : 0xffffffffu;
        uint64_t bt = way ? t_w : ~0ull;
        uint32_t bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint32_t of = __shfl_xor_sync(0xffffffffu, bf, o);
          const uint64_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
          const uint32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
          if (of < bf || (of == bf && (ot < bt || (ot == bt && ol < bl)))) {
            bf = of;
            bt = ot;
            bl = ol;
          }
        }
        w = static_cast<int>(bl);
        ++n_evict;
      }
      if (lane == static_cast<uint32_t>(w)) {
        k_w = k;
        v_w = ver;
        f_w = 1;
        t_w = t;
      }
      warp_store_row<F16>(cvec, e0 + w, vecs + uint64_t(i) * dim, dim);
      ++n_ins;
    }
    if (way) {
      ckeys[e0 + lane] = k_w;
      cver[e0 + lane] = v_w;
      cfreq[e0 + lane] = static_cast<uint8_t>(f_w);
      ctouch[e0 + lane] = t_w;
    }
    if (lane == 0) set_acc[s] = acc;
  }
  if (lane == 0 && (n_ins | n_evict | n_refresh)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sInsertions]), n_ins);
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sEvictions]), n_evict);
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sRefresh]), n_refresh);
    if (admitted_out) atomicAdd(reinterpret_cast<unsigned long long*>(admitted_out), n_ins);
  }
}

// ---- K7, narrow sets (ways <= 8): four sets per warp, an 8-lane group each -------------
// The same replay as k_insert_sets (entries of a set in input order; resident -> version-gated
// refresh, else the lowest free way, else the (freq, last_touch, way) minimum is evicted),
// with a set's ways on the 8 lanes of one group: four sets' dependent load chains in flight per
// warp instead of one. Rows are copied by the group (lane l of 8: float4s l, l + 8, ...).
template <bool F16>
__device__ __forceinline__ void group_store_row(void* cvec, uint64_t e, const float* src, uint32_t dim, uint32_t gl) {
  const uint32_t nvec = dim / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  if constexpr (F16) {
    uint2* d = reinterpret_cast<uint2*>(static_cast<__half*>(cvec) + e * dim);
    for (uint32_t q = gl; q < nvec; q += 8) {
      const float4 x = __ldg(s4 + q);
      const __half2 lo = __floats2half2_rn(x.x, x.y), hi = __floats2half2_rn(x.z, x.w);
      d[q] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  } else {
    float4* d4 = reinterpret_cast<float4*>(static_cast<float*>(cvec) + e * dim);
    for (uint32_t q = gl; q < nvec; q += 8) d4[q] = __ldg(s4 + q);
  }
}

template <bool F16>
__global__ void __launch_bounds__(256) k_insert_sets8(const uint32_t* __restrict__ sets_sorted,
                                                     const uint32_t* __restrict__ idx_sorted,
                                                     const uint32_t* __restrict__ seg_start, const uint64_t* counts,
                                                     const uint64_t* __restrict__ keys, const float* __restrict__ vecs,
                                                     const uint64_t* __restrict__ versions,
                                                     const uint32_t* __restrict__ rank, uint32_t ways, uint32_t dim,
                                                     uint64_t aging_period, uint32_t invalid_set, uint64_t* ckeys,
                                                     uint64_t* cver, uint8_t* cfreq, uint64_t* ctouch, uint64_t* set_acc,
                                                     void* cvec, uint64_t* state, uint64_t* admitted_out,
                                                     const uint32_t* __restrict__ entry_of,
                                                     const uint8_t* __restrict__ entry_valid) {
  // entry_of != nullptr: the segments are a QUERY's (cache_insert_after_query): access u is
  // insert entry entry_of[u] (UINT32_MAX: a hit), taken only when entry_valid[] — the query's
  // set grouping serves the insert directly, no compacted copy of it
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t lane = lane_id(), g = lane >> 3, gl = lane & 7u;
  const uint32_t gmask = 0xffu << (8 * g);
  const uint64_t U = counts[1];
  const uint64_t clock0 = state[kSnap];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_groups = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * 4;
  uint64_t n_ins = 0, n_evict = 0, n_refresh = 0;
  for (uint64_t u = warp * 4 + g; u < U; u += n_groups) {
    const uint32_t lo = seg_start[u], hi = seg_start[u + 1];
    const uint32_t s32 = sets_sorted[lo];
    if (s32 == invalid_set) continue;
    if (entry_of) {  // a set none of whose accesses is an insert entry is left alone
      bool any = false;
      for (uint32_t j = lo; j < hi && !any; ++j) {
        const uint32_t m = entry_of[idx_sorted[j]];
        any = m != 0xffffffffu && entry_valid[m];
      }
      if (!any) continue;
    }
    const uint64_t s = s32, e0 = s * ways;
    const bool way = gl < ways;
    // the set's metadata and its first entry are loaded together
    uint64_t k_w = way ? ckeys[e0 + gl] : 0, v_w = way ? cver[e0 + gl] : 0, t_w = way ? ctouch[e0 + gl] : 0;
    uint32_t f_w = way ? cfreq[e0 + gl] : 0;
    uint64_t acc = set_acc[s];
    for (uint32_t j = lo; j < hi; ++j) {
      uint32_t i = idx_sorted[j];
      if (entry_of) {
        const uint32_t m = entry_of[i];
        if (m == 0xffffffffu || !entry_valid[m]) continue;
        i = m;
      }
      const uint64_t k = keys[i], ver = versions ? versions[i] : hps::kBulkLoadVersion;
      const uint64_t t = clock0 + rank[i] + 1;
      if (++acc >= aging_period) {
        acc = 0;
        f_w = age_freq(f_w);
      }
      const uint32_t res = (__ballot_sync(gmask, way && f_w != 0 && k_w == k) >> (8 * g)) & 0xffu;
      if (res) {  // resident: refresh semantics
        const int w = __ffs(res) - 1;
        const uint64_t vw = __shfl_sync(gmask, v_w, 8 * g + w);
        if (ver > vw) {
          group_store_row<F16>(cvec, e0 + w, vecs + uint64_t(i) * dim, dim, gl);
          if (gl == static_cast<uint32_t>(w)) v_w = ver;
          ++n_refresh;
        }
        continue;
      }
      const uint32_t free_ways = (__ballot_sync(gmask, way && f_w == 0) >> (8 * g)) & 0xffu;
      int w;
      if (free_ways) {
        w = __ffs(free_ways) - 1;
      } else {  // victim = min (freq, last_touch, way) over the group's lanes
        uint32_t bf = way ? f_w : 0xffffffffu;
        uint64_t bt = way ? t_w : ~0ull;
        uint32_t bl = gl;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          const uint32_t of = __shfl_xor_sync(gmask, bf, o);
          const uint64_t ot = __shfl_xor_sync(gmask, bt, o);
          const uint32_t ol = __shfl_xor_sync(gmask, bl, o);
          if (of < bf || (of == bf && (ot < bt || (ot == bt && ol < bl)))) {
            bf = of;
            bt = ot;
            bl = ol;
          }
        }
        w = static_cast<int>(bl);
        ++n_evict;
      }
      if (gl == static_cast<uint32_t>(w)) {
        k_w = k;
        v_w = ver;
        f_w = 1;
        t_w = t;
      }
      group_store_row<F16>(cvec, e0 + w, vecs + uint64_t(i) * dim, dim, gl);
      ++n_ins;
    }
    if (way) {
      ckeys[e0 + gl] = k_w;
      cver[e0 + gl] = v_w;
      cfreq[e0 + gl] = static_cast<uint8_t>(f_w);
      ctouch[e0 + gl] = t_w;
    }
    if (gl == 0) set_acc[s] = acc;
  }
  // counts are per group (every lane of a group counted the same events): lane gl == 0 adds;
  // summed per CTA in shared memory first, so a large batch's thousands of inserting warps
  // do not serialise on the three global counters
  __shared__ unsigned long long s_cnt[3];
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0ull;
  __syncthreads();
  if (gl != 0) n_ins = n_evict = n_refresh = 0;
  n_ins = warp_sum(n_ins);
  n_evict = warp_sum(n_evict);
  n_refresh = warp_sum(n_refresh);
  if (lane == 0 && (n_ins | n_evict | n_refresh)) {
    atomicAdd(&s_cnt[0], static_cast<unsigned long long>(n_ins));
    atomicAdd(&s_cnt[1], static_cast<unsigned long long>(n_evict));
    atomicAdd(&s_cnt[2], static_cast<unsigned long long>(n_refresh));
  }
  __syncthreads();
  if (threadIdx.x == 0 && (s_cnt[0] | s_cnt[1] | s_cnt[2])) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sInsertions]), s_cnt[0]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sEvictions]), s_cnt[1]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sRefresh]), s_cnt[2]);
    if (admitted_out) atomicAdd(reinterpret_cast<unsigned long long*>(admitted_out), s_cnt[0]);
  }
}

// ---- K8: refresh, one warp per touched set ------------------------------------------
template <bool F16>
__global__ void __launch_bounds__(256) k_refresh_sets(const uint32_t* __restrict__ sets_sorted,
                                                      const uint32_t* __restrict__ idx_sorted,
                                                      const uint32_t* __restrict__ seg_start, const uint64_t* counts,
                                                      const uint64_t* __restrict__ keys, const float* __restrict__ vecs,
                                                      const uint64_t* __restrict__ versions, uint32_t ways,
                                                      uint32_t dim, uint32_t invalid_set, const uint64_t* ckeys,
                                                      uint64_t* cver, const uint8_t* cfreq, void* cvec,
                                                      uint64_t* state, uint64_t* replaced_out) {
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t lane = lane_id();
  const uint64_t U = counts[1];
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t n_rep = 0;
  for (uint64_t u = warp; u < U; u += n_warps) {
    const uint32_t lo = seg_start[u], hi = seg_start[u + 1];
    const uint32_t s32 = sets_sorted[lo];
    if (s32 == invalid_set) continue;
    const uint64_t e0 = uint64_t(s32) * ways;
    const bool way = lane < ways;
    const uint64_t k_w = way ? ckeys[e0 + lane] : 0;
    const uint32_t f_w = way ? cfreq[e0 + lane] : 0;
    uint64_t v_w = way ? cver[e0 + lane] : 0;
    for (uint32_t j = lo; j < hi; ++j) {
      const uint32_t i = idx_sorted[j];
      const uint64_t k = keys[i], ver = versions[i];
      const uint32_t res = __ballot_sync(0xffffffffu, way && f_w != 0 && k_w == k);
      if (!res) continue;
      const int w = __ffs(res) - 1;
      const uint64_t vw = __shfl_sync(0xffffffffu, v_w, w);
      if (ver > vw) {
        warp_store_row<F16>(cvec, e0 + w, vecs + uint64_t(i) * dim, dim);
        if (lane == static_cast<uint32_t>(w)) v_w = ver;
        ++n_rep;
      }
    }
    if (way) cver[e0 + lane] = v_w;
  }
  if (lane == 0 && n_rep) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&state[kStats + sRefresh]), n_rep);
    if (replaced_out) atomicAdd(reinterpret_cast<unsigned long long*>(replaced_out), n_rep);
  }
}

__global__ void k_count_resident(const uint8_t* __restrict__ freq, uint64_t n, unsigned long long* out) {
  uint64_t c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    c += freq[i] != 0;
  c = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(c));
  if (lane_id() == 0 && c) atomicAdd(out, static_cast<unsigned long long>(c));
}

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return HPS_GPU_OK;
  if (cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    set_last_error("cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}

int check_cache(hps_gpu_cache c) {
  if (!c) {
    set_last_error("null cache handle");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  return HPS_GPU_OK;
}

int lpr_for(uint32_t dim) {
  const uint32_t nvec = dim / 4;
  return nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
}

// Small batches (n_max <= kSmallSort): the stable (set id, input index) sort and the set
// segments in ONE single-CTA kernel (block radix sort in shared memory + a block scan over
// the segment heads) instead of histogram + onesweep passes + a segment scan: a batch of
// a few keys is bound by launches, not bytes. Same outputs as the multi-kernel path.
constexpr int kSmallSortThreads = 512;
constexpr int kSmallSortIPT = 4;
constexpr uint64_t kSmallSort = uint64_t(kSmallSortThreads) * kSmallSortIPT;

__global__ void __launch_bounds__(kSmallSortThreads) k_small_sort_segment(const uint32_t* __restrict__ sets,
                                                                          uint64_t* counts, int bits,
                                                                          uint32_t* __restrict__ sets_out,
                                                                          uint32_t* __restrict__ idx_out,
                                                                          uint32_t* __restrict__ seg_start) {
  pdl_wait();
  pdl_launch_dependents();
  using Sort = cub::BlockRadixSort<uint32_t, kSmallSortThreads, kSmallSortIPT, uint32_t>;
  using Scan = cub::BlockScan<uint32_t, kSmallSortThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_key[kSmallSort];
  const uint32_t n = static_cast<uint32_t>(counts[0]);
  const uint32_t pad = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);  // pads sort after equal keys (stable)
  uint32_t k[kSmallSortIPT], v[kSmallSortIPT];
#pragma unroll
  for (int q = 0; q < kSmallSortIPT; ++q) {  // blocked arrangement: item i = t * IPT + q
    const uint32_t i = threadIdx.x * kSmallSortIPT + q;
    k[q] = i < n ? sets[i] : pad;
    v[q] = i;
  }
  Sort(tmp.sort).Sort(k, v, 0, bits <= 0 ? 1 : bits);
#pragma unroll
  for (int q = 0; q < kSmallSortIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallSortIPT + q;
    s_key[i] = k[q];
    if (i < n) {
      sets_out[i] = k[q];
      idx_out[i] = v[q];
    }
  }
  __syncthreads();
  uint32_t head[kSmallSortIPT], excl[kSmallSortIPT], total = 0;
#pragma unroll
  for (int q = 0; q < kSmallSortIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallSortIPT + q;
    head[q] = (i < n && (i == 0 || s_key[i] != s_key[i - 1])) ? 1u : 0u;
  }
  Scan(tmp.scan).ExclusiveSum(head, excl, total);
#pragma unroll
  for (int q = 0; q < kSmallSortIPT; ++q)
    if (head[q]) seg_start[excl[q]] = threadIdx.x * kSmallSortIPT + q;
  if (threadIdx.x == 0) {
    counts[1] = total;
    seg_start[total] = n;
  }
}

// One device-wide scan of the cache: its own pre-zeroed region when the caller armed them
// (cache_arm_scans), else the shared region with a memset first.
template <class Op>
cudaError_t cache_scan(hps_gpu_cache c, const Op& op, uint64_t n_max) {
  cudaStream_t st = c->ctx->stream;
  const uint64_t tiles = scan_tiles(n_max);
  if (c->scan_slot < 0 || c->scan_slot >= kScanRegions || tiles <= 1) return launch_scan(op, n_max, c->ws_scan, st);
  uint64_t* status = c->ws_scan_multi + uint64_t(c->scan_slot++) * (scan_tiles(c->max_batch) + 2);
  k_scan<Op><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, status, reinterpret_cast<uint32_t*>(status + tiles));
  return cudaGetLastError();
}

// ---- counting grouping (large caches: sets >= 8 x max_batch) -----------------------------
// The same products as the radix sort — every set's accesses contiguous, in input order —
// from per-set counters instead of 3 digit passes: an arrival ticket per access, each set's
// first arrival reserves the set's range (one counter), every access lands at
// range + ticket, and one thread per range puts it back into input order (insertion sort: a
// range holds ~1 access when the sets outnumber the batch 8:1) and zeroes the counter.
// Segments come out in the order of their first-arriving access, not by set id: every
// consumer treats segments independently.
__global__ void __launch_bounds__(256) k_group_count(const uint32_t* __restrict__ sets, const uint64_t* counts,
                                                     uint32_t* cnt, uint32_t* __restrict__ ticket,
                                                     unsigned long long* range_total) {
  pdl_wait();
  pdl_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x == 0) *range_total = 0ull;  // k_group_alloc's allocator
  const uint64_t n = counts[0];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    ticket[i] = atomicAdd(&cnt[sets[i]], 1u);
}
// Each set's first arrival reserves its range from one counter (warp-aggregated): the ranges
// come out in allocation order, which no consumer depends on (segments are independent).
__global__ void __launch_bounds__(256) k_group_alloc(const uint32_t* __restrict__ sets, const uint32_t* __restrict__ ticket,
                                                     uint32_t* cnt, const uint64_t* counts,
                                                     unsigned long long* range_total) {
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t n = counts[0];
  const uint32_t lane = lane_id();
  for (uint64_t i0 = blockIdx.x * uint64_t(blockDim.x); i0 < n; i0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool lead = i < n && ticket[i] == 0;
    const uint32_t s = lead ? sets[i] : 0u;
    const uint32_t len = lead ? cnt[s] : 0u;
    const uint32_t incl = warp_incl_scan(len);
    unsigned long long base = 0;
    if (lane == 31 && incl) base = atomicAdd(range_total, static_cast<unsigned long long>(incl));
    base = __shfl_sync(0xffffffffu, base, 31);
    if (lead) cnt[s] = static_cast<uint32_t>(base + incl - len);
  }
}
__global__ void __launch_bounds__(256) k_group_place(const uint32_t* __restrict__ sets, const uint32_t* __restrict__ ticket,
                                                     const uint32_t* __restrict__ cnt, const uint64_t* counts,
                                                     uint32_t* __restrict__ out_set, uint32_t* __restrict__ out_idx) {
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t n = counts[0];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = sets[i];
    const uint32_t pos = cnt[s] + ticket[i];
    out_set[pos] = s;
    out_idx[pos] = static_cast<uint32_t>(i);
  }
}
__global__ void __launch_bounds__(256) k_group_fix(const uint32_t* __restrict__ out_set, uint32_t* out_idx,
                                                   const uint64_t* counts, uint32_t* cnt) {
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t n = counts[0];
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = out_set[j];
    if (j > 0 && out_set[j - 1] == s) continue;  // not the range's head
    uint64_t L = 1;
    while (j + L < n && out_set[j + L] == s) ++L;
    for (uint64_t a = j + 1; a < j + L; ++a) {  // input order (insertion sort)
      const uint32_t v = out_idx[a];
      uint64_t b = a;
      while (b > j && out_idx[b - 1] > v) {
        out_idx[b] = out_idx[b - 1];
        --b;
      }
      out_idx[b] = v;
    }
    cnt[s] = 0u;  // the counter is zero at rest again
  }
}

// Stable sort of (set id, input index) + set segments. Sizes come from c->ws_counts[0].
int sort_and_segment(hps_gpu_cache c, uint64_t n, int bits, const uint32_t** sets_sorted,
                     const uint32_t** idx_sorted, bool distinct = false) {
  cudaStream_t st = c->ctx->stream;
  // only for distinct keys (the read-through's deduplicated query): a range then holds the
  // distinct keys of one set, ~1 when the sets outnumber the batch 8:1; repeated keys (the
  // public query/insert/refresh entries) could pile thousands into one range — radix sort there
  if (c->count_group && distinct && n > kSmallSort) {
    const int g = grid_for(n, 256, kNumSMs * 8);
    auto* range_total = reinterpret_cast<unsigned long long*>(c->ws_counts + 6);
    HPSG_CUDA(launch_k(true, k_group_count, g, 256, 0, st, static_cast<const uint32_t*>(c->ws_set),
                       static_cast<const uint64_t*>(c->ws_counts), c->ws_setcnt, c->ws_ticket, range_total));
    HPSG_CUDA(launch_k(true, k_group_alloc, g, 256, 0, st, static_cast<const uint32_t*>(c->ws_set),
                       static_cast<const uint32_t*>(c->ws_ticket), c->ws_setcnt,
                       static_cast<const uint64_t*>(c->ws_counts), range_total));
    HPSG_CUDA(launch_k(true, k_group_place, g, 256, 0, st, static_cast<const uint32_t*>(c->ws_set),
                       static_cast<const uint32_t*>(c->ws_ticket), static_cast<const uint32_t*>(c->ws_setcnt),
                       static_cast<const uint64_t*>(c->ws_counts), c->ws_keys_b, c->ws_vals_b));
    HPSG_CUDA(launch_k(true, k_group_fix, g, 256, 0, st, static_cast<const uint32_t*>(c->ws_keys_b), c->ws_vals_b,
                       static_cast<const uint64_t*>(c->ws_counts), c->ws_setcnt));
    *sets_sorted = c->ws_keys_b;
    *idx_sorted = c->ws_vals_b;
    SetSegOp op{*sets_sorted, c->ws_seg, c->ws_counts};
    HPSG_CUDA(cache_scan(c, op, n));
    HPSG_CHECK_LAUNCH("counting set grouping");
    return HPS_GPU_OK;
  }
  if (n <= kSmallSort && !c->no_small_sort) {
    launch_k(true, k_small_sort_segment, 1, kSmallSortThreads, 0, st, c->ws_set, c->ws_counts, bits, c->ws_keys_b, c->ws_vals_b,
                                                          c->ws_seg);
    HPSG_CHECK_LAUNCH("small sort + segments");
    *sets_sorted = c->ws_keys_b;
    *idx_sorted = c->ws_vals_b;
    return HPS_GPU_OK;
  }
  cudaError_t err;
  const bool in_b = radix_sort_pairs(st, c->ws_set, nullptr, c->ws_vals_a, c->ws_keys_b, c->ws_vals_b, c->ws_counts,
                                     n, bits, c->ws_sort, &err);
  if (err != cudaSuccess) return cuda_status(err, "cache radix sort");
  *sets_sorted = in_b ? c->ws_keys_b : c->ws_set;
  *idx_sorted = in_b ? c->ws_vals_b : c->ws_vals_a;
  SetSegOp op{*sets_sorted, c->ws_seg, c->ws_counts};
  HPSG_CUDA(cache_scan(c, op, n));
  HPSG_CHECK_LAUNCH("set segments");
  return HPS_GPU_OK;
}

int set_warps_grid(uint64_t n) { return grid_for(n * 32, 256, kNumSMs * 16); }

// An insert of a query's misses (the read-through's migration) grouped by set WITHOUT a sort:
// the query's access list is already sorted by (set, query position), and the misses are a
// subsequence of it whose query positions ascend with their insert positions (the missing
// list is ascending). Keeping, in list order, the elements that missed and are valid insert
// entries gives exactly the stable set sort of the insert's valid entries — the segment of
// skipped entries (absent from the lower tier, non-finite) is simply not there. Element j's
// insert position is the query's miss rank of its access (SplitOp).
struct DeriveOp {
  const uint32_t* q_sets;
  const uint32_t* q_idx;
  const uint64_t* q_n;        // the query's access count
  const uint32_t* miss_rank;  // query access -> insert entry (UINT32_MAX: a hit)
  const uint8_t* valid;       // per insert entry (k_entry_prep)
  uint32_t* out_set;
  uint32_t* out_idx;
  uint64_t* dcounts;
  __device__ uint64_t size() const { return *q_n; }
  __device__ uint32_t count(uint64_t j) const {
    const uint32_t m = miss_rank[q_idx[j]];
    return (m != 0xffffffffu && valid[m]) ? 1u : 0u;
  }
  __device__ void emit(uint64_t j, uint64_t excl, uint32_t c) const {
    if (c) {
      out_set[excl] = q_sets[j];
      out_idx[excl] = miss_rank[q_idx[j]];
    }
  }
  __device__ void total(uint64_t t) const { dcounts[0] = t; }
};

}  // namespace

extern "C" {

int hps_gpu_cache_create(hps_gpu_ctx ctx, const hps_cache_config* cfg, hps_gpu_cache* out) {
  if (!ctx || !cfg || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  const uint32_t ways = cfg->ways ? cfg->ways : 8;
  if (ways > 32 || cfg->capacity < ways || cfg->capacity % ways != 0 || cfg->dim == 0 || cfg->dim > 4096 ||
      cfg->max_batch == 0 || cfg->max_batch >= (1ull << 31)) {
    set_last_error("cache config: need 1<=ways<=32, capacity % ways == 0, 1<=dim<=4096, 1<=max_batch<2^31");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (cfg->capacity / ways >= 0xffffffffull) return HPS_GPU_E_INVALID_ARGUMENT;
  if (cfg->dtype != HPS_DTYPE_F32 && cfg->dtype != HPS_DTYPE_F16) {
    set_last_error("cache config: dtype must be HPS_DTYPE_F32 or HPS_DTYPE_F16");
    return HPS_GPU_E_DTYPE_MISMATCH;
  }
  HPSG_CUDA(cudaSetDevice(ctx->device));
  auto c = new hps_gpu_cache_s;
  c->ctx = ctx;
  c->capacity = cfg->capacity;
  c->ways = ways;
  c->dim_io = cfg->dim;
  c->dim = padded_dim(cfg->dim);
  c->f16 = cfg->dtype == HPS_DTYPE_F16;
  if (const char* e = std::getenv("HPS_GPU_NO_SMALL_SORT")) c->no_small_sort = e[0] == '1';
  c->num_sets = cfg->capacity / ways;
  const uint64_t interval = cfg->aging_interval ? cfg->aging_interval : 10 * cfg->capacity;
  c->aging_period = std::max<uint64_t>(1, interval / c->num_sets);
  c->max_batch = cfg->max_batch;
  c->set_mod = hps::FastMod64(c->num_sets);
  c->set_bits = std::max(1, bits_for(c->num_sets));  // ids 0..num_sets (num_sets = invalid marker)
  const uint64_t cap = c->capacity, n = c->max_batch;
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dalloc(&c->d_keys, cap));
  A(dalloc(&c->d_ver, cap));
  A(dalloc(&c->d_touch, cap));
  A(dalloc(&c->d_freq, cap));
  A(dalloc(&c->d_set_acc, c->num_sets));
  A(dalloc(reinterpret_cast<uint8_t**>(&c->d_vec), cap * c->dim * (c->f16 ? 2 : 4)));
  A(dalloc(&c->d_state, 16));
  A(dalloc(&c->ws_set, n));
  A(dalloc(&c->ws_keys_b, n));
  A(dalloc(&c->ws_vals_a, n));
  A(dalloc(&c->ws_vals_b, n));
  A(dalloc(&c->ws_hit, n));
  A(dalloc(&c->ws_rank, n));
  A(dalloc(&c->ws_seg, n + 2));
  c->sort_words = sort_ws_words(n, (c->set_bits + 7) / 8);
  A(dalloc(&c->ws_sort, c->sort_words));
  A(dalloc(&c->ws_scan, scan_tiles(n) + 2));
  A(dalloc(&c->ws_counts, 8));
  A(dalloc(&c->ws_scan_multi, kScanRegions * (scan_tiles(n) + 2)));
  A(dalloc(&c->ws_der_set, n));
  A(dalloc(&c->ws_der_idx, n));
  A(dalloc(&c->ws_der_pos, n));
  A(dalloc(&c->ws_qmiss, n));
  {  // the counting grouping pays off when sets outnumber a batch (segments of ~1 access)
    const char* e = std::getenv("HPS_GPU_COUNT_GROUP");
    c->count_group = e ? std::atoi(e) == 1 : c->num_sets >= 8 * n;
    if (c->count_group) {
      A(dalloc(&c->ws_setcnt, c->num_sets + 1));
      A(dalloc(&c->ws_ticket, n));
      if (!st && cudaMemset(c->ws_setcnt, 0, (c->num_sets + 1) * sizeof(uint32_t)) != cudaSuccess) st = HPS_GPU_E_CUDA;
    }
  }
  A(dalloc(&c->ws_dcounts, 4));
  if (c->dim != c->dim_io) A(dalloc(&c->ws_io, n * c->dim));
  if (st) {
    hps_gpu_cache_destroy(c);
    return st;
  }
  cudaStream_t s = ctx->stream;
  HPSG_CUDA(cudaMemsetAsync(c->d_freq, 0, cap, s));
  HPSG_CUDA(cudaMemsetAsync(c->d_keys, 0, cap * 8, s));
  HPSG_CUDA(cudaMemsetAsync(c->d_ver, 0, cap * 8, s));
  HPSG_CUDA(cudaMemsetAsync(c->d_touch, 0, cap * 8, s));
  HPSG_CUDA(cudaMemsetAsync(c->d_set_acc, 0, c->num_sets * 8, s));
  HPSG_CUDA(cudaMemsetAsync(c->d_vec, 0, cap * c->dim * (c->f16 ? 2 : 4), s));
  HPSG_CUDA(cudaMemsetAsync(c->d_state, 0, 16 * 8, s));
  HPSG_CUDA(cudaMemsetAsync(c->ws_counts, 0, 8 * 8, s));
  HPSG_CUDA(cudaStreamSynchronize(s));
  *out = c;
  return HPS_GPU_OK;
}

int hps_gpu_cache_destroy(hps_gpu_cache c) {
  if (!c) return HPS_GPU_OK;
  void* ptrs[] = {c->d_keys,    c->d_ver,    c->d_touch,   c->d_freq, c->d_set_acc, c->d_vec,
                  c->d_state,   c->ws_set,   c->ws_keys_b, c->ws_vals_a, c->ws_vals_b, c->ws_hit,
                  c->ws_rank,   c->ws_seg,   c->ws_sort,   c->ws_scan, c->ws_counts, c->ws_io,
                  c->ws_der_set, c->ws_der_idx, c->ws_der_pos, c->ws_dcounts, c->ws_qmiss, c->ws_setcnt,
                  c->ws_ticket, c->ws_scan_multi};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete c;
  return HPS_GPU_OK;
}

// HPS_GPU_CACHE_PHASES=1 (debug): per-stage device times of each query, to stderr.
struct QueryPhases {
  bool on = false;
  cudaEvent_t ev[6] = {};
  int k = 0;
  explicit QueryPhases(cudaStream_t st) : st_(st) {
    const char* e = std::getenv("HPS_GPU_CACHE_PHASES");
    on = e && e[0] == '1';
    if (on)
      for (auto& x : ev) cudaEventCreate(&x);
  }
  void mark() {
    if (on && k < 6) cudaEventRecord(ev[k++], st_);
  }
  ~QueryPhases() {
    if (!on) return;
    cudaEventSynchronize(ev[k - 1]);
    std::fprintf(stderr, "# cache query phases (us):");
    for (int i = 1; i < k; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      std::fprintf(stderr, " %.1f", ms * 1000.f);
    }
    std::fprintf(stderr, "  [probe+split | gather | sort+segment | meta]\n");
    for (auto& x : ev) cudaEventDestroy(x);
  }
  cudaStream_t st_;
};

}  // extern "C"

// n: the key count, or (d_n != nullptr) its bound with the count on the device.
int hpsg::cache_query(hps_gpu_cache c, const uint64_t* keys, uint64_t n, const uint64_t* d_n, float* found_vecs,
                      uint32_t* found_idx, uint32_t* missing_idx, uint64_t* counts, bool scatter_found) {
  if (int s = check_cache(c)) return s;
  const bool distinct = c->query_distinct;  // (set by the read-through for this call only)
  c->query_distinct = false;
  if (!found_idx || !missing_idx || !counts) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n > c->max_batch) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = c->ctx->stream;
  if (n == 0) {
    HPSG_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(uint64_t), st));
    return HPS_GPU_OK;
  }
  if (!keys) return HPS_GPU_E_INVALID_ARGUMENT;
  QueryPhases ph(st);
  ph.mark();
  launch_k(true, k_probe, grid_for(n, 256, kNumSMs * 16), 256, 0, st, keys, n, c->set_mod, c->ways, c->d_keys, c->d_freq,
                                                          c->ws_set, c->ws_hit, c->d_state, c->ws_counts, d_n);
  SplitOp op{c->ws_hit, found_idx, missing_idx, counts, c->ws_counts, c->d_state + kStats, c->ws_qmiss};
  HPSG_CUDA(cache_scan(c, op, n));
  HPSG_CHECK_LAUNCH("cache probe/split");
  ph.mark();
  if (found_vecs) {
    const int lpr = lpr_for(c->dim);
    const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
#define HPSG_G(L)                                                                                                   \
  (c->f16 ? launch_k(true, k_gather<L, true>, grid, 256, 0, st, found_idx, c->ws_counts, c->ws_set, c->ws_hit, c->ways, c->d_vec, \
                                                     c->dim, found_vecs, scatter_found ? 1 : 0)                                              \
          : launch_k(true, k_gather<L, false>, grid, 256, 0, st, found_idx, c->ws_counts, c->ws_set, c->ws_hit, c->ways, c->d_vec,\
                                                      c->dim, found_vecs, scatter_found ? 1 : 0))
    switch (lpr) {
      case 32: HPSG_G(32); break;
      case 16: HPSG_G(16); break;
      case 8: HPSG_G(8); break;
      case 4: HPSG_G(4); break;
      case 2: HPSG_G(2); break;
      default: HPSG_G(1); break;
    }
#undef HPSG_G
    HPSG_CHECK_LAUNCH("cache gather");
  }
  ph.mark();
  const uint32_t* sets_sorted;
  const uint32_t* idx_sorted;
  if (int s = sort_and_segment(c, n, c->set_bits, &sets_sorted, &idx_sorted, distinct)) return s;
  c->q_sets = sets_sorted;
  c->q_idx = idx_sorted;
  ph.mark();
  if (c->ways <= 8) {
    auto* n_huge = reinterpret_cast<unsigned long long*>(c->ws_counts + 4);
    launch_k(true, k_query_meta_lanes, grid_for((n + 31) / 32 * 32, 256, kNumSMs * 16), 256, 0, st, 
        sets_sorted, idx_sorted, c->ws_seg, c->ws_counts, c->ws_hit, c->ways, c->aging_period, c->d_freq, c->d_touch,
        c->d_set_acc, c->d_state, c->ws_rank, n_huge);
    launch_k(true, k_query_meta_huge, kNumSMs, 256, 0, st, sets_sorted, idx_sorted, c->ws_seg, c->ws_rank,
                                               reinterpret_cast<const uint64_t*>(n_huge), c->ws_hit, c->ways,
                                               c->aging_period, c->d_freq, c->d_touch, c->d_set_acc, c->d_state);
  } else
    launch_k(true, k_query_meta, set_warps_grid(n), 256, 0, st, sets_sorted, idx_sorted, c->ws_seg, c->ws_counts, c->ws_hit,
                                                    c->ways, c->aging_period, c->d_freq, c->d_touch, c->d_set_acc,
                                                    c->d_state);
  HPSG_CHECK_LAUNCH("cache meta");
  ph.mark();
  return HPS_GPU_OK;
}

extern "C" {

int hps_gpu_cache_query(hps_gpu_cache c, const uint64_t* keys, uint64_t n, float* found_vecs, uint32_t* found_idx,
                        uint32_t* missing_idx, uint64_t* counts) {
  if (c && c->dim != c->dim_io && found_vecs && n && n <= c->max_batch) {  // padded rows: gather, then narrow
    int s = cache_query(c, keys, n, nullptr, c->ws_io, found_idx, missing_idx, counts);
    if (!s && rows_narrow(found_vecs, c->dim_io, c->ws_io, c->dim, n, c->ctx->stream) != cudaSuccess) s = HPS_GPU_E_CUDA;
    return s;
  }
  return cache_query(c, keys, n, nullptr, found_vecs, found_idx, missing_idx, counts);
}

// Padded rows: the caller's [n x dim_io] entries widened into the staging (zero padding).
static const float* widen_entries(hps_gpu_cache c, const float* vecs, uint64_t n, int* status) {
  *status = HPS_GPU_OK;
  if (!c || c->dim == c->dim_io || !vecs || n == 0 || n > c->max_batch) return vecs;
  if (rows_widen(c->ws_io, c->dim, vecs, c->dim_io, n, c->ctx->stream) != cudaSuccess) *status = HPS_GPU_E_CUDA;
  return c->ws_io;
}

static int entry_prep(hps_gpu_cache c, const uint64_t* keys, const float* vecs, uint64_t n,
                      const uint64_t* d_n = nullptr, const uint8_t* skip = nullptr, uint64_t* zero_out = nullptr) {
  cudaStream_t st = c->ctx->stream;
  const int lpr = lpr_for(c->dim);
  const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
  const uint32_t invalid = static_cast<uint32_t>(c->num_sets);
#define HPSG_P(L) launch_k(true, k_entry_prep<L>, grid, 256, 0, st, keys, vecs, n, c->dim, c->set_mod, invalid, c->ws_set, c->ws_hit, c->ctx->d_status, c->ws_counts, d_n, skip, c->f16 ? 1 : 0, zero_out)
  switch (lpr) {
    case 32: HPSG_P(32); break;
    case 16: HPSG_P(16); break;
    case 8: HPSG_P(8); break;
    case 4: HPSG_P(4); break;
    case 2: HPSG_P(2); break;
    default: HPSG_P(1); break;
  }
#undef HPSG_P
  HPSG_CHECK_LAUNCH("cache entry prep");
  return HPS_GPU_OK;
}

static int insert_impl(hps_gpu_cache c, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                       uint64_t n, const uint64_t* d_n, uint64_t* admitted_out, const uint8_t* skip = nullptr) {
  if (int s = check_cache(c)) return s;
  if (n > c->max_batch) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = c->ctx->stream;
  if (n == 0) {
    if (admitted_out) HPSG_CUDA(cudaMemsetAsync(admitted_out, 0, sizeof(uint64_t), st));
    return HPS_GPU_OK;
  }
  if (!keys || !vecs) return HPS_GPU_E_INVALID_ARGUMENT;
  if (int s = entry_prep(c, keys, vecs, n, d_n, skip, admitted_out)) return s;  // zeroes *admitted_out
  RankOp rop{c->ws_hit, c->ws_rank, c->ws_counts, c->d_state};
  HPSG_CUDA(cache_scan(c, rop, n));
  const uint32_t* sets_sorted;
  const uint32_t* idx_sorted;
  if (int s = sort_and_segment(c, n, bits_for(c->num_sets), &sets_sorted, &idx_sorted)) return s;
  if (c->ways <= 8)  // four sets per warp
    launch_k(true, (c->f16 ? k_insert_sets8<true> : k_insert_sets8<false>), grid_for((n + 3) / 4 * 32, 256, kNumSMs * 16),
             256, 0, st, sets_sorted, idx_sorted, c->ws_seg, c->ws_counts, keys, vecs, versions, c->ws_rank, c->ways,
             c->dim, c->aging_period, static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_touch,
             c->d_set_acc, c->d_vec, c->d_state, admitted_out, static_cast<const uint32_t*>(nullptr),
             static_cast<const uint8_t*>(nullptr));
  else
  launch_k(true, (c->f16 ? k_insert_sets<true> : k_insert_sets<false>), set_warps_grid(n), 256, 0, st, 
      sets_sorted, idx_sorted, c->ws_seg, c->ws_counts, keys, vecs, versions, c->ws_rank, c->ways, c->dim,
      c->aging_period, static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_touch, c->d_set_acc,
      c->d_vec, c->d_state, admitted_out);
  HPSG_CHECK_LAUNCH("cache insert");
  return HPS_GPU_OK;
}

}  // extern "C"

namespace hpsg {
void cache_mark_distinct_query(hps_gpu_cache c) {
  if (c) c->query_distinct = true;
}
// The read-through's scans (query split, grouping, segments, insert rank, derivation,
// segments) each take a region zeroed here by ONE memset; disarmed at the call's end.
int cache_arm_scans(hps_gpu_cache c, bool on, uint64_t n_max) {
  if (!c) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!on || scan_tiles(n_max) <= 1) {  // (single-tile scans need no zeroed words)
    c->scan_slot = -1;
    return HPS_GPU_OK;
  }
  HPSG_CUDA(cudaMemsetAsync(c->ws_scan_multi, 0, kScanRegions * (scan_tiles(c->max_batch) + 2) * sizeof(uint64_t),
                            c->ctx->stream));
  c->scan_slot = 0;
  return HPS_GPU_OK;
}
// The read-through's migration: insert its distinct misses (entries [0, *d_count) of keys/vecs,
// skip[] = absent from the lower tier) right after cache_query of the same call, reusing the
// query's set-sorted list (DeriveOp) instead of sorting the entries again. Same results as
// hps_gpu_cache_insert_count on those entries (bulk-load versions).
int cache_insert_after_query(hps_gpu_cache c, const uint64_t* keys, const float* vecs, uint64_t n_max,
                             const uint64_t* d_count, const uint8_t* skip, uint64_t* admitted_out,
                             const uint64_t* q_n, uint64_t q_n_max) {
  if (int s = check_cache(c)) return s;
  if (n_max > c->max_batch || !c->q_sets || !keys || !vecs || !d_count || !q_n)
    return HPS_GPU_E_INVALID_ARGUMENT;
  if (n_max == 0) return HPS_GPU_OK;
  cudaStream_t st = c->ctx->stream;
  {  // k_entry_prep: validity + the call's admitted count; its set ids go to scratch (the
     // query's sorted list may live in ws_set)
    const int lpr = lpr_for(c->dim);
    const int grid = grid_for(n_max * lpr, 256, kNumSMs * 16);
    const uint32_t invalid = static_cast<uint32_t>(c->num_sets);
#define HPSG_P(L) launch_k(true, k_entry_prep<L>, grid, 256, 0, st, keys, vecs, n_max, c->dim, c->set_mod, invalid, c->ws_der_pos, c->ws_hit, c->ctx->d_status, c->ws_counts, d_count, skip, c->f16 ? 1 : 0, admitted_out)
    switch (lpr) {
      case 32: HPSG_P(32); break;
      case 16: HPSG_P(16); break;
      case 8: HPSG_P(8); break;
      case 4: HPSG_P(4); break;
      case 2: HPSG_P(2); break;
      default: HPSG_P(1); break;
    }
#undef HPSG_P
    HPSG_CHECK_LAUNCH("cache entry prep (after query)");
  }
  RankOp rop{c->ws_hit, c->ws_rank, c->ws_counts, c->d_state};
  HPSG_CUDA(cache_scan(c, rop, n_max));
  if (c->ways <= 8) {  // the query's own segments, entries mapped inside the insert kernel
    launch_k(true, (c->f16 ? k_insert_sets8<true> : k_insert_sets8<false>),
             grid_for((q_n_max + 3) / 4 * 32, 256, kNumSMs * 16), 256, 0, st, c->q_sets, c->q_idx,
             static_cast<const uint32_t*>(c->ws_seg), static_cast<const uint64_t*>(c->ws_counts), keys, vecs,
             static_cast<const uint64_t*>(nullptr), static_cast<const uint32_t*>(c->ws_rank), c->ways, c->dim,
             c->aging_period, static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_touch,
             c->d_set_acc, c->d_vec, c->d_state, admitted_out, static_cast<const uint32_t*>(c->ws_qmiss),
             static_cast<const uint8_t*>(c->ws_hit));
    HPSG_CHECK_LAUNCH("cache insert (query segments)");
    return HPS_GPU_OK;
  }
  DeriveOp dop{c->q_sets, c->q_idx, q_n, c->ws_qmiss, c->ws_hit, c->ws_der_set, c->ws_der_idx, c->ws_dcounts};
  HPSG_CUDA(cache_scan(c, dop, q_n_max));
  SetSegOp sop{c->ws_der_set, c->ws_seg, c->ws_dcounts};
  HPSG_CUDA(cache_scan(c, sop, n_max));
  HPSG_CHECK_LAUNCH("cache derived set grouping");
  if (c->ways <= 8)
    launch_k(true, (c->f16 ? k_insert_sets8<true> : k_insert_sets8<false>), grid_for((n_max + 3) / 4 * 32, 256, kNumSMs * 16),
             256, 0, st, static_cast<const uint32_t*>(c->ws_der_set), static_cast<const uint32_t*>(c->ws_der_idx),
             static_cast<const uint32_t*>(c->ws_seg), static_cast<const uint64_t*>(c->ws_dcounts), keys, vecs,
             static_cast<const uint64_t*>(nullptr), static_cast<const uint32_t*>(c->ws_rank), c->ways, c->dim,
             c->aging_period, static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_touch,
             c->d_set_acc, c->d_vec, c->d_state, admitted_out, static_cast<const uint32_t*>(nullptr),
             static_cast<const uint8_t*>(nullptr));
  else
    launch_k(true, (c->f16 ? k_insert_sets<true> : k_insert_sets<false>), set_warps_grid(n_max), 256, 0, st,
             static_cast<const uint32_t*>(c->ws_der_set), static_cast<const uint32_t*>(c->ws_der_idx),
             static_cast<const uint32_t*>(c->ws_seg), static_cast<const uint64_t*>(c->ws_dcounts), keys, vecs,
             static_cast<const uint64_t*>(nullptr), static_cast<const uint32_t*>(c->ws_rank), c->ways, c->dim,
             c->aging_period, static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_touch,
             c->d_set_acc, c->d_vec, c->d_state, admitted_out);
  HPSG_CHECK_LAUNCH("cache insert (after query)");
  return HPS_GPU_OK;
}
}  // namespace hpsg

extern "C" {

int hps_gpu_cache_insert(hps_gpu_cache c, const uint64_t* keys, const float* vecs, const uint64_t* versions, uint64_t n,
                         uint64_t* admitted_out) {
  if (n && !versions) return HPS_GPU_E_INVALID_ARGUMENT;
  int s = HPS_GPU_OK;
  vecs = widen_entries(c, vecs, n, &s);
  return s ? s : insert_impl(c, keys, vecs, versions, n, nullptr, admitted_out);
}

int hps_gpu_cache_insert_count(hps_gpu_cache c, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                               uint64_t n_max, const uint64_t* d_count, const uint8_t* skip, uint64_t* admitted_out) {
  if (!d_count) return HPS_GPU_E_INVALID_ARGUMENT;
  int s = HPS_GPU_OK;
  vecs = widen_entries(c, vecs, n_max, &s);
  return s ? s : insert_impl(c, keys, vecs, versions, n_max, d_count, admitted_out, skip);
}

int hps_gpu_cache_refresh(hps_gpu_cache c, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                          uint64_t n, uint64_t* replaced_out) {
  if (int s = check_cache(c)) return s;
  if (n > c->max_batch) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = c->ctx->stream;
  if (n == 0) {
    if (replaced_out) HPSG_CUDA(cudaMemsetAsync(replaced_out, 0, sizeof(uint64_t), st));
    return HPS_GPU_OK;
  }
  if (!keys || !vecs || !versions) return HPS_GPU_E_INVALID_ARGUMENT;
  {
    int s = HPS_GPU_OK;
    vecs = widen_entries(c, vecs, n, &s);
    if (s) return s;
  }
  if (int s = entry_prep(c, keys, vecs, n, nullptr, nullptr, replaced_out)) return s;  // zeroes *replaced_out
  const uint32_t* sets_sorted;
  const uint32_t* idx_sorted;
  if (int s = sort_and_segment(c, n, bits_for(c->num_sets), &sets_sorted, &idx_sorted)) return s;
  launch_k(true, (c->f16 ? k_refresh_sets<true> : k_refresh_sets<false>), set_warps_grid(n), 256, 0, st, 
      sets_sorted, idx_sorted, c->ws_seg, c->ws_counts, keys, vecs, versions, c->ways, c->dim,
      static_cast<uint32_t>(c->num_sets), c->d_keys, c->d_ver, c->d_freq, c->d_vec, c->d_state, replaced_out);
  HPSG_CHECK_LAUNCH("cache refresh");
  return HPS_GPU_OK;
}

}  // extern "C"

namespace hpsg {
int cache_info(hps_gpu_cache c, hps_gpu_ctx* ctx, uint32_t* dim) {
  if (int s = check_cache(c)) return s;
  *ctx = c->ctx;
  *dim = c->dim_io;  // (the caller's dim; rows are stored padded when it is not a multiple of 4)
  return HPS_GPU_OK;
}
uint64_t cache_max_batch(hps_gpu_cache c) { return c ? c->max_batch : 0; }
}  // namespace hpsg

extern "C" {

int hps_gpu_cache_stats(hps_gpu_cache c, hps_cache_stats* out) {
  if (int s = check_cache(c)) return s;
  if (!out) return HPS_GPU_E_INVALID_ARGUMENT;
  uint64_t h[7];
  HPSG_CUDA(cudaMemcpyAsync(h, c->d_state + kStats, sizeof(h), cudaMemcpyDeviceToHost, c->ctx->stream));
  HPSG_CUDA(cudaStreamSynchronize(c->ctx->stream));
  out->queries = h[sQueries];
  out->hits = h[sHits];
  out->misses = h[sMisses];
  out->insertions = h[sInsertions];
  out->admissions_rejected = h[sRejected];
  out->refresh_replacements = h[sRefresh];
  out->evictions = h[sEvictions];
  return HPS_GPU_OK;
}

int hps_gpu_cache_reset_stats(hps_gpu_cache c) {
  if (int s = check_cache(c)) return s;
  HPSG_CUDA(cudaMemsetAsync(c->d_state + kStats, 0, 7 * sizeof(uint64_t), c->ctx->stream));
  return HPS_GPU_OK;
}

int hps_gpu_cache_debug_export(hps_gpu_cache c, uint64_t* keys, uint64_t* versions, uint8_t* freq,
                               uint64_t* last_touch, uint64_t* set_access, void* vecs) {
  if (int s = check_cache(c)) return s;
  cudaStream_t st = c->ctx->stream;
  const uint64_t cap = c->capacity;
  if (keys) HPSG_CUDA(cudaMemcpyAsync(keys, c->d_keys, cap * 8, cudaMemcpyDeviceToDevice, st));
  if (versions) HPSG_CUDA(cudaMemcpyAsync(versions, c->d_ver, cap * 8, cudaMemcpyDeviceToDevice, st));
  if (freq) HPSG_CUDA(cudaMemcpyAsync(freq, c->d_freq, cap, cudaMemcpyDeviceToDevice, st));
  if (last_touch) HPSG_CUDA(cudaMemcpyAsync(last_touch, c->d_touch, cap * 8, cudaMemcpyDeviceToDevice, st));
  if (set_access) HPSG_CUDA(cudaMemcpyAsync(set_access, c->d_set_acc, c->num_sets * 8, cudaMemcpyDeviceToDevice, st));
  if (vecs)
    HPSG_CUDA(rows_narrow(vecs, c->dim_io, c->d_vec, c->dim, cap, st, c->f16 ? 2 : 4));
  return HPS_GPU_OK;
}

int hps_gpu_cache_size(hps_gpu_cache c, uint64_t* n_host) {
  if (int s = check_cache(c)) return s;
  if (!n_host) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = c->ctx->stream;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(c->d_state + kScratch);
  HPSG_CUDA(cudaMemsetAsync(d, 0, 8, st));
  k_count_resident<<<grid_for(c->capacity, 256, kNumSMs * 8), 256, 0, st>>>(c->d_freq, c->capacity, d);
  HPSG_CHECK_LAUNCH("k_count_resident");
  HPSG_CUDA(cudaMemcpyAsync(n_host, d, 8, cudaMemcpyDeviceToHost, st));
  HPSG_CUDA(cudaStreamSynchronize(st));
  return HPS_GPU_OK;
}

}  // extern "C"
