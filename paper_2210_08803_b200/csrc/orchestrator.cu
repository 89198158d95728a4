// orchestrator.cu — the orchestrator's batch lookup on the GPU:
// the HPS cache (L1) in front of a GPU-resident table (the lower tier), duplicate keys
// served from ONE tier probe per distinct key.
//
//   K14a  dedup      distinct keys in order of first occurrence + the inverse map
//                    (one CTA in shared memory up to kSmallDedup keys; above it an
//                    open-addressing claim table of u32 owners in HBM/L2 and a first-occurrence
//                    scan; the inverse is resolved by the expand)
//   K6    cache query of the distinct keys (count on the device)
//   K14b  read-through: hits from the cache, misses from the table (default vector when
//                    absent), the source tier of each distinct key
//   K7    distinct misses present in the table are inserted into the cache (once each)
//   K14c  expand: out[i] = row of inverse[i], source counts per input key
//
// The whole lookup is asynchronous, never allocates and is capturable into a CUDA graph.
#include <cstdlib>

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "primitives.cuh"
#include "table_internal.cuh"

using namespace hpsg;

namespace hpsg {
int cache_query(hps_gpu_cache c, const uint64_t* keys, uint64_t n, const uint64_t* d_n, float* found_vecs,
                uint32_t* found_idx, uint32_t* missing_idx, uint64_t* counts, bool scatter_found);
int cache_info(hps_gpu_cache c, hps_gpu_ctx* ctx, uint32_t* dim);
uint64_t cache_max_batch(hps_gpu_cache c);
void cache_mark_distinct_query(hps_gpu_cache c);
int cache_arm_scans(hps_gpu_cache c, bool on, uint64_t n_max);
int cache_insert_after_query(hps_gpu_cache c, const uint64_t* keys, const float* vecs, uint64_t n_max,
                             const uint64_t* d_count, const uint8_t* skip, uint64_t* admitted_out,
                             const uint64_t* q_n, uint64_t q_n_max);
}  // namespace hpsg

struct hps_gpu_readthrough_s {
  hps_gpu_cache cache = nullptr;
  hps_gpu_table tbl = nullptr;
  uint32_t table = 0, dim = 0;
  uint64_t max_batch = 0, claim_cap = 0;
  hps_gpu_ctx ctx = nullptr;
  // workspaces (sized at create)
  uint32_t* claim = nullptr;     // [claim_cap] owner (min input position) per slot, 0xffffffff = empty
  uint32_t* slot_of = nullptr;   // [max_batch] claim slot of each input key
  uint32_t* uid_at = nullptr;    // [max_batch] distinct id, valid at first occurrences
  uint32_t* inverse = nullptr;   // [max_batch]
  uint64_t* ukeys = nullptr;     // [max_batch] distinct keys
  uint64_t* counts = nullptr;    // [0] U  [2..3] cache query counts (found, missing)  [4] admitted
  uint64_t* scan = nullptr;
  float* found = nullptr;        // [max_batch x dim]
  uint32_t* found_idx = nullptr;
  uint32_t* missing_idx = nullptr;
  float* urows = nullptr;        // [max_batch x dim] row of each distinct key
  uint64_t* miss_keys = nullptr;
  float* miss_vecs = nullptr;
  uint8_t* miss_absent = nullptr;
  uint8_t* src = nullptr;        // [max_batch] source tier of each distinct key
};

namespace {

constexpr uint32_t kEmptyOwner = 0xffffffffu;
constexpr int kSmallDedupThreads = 512;
constexpr int kSmallDedupIPT = 4;
constexpr uint64_t kSmallDedup = uint64_t(kSmallDedupThreads) * kSmallDedupIPT;  // 2048 keys
constexpr uint32_t kSmallClaim = 2 * kSmallDedup;                                 // power of two

// Small batches (the latency end of config 4's sweep): the whole dedup in one CTA — keys
// and the claim table in shared memory, a block scan over the first-occurrence flags.
__global__ void __launch_bounds__(kSmallDedupThreads) k_dedup_small(const uint64_t* __restrict__ keys, uint32_t n,
                                                                    uint64_t* __restrict__ ukeys,
                                                                    uint32_t* __restrict__ inverse,
                                                                    uint64_t* __restrict__ counts,
                                                                    uint64_t* __restrict__ source_counts) {
  pdl_wait();
  pdl_launch_dependents();
  using Scan = cub::BlockScan<uint32_t, kSmallDedupThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t s_key[kSmallDedup];
  __shared__ uint32_t s_claim[kSmallClaim];
  __shared__ uint32_t s_uid[kSmallDedup];
  for (uint32_t e = threadIdx.x; e < kSmallClaim; e += blockDim.x) s_claim[e] = kEmptyOwner;
  uint32_t slot[kSmallDedupIPT];
  uint64_t k[kSmallDedupIPT];
#pragma unroll
  for (int q = 0; q < kSmallDedupIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallDedupIPT + q;
    k[q] = i < n ? keys[i] : 0;
    if (i < n) s_key[i] = k[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSmallDedupIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallDedupIPT + q;
    slot[q] = 0;
    if (i >= n) continue;
    uint32_t h = static_cast<uint32_t>(hps::key_hash(k[q])) & (kSmallClaim - 1);
    while (true) {
      uint32_t o = s_claim[h];
      if (o == kEmptyOwner) {
        o = atomicCAS(&s_claim[h], kEmptyOwner, i);
        if (o == kEmptyOwner) break;
      }
      if (s_key[o] == k[q]) {  // same key: the earliest position owns the slot
        atomicMin(&s_claim[h], i);
        break;
      }
      h = (h + 1) & (kSmallClaim - 1);
    }
    slot[q] = h;
  }
  __syncthreads();
  uint32_t first[kSmallDedupIPT], excl[kSmallDedupIPT], total = 0;
#pragma unroll
  for (int q = 0; q < kSmallDedupIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallDedupIPT + q;
    first[q] = (i < n && s_claim[slot[q]] == i) ? 1u : 0u;
  }
  Scan(tmp).ExclusiveSum(first, excl, total);
#pragma unroll
  for (int q = 0; q < kSmallDedupIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallDedupIPT + q;
    if (first[q]) {
      ukeys[excl[q]] = k[q];
      s_uid[i] = excl[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSmallDedupIPT; ++q) {
    const uint32_t i = threadIdx.x * kSmallDedupIPT + q;
    if (i < n) inverse[i] = s_uid[s_claim[slot[q]]];
  }
  if (threadIdx.x == 0) counts[0] = total;
  if (source_counts && threadIdx.x < 4) source_counts[threadIdx.x] = 0;
}

// Large batches, pass 1: claim. Slot = key_hash & (cap-1), linear probing; the owner of a
// slot is the minimum input position holding its key (CAS from empty, atomicMin among
// equal keys — the owner always names a position with that key, so the key compare reads
// keys[owner]).
__global__ void __launch_bounds__(256) k_dedup_claim(const uint64_t* __restrict__ keys, uint64_t n,
                                                     uint32_t* __restrict__ claim, uint64_t mask,
                                                     uint32_t* __restrict__ slot_of, uint64_t* source_counts,
                                                     uint64_t* scan_zero, uint32_t scan_words) {
  pdl_wait();
  pdl_launch_dependents();
  if (source_counts && blockIdx.x == 0 && threadIdx.x < 4) source_counts[threadIdx.x] = 0;
  // the first-occurrence scan's look-back words, zeroed here (it runs next): no memset node
  if (blockIdx.x == 0)
    for (uint32_t w = threadIdx.x; w < scan_words; w += blockDim.x) scan_zero[w] = 0;
  // (whole warps iterate together: the match below needs every lane)
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i0 = blockIdx.x * uint64_t(blockDim.x); i0 < n; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < n;
    const uint64_t k = valid ? keys[i] : 0;
    // a Zipf-hot key repeats within a warp: only its first lane (the smallest position)
    // claims; the others take its slot
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? k : ~k) & __ballot_sync(0xffffffffu, valid);
    const int leader = peers ? __ffs(peers) - 1 : 0;
    uint64_t h = hps::key_hash(k) & mask;
    if (valid && static_cast<int>(lane_id()) == leader) {
      while (true) {
        uint32_t o = claim[h];
        if (o == kEmptyOwner) {
          o = atomicCAS(&claim[h], kEmptyOwner, static_cast<uint32_t>(i));
          if (o == kEmptyOwner) break;
        }
        if (keys[o] == k) {
          if (o > i) atomicMin(&claim[h], static_cast<uint32_t>(i));  // (owners only decrease)
          break;
        }
        h = (h + 1) & mask;
      }
    }
    h = __shfl_sync(0xffffffffu, h, leader);
    if (valid) slot_of[i] = static_cast<uint32_t>(h);
  }
}

// pass 2: first occurrences in input order -> distinct ids (decoupled look-back scan)
struct FirstOp {
  const uint64_t* keys;
  const uint32_t* claim;
  const uint32_t* slot_of;
  uint64_t n;
  uint64_t* ukeys;
  uint32_t* uid_at;
  uint64_t* counts;
  __device__ uint64_t size() const { return n; }
  __device__ uint32_t count(uint64_t i) const { return claim[slot_of[i]] == static_cast<uint32_t>(i) ? 1u : 0u; }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    if (c) {
      ukeys[excl] = keys[i];
      uid_at[i] = static_cast<uint32_t>(excl);
    }
  }
  __device__ void total(uint64_t t) const { counts[0] = t; }
};

// pass 3, the inverse map inverse[i] = uid_at[claim[slot_of[i]]], is resolved inside k_expand
// (the claim table's last reader; a memset node after it empties the table for the next call).

// K14c: out[i] = urows[inverse[i]] (LPR lanes per row, 128-bit), per-key source counts
// (warp-aggregated atomics into source_counts[0..3]).
template <int LPR>
// (claim != nullptr: the large-batch dedup's inverse is resolved here — uid_at[claim[slot_of[i]]]
// — instead of by a separate pass; the claim table is reset after this kernel)
__global__ void __launch_bounds__(256) k_expand(const float* __restrict__ urows, const uint32_t* __restrict__ inverse,
                                                const uint8_t* __restrict__ src, uint64_t n, uint32_t dim,
                                                float* __restrict__ out, unsigned long long* source_counts,
                                                const uint32_t* __restrict__ claim, const uint32_t* __restrict__ slot_of,
                                                const uint32_t* __restrict__ uid_at) {
  pdl_wait();
  pdl_launch_dependents();
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint32_t c0 = 0, c1 = 0, c3 = 0;
  // a warp takes 32 * G consecutive outputs: their distinct ids in one coalesced load (lane l
  // holds ids l, l + 32, ...), then the rows stream 4 per group in flight
  constexpr int R = 4;
  for (uint64_t i0 = warp * 32 * G; i0 < n; i0 += n_warps * 32 * G) {
    uint32_t my_u[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const uint64_t i = i0 + q * 32 + lane;
      my_u[q] = i < n ? (claim ? uid_at[claim[slot_of[i]]] : inverse[i]) : 0u;
      if (i < n && source_counts) {
        const uint8_t sv = src[my_u[q]];
        c0 += sv == 0;
        c1 += sv == 1;
        c3 += sv == 3;
      }
    }
    for (uint32_t r0 = 0; r0 < 32 * G; r0 += R * G) {  // output r0 + r * G + grp
      float4 x[R];
      uint64_t dst[R];
      bool ok[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t o = r0 + r * G + grp;
        // (o / 32 is the same for every lane: G divides 32) — select it without local memory
        const uint32_t q = o / 32;
        uint32_t mine = my_u[0];
#pragma unroll
        for (int qq = 1; qq < G; ++qq) mine = qq == static_cast<int>(q) ? my_u[qq] : mine;
        const uint32_t u = __shfl_sync(0xffffffffu, mine, o % 32);
        const uint64_t i = i0 + o;
        ok[r] = i < n;
        dst[r] = i;
        x[r] = (ok[r] && gl < nvec) ? reinterpret_cast<const float4*>(urows + uint64_t(u) * dim)[gl]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok[r])
          for (uint32_t v = gl + LPR; v < nvec; v += LPR)  // rows wider than one pass of the group
            reinterpret_cast<float4*>(out + i * dim)[v] = reinterpret_cast<const float4*>(urows + uint64_t(u) * dim)[v];
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ok[r] && gl < nvec) __stcs(reinterpret_cast<float4*>(out + dst[r] * dim) + gl, x[r]);  // streamed out
    }
  }
  if (source_counts) {  // per-CTA sums first: one global atomic per counter per CTA
    __shared__ unsigned long long s_c[3];
    if (threadIdx.x < 3) s_c[threadIdx.x] = 0ull;
    __syncthreads();
    c0 = warp_sum(c0);
    c1 = warp_sum(c1);
    c3 = warp_sum(c3);
    if (lane == 0) {
      if (c0) atomicAdd(&s_c[0], static_cast<unsigned long long>(c0));
      if (c1) atomicAdd(&s_c[1], static_cast<unsigned long long>(c1));
      if (c3) atomicAdd(&s_c[2], static_cast<unsigned long long>(c3));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_c[0]) atomicAdd(&source_counts[0], s_c[0]);
      if (s_c[1]) atomicAdd(&source_counts[1], s_c[1]);
      if (s_c[2]) atomicAdd(&source_counts[3], s_c[2]);
    }
  }
}

uint64_t claim_cap_for(uint64_t n) {
  uint64_t c = 1024;
  while (c < 2 * n) c <<= 1;
  return c;
}

int lpr_for(uint32_t dim) {
  const uint32_t nvec = dim / 4;
  return nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
}

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    set_last_error("readthrough: cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}

}  // namespace

extern "C" {

int hps_gpu_readthrough_create(hps_gpu_cache cache, hps_gpu_table tbl, uint32_t table, uint64_t max_batch,
                               hps_gpu_readthrough* out) {
  if (!cache || !tbl || !out || max_batch == 0 || max_batch >= (1ull << 31)) return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  hps_gpu_ctx ctx = nullptr;
  uint32_t cdim = 0;
  if (int s = cache_info(cache, &ctx, &cdim)) return s;
  if (table >= tbl->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (cdim != tbl->dim_io) {
    set_last_error("readthrough: cache dim != table dim");
    return HPS_GPU_E_DIM_MISMATCH;
  }
  if (cdim % 4 != 0) {
    set_last_error("readthrough: needs dim % 4 == 0 (padded rows are not served by the orchestrator)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (ctx != tbl->ctx) {
    set_last_error("readthrough: cache and table must share one context");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (max_batch > cache_max_batch(cache)) {
    set_last_error("readthrough: max_batch exceeds the cache's max_batch");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  HPSG_CUDA(cudaSetDevice(ctx->device));
  auto* r = new hps_gpu_readthrough_s;
  r->cache = cache;
  r->tbl = tbl;
  r->table = table;
  r->dim = cdim;
  r->ctx = ctx;
  r->max_batch = max_batch;
  r->claim_cap = claim_cap_for(max_batch);
  const uint64_t n = max_batch, D = cdim;
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dalloc(&r->claim, r->claim_cap));
  A(dalloc(&r->slot_of, n));
  A(dalloc(&r->uid_at, n));
  A(dalloc(&r->inverse, n));
  A(dalloc(&r->ukeys, n));
  A(dalloc(&r->counts, 8));
  A(dalloc(&r->scan, scan_tiles(n) + 2));
  A(dalloc(&r->found, n * D));
  A(dalloc(&r->found_idx, n));
  A(dalloc(&r->missing_idx, n));
  A(dalloc(&r->urows, n * D));
  A(dalloc(&r->miss_keys, n));
  A(dalloc(&r->miss_vecs, n * D));
  A(dalloc(&r->miss_absent, n));
  A(dalloc(&r->src, n));
  if (st) {
    hps_gpu_readthrough_destroy(r);
    return st;
  }
  HPSG_CUDA(cudaMemsetAsync(r->claim, 0xff, r->claim_cap * sizeof(uint32_t), ctx->stream));
  HPSG_CUDA(cudaMemsetAsync(r->counts, 0, 8 * sizeof(uint64_t), ctx->stream));
  HPSG_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = r;
  return HPS_GPU_OK;
}

int hps_gpu_readthrough_destroy(hps_gpu_readthrough r) {
  if (!r) return HPS_GPU_OK;
  void* ptrs[] = {r->claim, r->slot_of, r->uid_at,    r->inverse,   r->ukeys,     r->counts,      r->scan, r->found,
                  r->found_idx, r->missing_idx, r->urows, r->miss_keys, r->miss_vecs, r->miss_absent, r->src};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete r;
  return HPS_GPU_OK;
}

int hps_gpu_readthrough_lookup(hps_gpu_readthrough r, const uint64_t* keys, uint64_t n, float* out,
                               uint64_t* source_counts_out, uint64_t* n_unique_out) {
  if (!r) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n > r->max_batch) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = r->ctx->stream;
  if (n == 0) {
    if (source_counts_out) HPSG_CUDA(cudaMemsetAsync(source_counts_out, 0, 4 * sizeof(uint64_t), st));
    if (n_unique_out) HPSG_CUDA(cudaMemsetAsync(n_unique_out, 0, sizeof(uint64_t), st));
    return HPS_GPU_OK;
  }
  if (!keys || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  const bool pdl = r->ctx->pdl;
  // K14a: distinct keys, first-occurrence order
  if (n <= kSmallDedup) {
    HPSG_CUDA(launch_k(pdl, k_dedup_small, 1, kSmallDedupThreads, 0, st, keys, static_cast<uint32_t>(n), r->ukeys,
                       r->inverse, r->counts, source_counts_out));
  } else {
    const uint64_t cap = claim_cap_for(n);
    const uint64_t tiles = scan_tiles(n);  // (> 1: n > kSmallDedup)
    HPSG_CUDA(launch_k(pdl, k_dedup_claim, grid_for(n, 256, kNumSMs * 8), 256, 0, st, keys, n, r->claim, cap - 1,
                       r->slot_of, source_counts_out, r->scan, static_cast<uint32_t>(tiles + 1)));
    FirstOp op{keys, r->claim, r->slot_of, n, r->ukeys, r->uid_at, r->counts};
    k_scan<FirstOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, r->scan,
                                                                       reinterpret_cast<uint32_t*>(r->scan + tiles));
    // (the inverse map is resolved by k_expand, the claim table's last reader)
  }
  const bool fused_inverse = n > kSmallDedup;
  HPSG_CHECK_LAUNCH("readthrough dedup");
  if (n_unique_out) HPSG_CUDA(cudaMemcpyAsync(n_unique_out, r->counts, 8, cudaMemcpyDeviceToDevice, st));
  // K6 on the distinct keys (one access per distinct key: SPEC.md:340)
  cache_mark_distinct_query(r->cache);  // its keys are distinct: counting set grouping allowed
  if (int s = cache_arm_scans(r->cache, true, n)) return s;
  struct Disarm {  // every exit of this call (errors included) disarms the regions
    hps_gpu_cache c;
    ~Disarm() { cache_arm_scans(c, false, 0); }
  } disarm{r->cache};
  // (the hits' rows go straight to urows[distinct id]: no compacted copy to move again)
  if (int s = cache_query(r->cache, r->ukeys, n, r->counts, r->urows, r->found_idx, r->missing_idx, r->counts + 2,
                          /*scatter_found=*/true))
    return s;
  // K14b: table rows / default vector per distinct miss (hits already in place), misses listed
  if (int s = table_read_through(r->tbl, r->table, r->ukeys, nullptr, r->found_idx, r->missing_idx, r->counts + 2, n,
                                 r->urows, r->miss_keys, r->miss_vecs, r->miss_absent, r->src, /*hits_in_place=*/true))
    return s;
  // K7: migrate the distinct misses present in the table (absent keys are never cached),
  // grouped by set from the query's own sorted access list (no second sort;
  // HPS_GPU_RT_SORT=1 sorts them again: A/B)
  static const bool resort = [] {
    const char* e = std::getenv("HPS_GPU_RT_SORT");
    return e && std::atoi(e) == 1;
  }();
  if (resort) {
    if (int s = hps_gpu_cache_insert_count(r->cache, r->miss_keys, r->miss_vecs, nullptr, n, r->counts + 3,
                                           r->miss_absent, r->counts + 4))
      return s;
  } else if (int s = cache_insert_after_query(r->cache, r->miss_keys, r->miss_vecs, n, r->counts + 3, r->miss_absent,
                                              r->counts + 4, r->counts, n)) {
    return s;
  }
  cache_arm_scans(r->cache, false, 0);  // (the guard repeats it harmlessly)
  // K14c: rows back in input order
  const int lpr = lpr_for(r->dim);
  const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
  auto* sc = reinterpret_cast<unsigned long long*>(source_counts_out);
  const uint32_t* e_claim = fused_inverse ? r->claim : nullptr;
#define HPSG_E(L) launch_k(pdl, k_expand<L>, grid, 256, 0, st, static_cast<const float*>(r->urows), \
                           static_cast<const uint32_t*>(r->inverse), static_cast<const uint8_t*>(r->src), n, r->dim, out, sc, \
                           e_claim, static_cast<const uint32_t*>(r->slot_of), static_cast<const uint32_t*>(r->uid_at))
  cudaError_t e;
  switch (lpr) {
    case 32: e = HPSG_E(32); break;
    case 16: e = HPSG_E(16); break;
    case 8: e = HPSG_E(8); break;
    case 4: e = HPSG_E(4); break;
    case 2: e = HPSG_E(2); break;
    default: e = HPSG_E(1); break;
  }
#undef HPSG_E
  HPSG_CUDA(e);
  HPSG_CHECK_LAUNCH("readthrough expand");
  if (fused_inverse)  // the claim table empty again for the next call (k_expand read it last)
    HPSG_CUDA(cudaMemsetAsync(r->claim, 0xff, claim_cap_for(n) * sizeof(uint32_t), st));
  return HPS_GPU_OK;
}

}  // extern "C"
