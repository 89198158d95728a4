// primitives.cuh — device-wide scan and stable radix sort, hand-written for sm_100a.
//
// Both are single-pass-per-digit "decoupled look-back" designs: tiles take a ticket
// from an atomic counter (so every tile a block waits on is already resident), publish
// their local aggregate at once, then resolve their exclusive prefix by looking back
// over predecessors' published words. All sizes are read from DEVICE memory so the
// whole backward pipeline is capturable in a CUDA graph with no host round trip.
#pragma once

#include "common.cuh"

namespace hpsg {

// ---------------------------------------------------------------------------------
// volatile 64/32-bit publish/observe for look-back words
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_vol64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_vol32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (static_cast<int>(lane_id()) >= o) v += t;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one value per thread (BLOCK <= 1024). Returns the
// exclusive prefix; *total receives the block sum. `scratch` holds >= 32 T.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* scratch, T* total) {
  constexpr int NW = BLOCK / 32;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  T inc = warp_incl_scan(v);
  if (l == 31) scratch[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = l < NW ? scratch[l] : T(0);
    T si = warp_incl_scan(s);
    if (l < NW) scratch[l] = si - s;
    if (l == NW - 1) scratch[NW] = si;
  }
  __syncthreads();
  T r = inc - v + scratch[w];
  *total = scratch[NW];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------
// Decoupled look-back exclusive scan over u32 counts with u64 prefixes.
//   Op::size()                       -> number of items (device-side)
//   Op::count(i)                     -> u32 count of item i
//   Op::emit(i, excl, count)         -> consume the prefix
//   Op::total(sum)                   -> called once by the last tile
// Workspace: tile status words (u64, zeroed) + one ticket counter (u32, zeroed).
// ---------------------------------------------------------------------------------
constexpr uint64_t kScanAgg = 1ull << 62;
constexpr uint64_t kScanInc = 2ull << 62;
constexpr uint64_t kScanVal = kScanAgg - 1;

constexpr int kScanBlock = 256;
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanBlock * kScanIPT;

template <class Op>
__global__ void __launch_bounds__(kScanBlock) k_scan(Op op, uint64_t* status, uint32_t* ticket) {
  __shared__ uint64_t s_scratch[33];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_tile;
  pdl_wait();
  pdl_launch_dependents();
  trace_begin(TraceOf<Op>::id);
  const uint64_t n = op.size();
  const uint64_t n_tiles = (n + kScanTile - 1) / kScanTile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  if (n_tiles == 0) {  // empty input: still publish the (zero) total
    if (tile == 0 && threadIdx.x == 0) op.total(0);
    return;
  }
  if (tile >= n_tiles) return;
  const uint64_t base = tile * kScanTile + uint64_t(threadIdx.x) * kScanIPT;
  uint64_t c[kScanIPT];  // counts may be packed (several u32 fields summed at once)
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    c[k] = (base + k < n) ? static_cast<uint64_t>(op.count(base + k)) : 0ull;
    sum += c[k];
  }
  uint64_t agg;
  uint64_t excl = block_excl_scan<kScanBlock>(sum, s_scratch, &agg);
  if (threadIdx.x < 32) {
    uint64_t prefix = 0;
    if (tile == 0) {
      if (threadIdx.x == 0) st_vol64(&status[0], kScanInc | agg);
    } else {
      if (threadIdx.x == 0) st_vol64(&status[tile], kScanAgg | agg);
      int64_t p = static_cast<int64_t>(tile) - 1;
      while (true) {
        const int64_t idx = p - static_cast<int64_t>(threadIdx.x);
        uint64_t s = kScanInc;  // beyond tile 0: acts as an inclusive zero
        if (idx >= 0) {
          do { s = ld_vol64(&status[idx]); } while ((s & ~kScanVal) == 0);
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (s & kScanInc) != 0);
        const int first = inc ? __ffs(inc) - 1 : 32;
        uint64_t v = (static_cast<int>(threadIdx.x) <= first && idx >= 0) ? (s & kScanVal) : 0;
        prefix += warp_sum(v);
        if (inc) break;
        p -= 32;
      }
      if (threadIdx.x == 0) st_vol64(&status[tile], kScanInc | (prefix + agg));
    }
    if (threadIdx.x == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint64_t run = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    if (base + k < n) op.emit(base + k, run, c[k]);
    run += c[k];
  }
  if (tile == n_tiles - 1 && threadIdx.x == kScanBlock - 1) op.total(s_prefix + agg);
  trace_end(TraceOf<Op>::id);
}

inline uint64_t scan_tiles(uint64_t n_max) { return (n_max + kScanTile - 1) / kScanTile; }

// The same scan when the input fits ONE tile (n_max <= kScanTile, known on the host): no
// tile ticket and no look-back status, so no zeroing memset before it (small batches are
// bound by the nodes of their chain, not by bytes).
template <class Op>
__global__ void __launch_bounds__(kScanBlock) k_scan_one(Op op) {
  __shared__ uint64_t s_scratch[33];
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t n = op.size();
  const uint64_t base = uint64_t(threadIdx.x) * kScanIPT;
  uint64_t c[kScanIPT];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    c[k] = (base + k < n) ? static_cast<uint64_t>(op.count(base + k)) : 0ull;
    sum += c[k];
  }
  uint64_t agg;
  uint64_t run = block_excl_scan<kScanBlock>(sum, s_scratch, &agg);
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    if (base + k < n) op.emit(base + k, run, c[k]);
    run += c[k];
  }
  if (threadIdx.x == kScanBlock - 1) op.total(agg);
}

// k_scan over up to n_max items (device size op.size()): one tile -> k_scan_one, else the
// decoupled look-back scan with its status words zeroed first.
template <class Op>
inline cudaError_t launch_scan(const Op& op, uint64_t n_max, uint64_t* status, cudaStream_t st) {
  const uint64_t tiles = scan_tiles(n_max);
  if (tiles <= 1) {
    return launch_k(true, k_scan_one<Op>, 1, kScanBlock, 0, st, op);
  }
  cudaError_t e = cudaMemsetAsync(status, 0, (tiles + 1) * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  k_scan<Op><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, status, reinterpret_cast<uint32_t*>(status + tiles));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits.
// ---------------------------------------------------------------------------------
constexpr int kSortBlock = 256;
constexpr int kSortIPT = 8;
constexpr int kSortTile = kSortBlock * kSortIPT;  // 2048 items
constexpr int kSortWarps = kSortBlock / 32;
constexpr uint32_t kSortAgg = 1u << 30;
constexpr uint32_t kSortInc = 2u << 30;
constexpr uint32_t kSortVal = kSortAgg - 1;

// Global histograms for every pass in one read of the keys.
static __global__ void __launch_bounds__(256) k_radix_hist(const uint32_t* __restrict__ keys, const uint64_t* d_n,
                                                    int passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&s_h[0][0])[i] = 0;
  pdl_wait();
  pdl_launch_dependents();
  trace_begin(kTrHist);
  __syncthreads();
  const uint64_t n = *d_n;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t v = (&s_h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
  trace_end(kTrHist);
}

__host__ __device__ __forceinline__ bool radix_pass_needed(uint32_t key_bound, int shift) {
  return shift == 0 || (key_bound > 0 && ((key_bound - 1) >> shift) != 0);
}
// Passes of an LSD sort over `passes` digits that run when every key is below key_bound
// (the rest are skipped by k_radix_pass): the result is in the second buffer iff this is odd.
__host__ __device__ __forceinline__ int radix_passes_run(uint32_t key_bound, int passes) {
  int e = 1;
  while (e < passes && radix_pass_needed(key_bound, 8 * e)) ++e;
  return e;
}

// One digit pass. vals_in == nullptr: the value of item i is i (identity payload).
static __global__ void __launch_bounds__(kSortBlock) k_radix_pass(const uint32_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out, const uint64_t* d_n,
                                                           int shift, const uint32_t* __restrict__ hist,
                                                           uint32_t* status, uint32_t* ticket,
                                                           const uint32_t* key_bound) {
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  __shared__ uint32_t s_whist[kSortWarps][256];
  __shared__ uint32_t s_doff[256];  // block-local exclusive start of each digit
  __shared__ uint32_t s_goff[256];  // global start of this tile's run of each digit
  __shared__ uint32_t s_scr[33];
  __shared__ uint32_t s_tile;

  pdl_wait();
  pdl_launch_dependents();
  // key_bound (optional): every key is below *key_bound, known only on the device. A pass
  // whose digit (and every higher one) is then zero for all keys would be an identity
  // permutation: skipped (radix_passes_run() names the buffer that holds the result).
  if (key_bound && shift > 0 && !radix_pass_needed(*key_bound, shift)) return;
  trace_begin(kTrPass0 + shift / 8);
  const uint64_t n = *d_n;
  const uint64_t n_tiles = (n + kSortTile - 1) / kSortTile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortBlock) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  if (tile >= n_tiles) return;

  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint64_t wbase = tile * kSortTile + uint64_t(w) * 32 * kSortIPT;
  uint32_t key[kSortIPT], val[kSortIPT], rank[kSortIPT];
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const uint64_t i = wbase + uint64_t(j) * 32 + l;
    const bool ok = i < n;
    key[j] = ok ? keys_in[i] : 0xffffffffu;
    val[j] = ok ? (vals_in ? vals_in[i] : static_cast<uint32_t>(i)) : 0u;
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const uint64_t i = wbase + uint64_t(j) * 32 + l;
    const bool ok = i < n;
    const uint32_t d = ok ? ((key[j] >> shift) & 255u) : 256u + l;  // invalid items never match
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t r = 0;
    if (ok) r = s_whist[w][d] + __popc(peers & lt);
    __syncwarp();
    if (ok && (__ffs(peers) - 1) == l) s_whist[w][d] += __popc(peers);
    __syncwarp();
    rank[j] = r;
  }
  __syncthreads();

  // Thread t owns digit t: per-warp exclusive offsets and the tile count.
  const uint32_t d = threadIdx.x;
  uint32_t cnt = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = s_whist[ww][d];
    s_whist[ww][d] = cnt;
    cnt += c;
  }
  if (tile == 0) {
    st_vol32(&status[d], kSortInc | cnt);
  } else {
    st_vol32(&status[tile * 256 + d], kSortAgg | cnt);
  }
  // global digit starts for this pass + block-local digit starts
  uint32_t tot;
  const uint32_t gstart = block_excl_scan<kSortBlock>(hist[d], s_scr, &tot);
  const uint32_t lstart = block_excl_scan<kSortBlock>(cnt, s_scr, &tot);
  s_doff[d] = lstart;
  uint32_t prefix = 0;
  if (tile > 0) {
    // Batched look-back: 16 predecessor words per round are loaded together, so a chain
    // of tiles that have only published aggregates costs ceil(k/16) L2 round trips.
    constexpr int kLB = 16;
    int64_t p = static_cast<int64_t>(tile) - 1;
    bool done = false;
    while (!done) {
      uint32_t sv[kLB];
#pragma unroll
      for (int q = 0; q < kLB; ++q) sv[q] = (p - q >= 0) ? ld_vol32(&status[(p - q) * 256 + d]) : kSortInc;
#pragma unroll
      for (int q = 0; q < kLB; ++q) {
        if (done) break;
        uint32_t s = sv[q];
        while ((s & ~kSortVal) == 0) s = ld_vol32(&status[(p - q) * 256 + d]);  // not yet published
        prefix += s & kSortVal;
        done = (s & kSortInc) != 0;
      }
      p -= kLB;
    }
    st_vol32(&status[tile * 256 + d], kSortInc | (prefix + cnt));
  }
  s_goff[d] = gstart + prefix;
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const uint64_t i = wbase + uint64_t(j) * 32 + l;
    if (i < n) {
      const uint32_t dj = (key[j] >> shift) & 255u;
      const uint32_t pos = s_doff[dj] + s_whist[w][dj] + rank[j];
      s_keys[pos] = key[j];
      s_vals[pos] = val[j];
    }
  }
  __syncthreads();
  const uint64_t tile_n = (n - tile * kSortTile) < uint64_t(kSortTile) ? (n - tile * kSortTile) : uint64_t(kSortTile);
  for (uint32_t i = threadIdx.x; i < tile_n; i += kSortBlock) {
    const uint32_t k = s_keys[i];
    const uint32_t dk = (k >> shift) & 255u;
    const uint32_t g = s_goff[dk] + (i - s_doff[dk]);
    keys_out[g] = k;
    vals_out[g] = s_vals[i];
  }
  trace_end(kTrPass0 + shift / 8);
}

inline uint64_t sort_tiles(uint64_t n_max) { return (n_max + kSortTile - 1) / kSortTile; }

// Workspace of one sort: [hist: 4*256 u32][tickets: 4 u32][status: passes*tiles*256 u32].
inline size_t sort_ws_words(uint64_t n_max, int passes) {
  return 4 * 256 + 4 + static_cast<size_t>(passes) * sort_tiles(n_max) * 256;
}

// Sort (keys_a, vals) by the low `bits` bits of the keys, stably. Results end in
// (keys_a, vals_a) or (keys_b, vals_b); returns true when in the _b buffers.
// vals_in == nullptr means identity values. `ws` must hold sort_ws_words() words.
inline bool radix_sort_pairs(cudaStream_t st, uint32_t* keys_a, const uint32_t* vals_in, uint32_t* vals_a,
                             uint32_t* keys_b, uint32_t* vals_b, const uint64_t* d_n, uint64_t n_max,
                             int bits, uint32_t* ws, cudaError_t* err) {
  const int passes = bits <= 0 ? 1 : (bits + 7) / 8;
  const uint64_t tiles = sort_tiles(n_max);
  uint32_t* hist = ws;
  uint32_t* tickets = ws + 4 * 256;
  uint32_t* status = tickets + 4;
  *err = cudaMemsetAsync(ws, 0, sort_ws_words(n_max, passes) * sizeof(uint32_t), st);
  if (*err != cudaSuccess) return false;
  k_radix_hist<<<grid_for(n_max, 256, kNumSMs * 2), 256, 0, st>>>(keys_a, d_n, passes, hist);
  const uint32_t* kin = keys_a;
  const uint32_t* vin = vals_in;
  bool in_b = false;
  for (int p = 0; p < passes; ++p) {
    uint32_t* kout = in_b ? keys_a : keys_b;
    uint32_t* vout = in_b ? vals_a : vals_b;
    k_radix_pass<<<static_cast<unsigned>(tiles), kSortBlock, 0, st>>>(
        kin, vin, kout, vout, d_n, 8 * p, hist + 256 * p, status + static_cast<size_t>(p) * tiles * 256, tickets + p,
        nullptr);
    kin = kout;
    vin = vout;
    in_b = !in_b;
  }
  *err = cudaGetLastError();
  return in_b;
}

}  // namespace hpsg
