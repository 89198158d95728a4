// backward.cu — K4 dedup + blocked segmented reduction and K5 fused sparse optimizers.
//
// Semantics (oracle/oracle.cpp reduce_and_update): every key
// occurrence receives d_out[bag] (or d_out[bag]/len for mean); the occurrences of one
// key are taken in canonical (occurrence) order and reduced by a 32-ary blocked tree:
// chunks of 32 summed sequentially from their first element, the chunk partials reduced
// the same way until one vector remains (plain sequential order up to 32 occurrences).
// Then SGD / AdaGrad / Adam update the row in place.
//
// Dedup without a global sort (sizes device-resident, graph-capturable). The training
// lookup's probe records each occurrence's row; then, on the table's side stream and
// concurrently with the pooling (table.cu record / fork_dedup):
//   k_count         : per-row occurrence counts in an L2-resident batch table (CTA-level
//                     shared-memory aggregation first, so hot rows take one atomic per
//                     CTA); each occurrence gets an arrival rank within its row
//   k_seg_alloc     : the rank-0 occurrence of each row allocates its segment — short rows
//                     (<= 32 occurrences) a CSR range of the short list, long rows an id —
//                     and leaves the locator in the batch table
//   k_scan<PlaceOp> : every occurrence drops its bag into its short segment at `rank`, or is
//                     compacted (canonical order) into the long list as (long id, bag)
//   long sort       : stable radix sort of the long list by long id (few bits) — each long
//                     segment contiguous, occurrences in canonical order
//   (no registration pass: each long segment registers its list start, first level-1 chunk,
//                     tree-node block, the sort's digit histogram counts and its chunk ->
//                     segment map entries when it is allocated: register_long)
// and at backward_update, the short and long reductions run side by side (disjoint rows):
//   k_reduce_short  : a warp owns 32 short segments: sorts each one's bags back into canonical
//                     order (warp rank), reduces and updates (bulk-copy or register path)
//   k_long (side)   : one warp per chunk -> level-1 partial; the last chunk to finish below
//                     a tree node sums that node's <= 32 children in order, up to the root,
//                     whose sum goes through the optimizer (hierarchical last-arriver)
// Every batch-table entry is reset to empty by the kernel that consumes it last.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "primitives.cuh"
#include "table_internal.cuh"

using namespace hpsg;

namespace {

struct BwdArgs {
  const uint64_t* counts;   // [0] = N occurrences; [1] <- unique rows (short + long segments)
  const uint32_t* occ_row;  // row of each occurrence (row_absent: no gradient)
  uint32_t* occ_rank;       // arrival rank of each occurrence within its row
  uint32_t* lead;           // k_dedup: per-CTA compact list of its leaders (rank-0 occurrences)
  const uint32_t* occ_bag;  // multi-hot: bag of each occurrence (nullptr: occurrence i is bag i)
  uint32_t* occ_ent;        // batch-table entry of each occurrence's row
  uint2* bt;                // batch table {row, UINT32_MAX + count -> segment locator}
  uint64_t bt_mask;
  uint32_t row_absent;
  unsigned long long* short_alloc;  // (segments << 32) | occurrences
  uint4* short_rec;                 // {row, first, len, batch-table entry}
  uint32_t* short_bag;
  uint32_t* n_long;                 // (the count half of long_alloc)
  unsigned long long* long_alloc;   // (segments << 32) | occurrences: id, list start of each long segment
  uint32_t* long_row;
  uint32_t* long_ent;
  uint32_t* long_len;
  uint32_t* long_start;     // first position of the segment in the sorted long list
  uint32_t* long_hist;      // histograms of the long sort's digit passes [passes x 256] (occurrence counts)
  int long_passes;
  uint32_t* lkey;           // long list: segment id (sort input)
  uint32_t* lval;           // long list: bag (sort input)
  const uint32_t* lval_b;   // the sort's second value buffer: the sorted bags are in lval or here
                            // (radix_passes_run: the passes above the segment count's digits are skipped)
  unsigned long long* long_occ;     // long-list length
  unsigned long long* long_chunks;  // level-1 chunks over all long segments
  const uint32_t* bag_len;  // mean combiner: bag lengths (nullptr: sum)
  const float* dout;
  uint32_t dim;
  uint32_t* long_base;
  uint32_t* task_long;
  float* partial;                   // level-1 partials [max_chunks x dim]
  float* partial2;                  // higher levels [max_chunks/32 + max_long x dim]
  uint32_t* long_hbase;             // long segment -> first node of its levels >= 2 in partial2
  uint32_t* node_cnt;               // arrivals per tree node (self-resetting)
  uint32_t* higher_total;           // allocator of partial2 nodes (zeroed per call)
  uint32_t* touched;                // kOptGrad: row -> 1 when its gradient was written
  uint32_t tma_rows;                // rows per warp buffer in short_tma
  uint32_t n_slots;                 // one-hot: occurrence i = sample * n_slots + slot
  float* W;
  float* S0;
  float* S1;
  int optimizer;
  hps_opt_params opt;
  bool grad_once;   // one-hot batch: every gradient row is read once (row stream: L2 evict_first)
};

// ---- batch table ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t bt_home(uint32_t row, uint64_t mask) {
  // Fibonacci hashing: the TOP log2(size) bits of the 64-bit product (the middle bits of it
  // cluster dense row ids: 4x the home collisions of a uniform hash on config 1)
  return static_cast<uint32_t>((uint64_t(row) * 0x9E3779B97F4A7C15ull) >> (64 - __popcll(mask)));
}
// Entry of `row` (inserted if absent), probing from `h`: each round reads a window of 4
// keys at once and CASes only the first free one, so a collision chain costs a quarter of
// the dependent round trips of slot-by-slot probing.
__device__ __forceinline__ uint32_t bt_insert_from(uint2* bt, uint64_t mask, uint32_t row, uint32_t h) {
  while (true) {
    uint32_t k[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) k[s] = __ldcg(&bt[(h + s) & mask].x);
    int free_s = -1;
#pragma unroll
    for (int s = 3; s >= 0; --s) {
      if (k[s] == row) return static_cast<uint32_t>((h + s) & mask);
      if (k[s] == kBtEmpty) free_s = s;
    }
    if (free_s < 0) {
      h = static_cast<uint32_t>((h + 4) & mask);
      continue;
    }
    // a key equal to `row` cannot sit after the first free slot of the window (entries are
    // never removed while a batch is being counted), so the free slot is where it belongs
    const uint32_t slot = static_cast<uint32_t>((h + free_s) & mask);
    const uint32_t old = atomicCAS(&bt[slot].x, kBtEmpty, row);
    if (old == kBtEmpty || old == row) return slot;
    h = slot;  // raced: re-read from this slot
  }
}
__device__ __forceinline__ uint32_t bt_insert(uint2* bt, uint64_t mask, uint32_t row) {
  return bt_insert_from(bt, mask, row, bt_home(row, mask));
}

__device__ __forceinline__ uint32_t higher_nodes(uint32_t m);

// A long leader (its row has more than kChunk occurrences) registers its segment right away
// (every lane of the warp calls it): id and start in the sorted long list from one packed
// atomic per warp — ids in allocator order, so the starts are the prefix of the lengths in id
// order, exactly where the stable sort by id will put each segment — its first level-1 chunk
// from a second counter (the chunk total is that counter) and its tree-node block.
// `hist`: where the sort's digit histograms are counted — the global ones, or a CTA's shared
// copy (k_dedup: flushed once per CTA, so the high digits' few bins, which every segment id
// shares, do not serialise thousands of global atomics).
__device__ __forceinline__ void register_long(const BwdArgs& a, bool lg, uint32_t row, uint32_t ent, uint32_t len,
                                              uint32_t* hist) {
  if (!__ballot_sync(0xffffffffu, lg)) return;
  const uint32_t lane = lane_id();
  const uint32_t m = lg ? (len + kChunk - 1) / kChunk : 0u;
  const uint32_t h = lg ? higher_nodes(m) : 0u;
  const unsigned long long mine = lg ? ((1ull << 32) | len) : 0ull;
  const unsigned long long incl = warp_incl_scan(mine);
  const unsigned long long cincl = warp_incl_scan(static_cast<unsigned long long>(m));
  const uint32_t hincl = warp_incl_scan(h);
  unsigned long long base = 0, cbase = 0;
  uint32_t hbase = 0;
  if (lane == 31) {
    base = atomicAdd(a.long_alloc, incl);
    cbase = atomicAdd(a.long_chunks, cincl);
    hbase = atomicAdd(a.higher_total, hincl);
  }
  base = __shfl_sync(0xffffffffu, base, 31);
  cbase = __shfl_sync(0xffffffffu, cbase, 31);
  hbase = __shfl_sync(0xffffffffu, hbase, 31);
  uint32_t j = 0, cb = 0;
  if (lg) {
    const unsigned long long pos = base + incl - mine;
    j = static_cast<uint32_t>(pos >> 32);
    cb = static_cast<uint32_t>(cbase + cincl - m);
    a.long_row[j] = row;
    a.long_ent[j] = ent;
    a.long_len[j] = len;
    a.long_start[j] = static_cast<uint32_t>(pos);
    a.long_base[j] = cb;
    a.long_hbase[j] = hbase + hincl - h;
    a.bt[ent].y = kLongFlag | j;
    // the long-list sort's digit histograms: segment j's len occurrences all carry key j
    for (int p = 0; p < a.long_passes; ++p) atomicAdd(&hist[256 * p + ((j >> (8 * p)) & 255u)], len);
  }
  // the chunk -> segment map of the long reduce, written by the whole warp per segment
  uint32_t todo = __ballot_sync(0xffffffffu, lg);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t sj = __shfl_sync(0xffffffffu, j, src), sb = __shfl_sync(0xffffffffu, cb, src);
    const uint32_t sm = __shfl_sync(0xffffffffu, m, src);
    for (uint32_t c = lane; c < sm; c += 32) a.task_long[sb + c] = sj;
  }
}

// ---- K4a-c fused: counts, allocation, placement in ONE persistent cooperative kernel ------
// One CTA per SM (64 KB shared hash + 512 threads: it sits beside the pooling kernel it
// overlaps); CTA c owns the contiguous occurrence chunk [c*n/G, (c+1)*n/G). Three grid
// barriers separate the phases that need every CTA's results:
//   P1 counts: shared-hash aggregation over the chunk, then ONE batch-table reservation
//      (CAS + add) per distinct row per CTA -> each occurrence's rank and table entry
//   P2 allocation: the rank-0 occurrence of each row (now final counts) takes a short
//      CSR range (one packed atomic per CTA, handed out in occurrence order) or a long id
//   P3 placement: short occurrences drop their bag at first + rank; long occurrences are
//      compacted in canonical order (per-CTA counts -> prefix over CTAs -> block scans)
// Batch-table words written by other CTAs are read through L2 (__ldcg) after a barrier.
constexpr int kDedupHash = 8192;
constexpr uint32_t kNoEnt = 0xffffffffu;
constexpr uint32_t kDirectEnt = 0x80000000u;  // occ_ent flag inside P1: counted directly

__device__ __forceinline__ uint32_t smem_hash_slot(uint32_t* s_key, uint32_t row) {
  uint32_t h = (row * 0x9e3779b1u) >> 19;  // 13 bits
  for (int probe = 0; probe < 128; ++probe) {
    const uint32_t cur = s_key[h];
    if (cur == row) return h;
    if (cur == kBtEmpty) {
      const uint32_t old = atomicCAS(&s_key[h], kBtEmpty, row);
      if (old == kBtEmpty || old == row) return h;
    }
    h = (h + 1) & (kDedupHash - 1);
  }
  return kNoEnt;
}

// Every pass walks the chunk in batches of kDedupIPT items per thread whose loads are all
// issued before any is consumed (these phases are latency-bound, not bandwidth-bound). Two
// shapes (choose_dedup_shape): 512 threads x 8 items, or 1024 threads x 4 (twice the warps
// to hide the phases' L2 round trips; config 2: 0.138 -> 0.12 ms; the Zipf configs, whose
// large chunks favour the deeper per-thread batches, keep 512 x 8).
template <int kDedupBlock, int kDedupIPT>
__global__ void __launch_bounds__(kDedupBlock, 1024 / kDedupBlock) k_dedup(BwdArgs a, uint32_t* coop) {
  extern __shared__ uint32_t s_dd[];
  uint32_t* s_key = s_dd;               // row, then its batch-table entry
  uint32_t* s_val = s_dd + kDedupHash;  // chunk count, then the CTA's base rank
  __shared__ unsigned long long s_scr[33];
  __shared__ unsigned long long s_cursor;
  __shared__ uint32_t s_scr32[33];
  __shared__ uint32_t s_nlead;
  __shared__ uint32_t s_lhist[4 * 256];  // this CTA's long-sort digit histograms (register_long)
  trace_begin(kTrCount);
  const uint64_t n = a.counts[0];
  if (a.counts[5]) {
    // the slot's previous record was never consumed by a backward (counts[5], cleared by the
    // reduces): its batch-table entries go back to empty first — read from its occ_ent (an
    // entry per present occurrence, kNoEnt per absent one) before P1 overwrites them. Every
    // CTA reads the same flag: it is set again only after the first barrier below.
    const uint64_t n_old = a.counts[6];
    for (uint64_t i = blockIdx.x * uint64_t(kDedupBlock) + threadIdx.x; i < n_old; i += uint64_t(gridDim.x) * kDedupBlock) {
      const uint32_t e = a.occ_ent[i];
      if (e != kNoEnt) a.bt[e] = make_uint2(kBtEmpty, 0xffffffffu);
    }
    grid_barrier_once(coop + 3);
  }
  const uint64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  const uint32_t lane = lane_id(), lt = lanemask_lt();
  constexpr uint64_t kBatch = uint64_t(kDedupBlock) * kDedupIPT;
  // ---- P1: counts and ranks
  for (int e = threadIdx.x; e < kDedupHash; e += kDedupBlock) {
    s_key[e] = kBtEmpty;
    s_val[e] = 0u;
  }
  __syncthreads();
  for (uint64_t b0 = c0; b0 < c1; b0 += kBatch) {
    uint32_t row[kDedupIPT];
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint64_t i = b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      row[k] = i < c1 ? a.occ_row[i] : a.row_absent;
    }
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k)  // the rows' batch-table home lines into L2 now: the
      if (row[k] != a.row_absent)        // reservations below then hit L2
        asm volatile("prefetch.global.L2 [%0];" ::"l"(&a.bt[bt_home(row[k], a.bt_mask)]));
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint64_t i = b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      if (row[k] == a.row_absent) {
        if (i < c1) a.occ_ent[i] = kNoEnt;  // (an unconsumed record's reset skips it)
        continue;
      }
      const uint32_t h = smem_hash_slot(s_key, row[k]);
      if (h != kNoEnt) {
        a.occ_rank[i] = atomicAdd(&s_val[h], 1u);
        a.occ_ent[i] = h;
      } else {  // shared hash full: count directly
        const uint32_t e = bt_insert(a.bt, a.bt_mask, row[k]);
        a.occ_rank[i] = atomicAdd(&a.bt[e].y, 1u) + 1u;
        a.occ_ent[i] = kDirectEnt | e;
      }
    }
  }
  trace_end(kTrCountLocal);
  __syncthreads();
  {  // one reservation per distinct row: every home-slot CAS in flight at once, the (rare,
     // sparse table) collisions resolved after, then every add in flight at once
    constexpr int kPer = kDedupHash / kDedupBlock;
    uint32_t key[kPer], ent[kPer], res[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      key[q] = s_key[threadIdx.x + kDedupBlock * q];
      ent[q] = key[q] != kBtEmpty ? bt_home(key[q], a.bt_mask) : kNoEnt;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      res[q] = ent[q] != kNoEnt ? atomicCAS(&a.bt[ent[q]].x, kBtEmpty, key[q]) : kBtEmpty;
    trace_end_after(kTrCountCas, res[0] ^ res[kPer - 1]);
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      if (ent[q] != kNoEnt && res[q] != kBtEmpty && res[q] != key[q])
        ent[q] = bt_insert_from(a.bt, a.bt_mask, key[q], static_cast<uint32_t>((ent[q] + 1) & a.bt_mask));
    trace_end_after(kTrCountProbe, ent[0] ^ ent[kPer - 1]);
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      res[q] = ent[q] != kNoEnt ? atomicAdd(&a.bt[ent[q]].y, s_val[threadIdx.x + kDedupBlock * q]) + 1u : 0u;

#pragma unroll
    for (int q = 0; q < kPer; ++q) {  // entry e is owned by this thread: no hazard with other threads
      s_key[threadIdx.x + kDedupBlock * q] = ent[q];
      s_val[threadIdx.x + kDedupBlock * q] = res[q];
    }
  }
  trace_end(kTrCountGlobal);
  if (threadIdx.x == 0) s_nlead = 0;
  __syncthreads();
  // final ranks and entries; the rank-0 occurrences (leaders) go to the CTA's leader list
  for (uint64_t b0 = c0; b0 < c1; b0 += kBatch) {
    uint32_t h[kDedupIPT], r[kDedupIPT];
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint64_t i = b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      h[k] = (i < c1 && a.occ_row[i] != a.row_absent) ? a.occ_ent[i] : kNoEnt;
      r[k] = h[k] != kNoEnt ? a.occ_rank[i] : 1u;
    }
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint64_t i = b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      if (h[k] != kNoEnt) {
        if (h[k] & kDirectEnt) {
          a.occ_ent[i] = h[k] & ~kDirectEnt;
        } else {
          r[k] += s_val[h[k]];
          a.occ_rank[i] = r[k];
          a.occ_ent[i] = s_key[h[k]];
        }
      }
      const bool is_lead = h[k] != kNoEnt && r[k] == 0u;
      const uint32_t m = __ballot_sync(0xffffffffu, is_lead);
      if (m) {
        uint32_t base = 0;
        if (lane == static_cast<uint32_t>(__ffs(m) - 1)) base = atomicAdd(&s_nlead, static_cast<uint32_t>(__popc(m)));
        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
        if (is_lead) a.lead[c0 + base + __popc(m & lt)] = static_cast<uint32_t>(i);
      }
    }
  }
  trace_end(kTrCount);
  grid_barrier_once(coop + 0);
  // this slot now holds a record whose batch-table entries await a backward (counts[5]; its
  // size in counts[6] for the reset above, should none come)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const_cast<uint64_t*>(a.counts)[6] = n;
    const_cast<uint64_t*>(a.counts)[5] = 1;
  }
  // ---- P2: allocation. Short leaders: the CTA reserves its CSR range with one packed
  // atomic, then hands it out in item order (block scans), so segment s+1 starts where
  // segment s ends. Long leaders: ids from a warp-aggregated counter.
  trace_begin(kTrAlloc);
  for (int e = threadIdx.x; e < a.long_passes * 256; e += kDedupBlock) s_lhist[e] = 0u;
  __syncthreads();
  const uint32_t nlead = s_nlead;  // (the CTA's own list: written before the grid barrier)
  const uint32_t* lead = a.lead + c0;
  if (nlead <= kBatch) {
    // one batch (every one-hot config): each thread's leaders contiguous, loaded once; the
    // block scan gives both the CTA's total (one atomic) and each thread's offset in it
    uint32_t ent[kDedupIPT], len[kDedupIPT], occ[kDedupIPT], row[kDedupIPT];
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint32_t q = threadIdx.x * kDedupIPT + k;
      occ[k] = q < nlead ? lead[q] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint32_t q = threadIdx.x * kDedupIPT + k;
      ent[k] = q < nlead ? a.occ_ent[occ[k]] : kNoEnt;
      row[k] = q < nlead ? a.occ_row[occ[k]] : 0u;
    }
    unsigned long long tmine = 0;
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      len[k] = ent[k] != kNoEnt ? __ldcg(&a.bt[ent[k]].y) + 1u : 0u;
      if (len[k] && len[k] <= kChunk) tmine += (1ull << 32) | len[k];
    }
    unsigned long long ttotal;
    const unsigned long long excl = block_excl_scan<kDedupBlock>(tmine, s_scr, &ttotal);
    if (threadIdx.x == 0) s_cursor = ttotal ? atomicAdd(a.short_alloc, ttotal) : 0ull;
    __syncthreads();
    unsigned long long pos = s_cursor + excl;
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const bool sh = len[k] && len[k] <= kChunk, lg = len[k] > kChunk;
      if (sh) {
        const uint32_t seg = static_cast<uint32_t>(pos >> 32), first = static_cast<uint32_t>(pos);
        a.short_rec[seg] = make_uint4(row[k], first, len[k], ent[k]);
        a.bt[ent[k]].y = first;
        pos += (1ull << 32) | len[k];
      }
      register_long(a, lg, row[k], ent[k], len[k], s_lhist);
    }
  } else {
    unsigned long long mine = 0;
    for (uint32_t b0 = 0; b0 < nlead; b0 += kBatch) {
      uint32_t len[kDedupIPT];
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        const uint32_t q = b0 + k * kDedupBlock + threadIdx.x;
        len[k] = q < nlead ? __ldcg(&a.bt[a.occ_ent[lead[q]]].y) + 1u : 0u;
      }
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k)
        if (len[k] && len[k] <= kChunk) mine += (1ull << 32) | len[k];
    }
    unsigned long long total;
    (void)block_excl_scan<kDedupBlock>(mine, s_scr, &total);
    if (threadIdx.x == 0) s_cursor = total ? atomicAdd(a.short_alloc, total) : 0ull;
    __syncthreads();
    unsigned long long run = s_cursor;
    for (uint32_t b0 = 0; b0 < nlead; b0 += kBatch) {  // each thread's leaders contiguous; block scan
      uint32_t ent[kDedupIPT], len[kDedupIPT], occ[kDedupIPT];
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        const uint32_t q = b0 + threadIdx.x * kDedupIPT + k;
        occ[k] = q < nlead ? lead[q] : 0u;
        ent[k] = q < nlead ? a.occ_ent[occ[k]] : kNoEnt;
      }
      unsigned long long tmine = 0;
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        len[k] = ent[k] != kNoEnt ? __ldcg(&a.bt[ent[k]].y) + 1u : 0u;
        if (len[k] && len[k] <= kChunk) tmine += (1ull << 32) | len[k];
      }
      unsigned long long ttotal;
      unsigned long long pos = run + block_excl_scan<kDedupBlock>(tmine, s_scr, &ttotal);
      run += ttotal;
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        const bool sh = len[k] && len[k] <= kChunk, lg = len[k] > kChunk;
        if (sh) {
          const uint32_t seg = static_cast<uint32_t>(pos >> 32), first = static_cast<uint32_t>(pos);
          a.short_rec[seg] = make_uint4(a.occ_row[occ[k]], first, len[k], ent[k]);
          a.bt[ent[k]].y = first;
          pos += (1ull << 32) | len[k];
        }
        register_long(a, lg, lg ? a.occ_row[occ[k]] : 0u, ent[k], len[k], s_lhist);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.long_passes * 256; e += kDedupBlock)
    if (const uint32_t v = s_lhist[e]) atomicAdd(&a.long_hist[e], v);
  trace_end(kTrAlloc);
  grid_barrier_once(coop + 1);
  // ---- P3: placement
  trace_begin(kTrPlace);
  // a chunk that fits one batch (every one-hot config) walks its items thread-contiguously and
  // keeps their locators: the long compaction after the barrier then needs no second pass
  // over the record (its canonical order is the thread order, its offsets the scan below)
  const bool one = c1 - c0 <= kBatch;
  // a larger chunk that fits the (now idle) shared hash keeps its locators there instead
  const bool cached = !one && c1 - c0 <= 2 * kDedupHash;
  uint32_t my_long = 0;
  uint32_t keep[kDedupIPT];
  for (uint64_t b0 = c0; b0 < c1; b0 += kBatch) {
    uint32_t ent[kDedupIPT], loc[kDedupIPT];
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      const uint64_t i = one ? b0 + uint64_t(threadIdx.x) * kDedupIPT + k : b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      ent[k] = (i < c1 && a.occ_row[i] != a.row_absent) ? a.occ_ent[i] : kNoEnt;
    }
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) loc[k] = ent[k] != kNoEnt ? __ldcg(&a.bt[ent[k]].y) : 0u;
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      keep[k] = loc[k];
      if (cached) {
        const uint64_t i = b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
        if (i < c1) s_dd[i - c0] = loc[k];
      }
      if (ent[k] == kNoEnt) continue;
      const uint64_t i = one ? b0 + uint64_t(threadIdx.x) * kDedupIPT + k : b0 + uint64_t(k) * kDedupBlock + threadIdx.x;
      if (loc[k] & kLongFlag) {
        ++my_long;
      } else {
        a.short_bag[loc[k] + a.occ_rank[i]] = a.occ_bag ? a.occ_bag[i] : static_cast<uint32_t>(i);
      }
    }
  }
  uint32_t cta_long;
  const uint32_t my_off = block_excl_scan<kDedupBlock>(my_long, s_scr32, &cta_long);
  if (threadIdx.x == 0) st_vol32(coop + 4 + blockIdx.x, cta_long);
  grid_barrier_once(coop + 2);
  uint32_t before = 0;
  for (uint32_t c = threadIdx.x; c < blockIdx.x; c += kDedupBlock) before += ld_vol32(coop + 4 + c);
  uint32_t lbase;
  (void)block_excl_scan<kDedupBlock>(before, s_scr32, &lbase);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *a.long_occ = lbase + cta_long;
  if (cta_long && one) {
    uint32_t pos = lbase + my_off;
#pragma unroll
    for (int k = 0; k < kDedupIPT; ++k) {
      if (!(keep[k] & kLongFlag)) continue;
      const uint64_t i = c0 + uint64_t(threadIdx.x) * kDedupIPT + k;
      a.lkey[pos] = keep[k] & ~kLongFlag;
      a.lval[pos] = a.occ_bag ? a.occ_bag[i] : static_cast<uint32_t>(i);
      ++pos;
    }
  } else if (cta_long) {  // canonical order: batches in order, each thread's kDedupIPT items contiguous
    for (uint64_t b0 = c0; b0 < c1; b0 += kBatch) {
      uint32_t loc[kDedupIPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        const uint64_t i = b0 + uint64_t(threadIdx.x) * kDedupIPT + k;
        if (cached) {
          loc[k] = i < c1 ? s_dd[i - c0] : 0u;
        } else {
          const uint32_t e = (i < c1 && a.occ_row[i] != a.row_absent) ? a.occ_ent[i] : kNoEnt;
          loc[k] = e != kNoEnt ? __ldcg(&a.bt[e].y) : 0u;
        }
      }
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) cnt += (loc[k] & kLongFlag) ? 1u : 0u;
      uint32_t ttotal;
      uint32_t pos = lbase + block_excl_scan<kDedupBlock>(cnt, s_scr32, &ttotal);
#pragma unroll
      for (int k = 0; k < kDedupIPT; ++k) {
        if (!(loc[k] & kLongFlag)) continue;
        const uint64_t i = b0 + uint64_t(threadIdx.x) * kDedupIPT + k;
        a.lkey[pos] = loc[k] & ~kLongFlag;
        a.lval[pos] = a.occ_bag ? a.occ_bag[i] : static_cast<uint32_t>(i);
        ++pos;
      }
      lbase += ttotal;
    }
  }
  trace_end(kTrPlace);
}

// ---- K4a-c flat: the same products from three full-occupancy kernels (no grid barriers) ---
// k_count_flat : one occurrence per thread; the lanes of a warp holding the same row are
//                merged (match_any) and their leader reserves the row's batch-table entry
//                with ONE CAS + ONE add: every occurrence gets its arrival rank and entry
// k_alloc_flat : the rank-0 occurrence of each row (its count is final now) takes a short
//                CSR range (block scan + one packed atomic per block) or a long id
// k_scan<PlaceOp>: short occurrences drop their bag at first + rank; long ones are compacted
//                in canonical order (decoupled look-back scan)
// Latency-bound phases at full occupancy: every load and atomic of a phase is in flight at
// once, instead of one persistent CTA per SM walking its chunk.
__global__ void __launch_bounds__(256) k_count_flat(BwdArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  trace_begin(kTrCount);
  const uint64_t n = a.counts[0];
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // (as k_dedup; the flat path's reset is table.cu k_reset_counts)
    const_cast<uint64_t*>(a.counts)[6] = n;
    const_cast<uint64_t*>(a.counts)[5] = 1;
  }
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (blockIdx.x * uint64_t(blockDim.x) >= n) return;  // whole warps past the end leave together
  // One-hot batches are walked slot-major (a warp holds 32 samples of one slot), so the rows of
  // small tables — hundreds of occurrences each — merge within warps (config 2's 3-row table:
  // 3 atomics per warp instead of 32 on the same three entries)
  uint64_t i = j;
  if (!a.occ_bag && a.n_slots > 1 && n % a.n_slots == 0) {
    const uint64_t ns = n / a.n_slots;
    i = (j % ns) * a.n_slots + j / ns;
  }
  const uint32_t row = j < n ? a.occ_row[i] : a.row_absent;
  const bool active = row != a.row_absent;
  const uint32_t peers = __match_any_sync(0xffffffffu, row);
  const int leader = __ffs(peers) - 1;
  uint32_t e = 0, base = 0;
  if (active && static_cast<int>(lane_id()) == leader) {
    e = bt_insert(a.bt, a.bt_mask, row);
    base = atomicAdd(&a.bt[e].y, static_cast<uint32_t>(__popc(peers))) + 1u;
  }
  e = __shfl_sync(0xffffffffu, e, leader);
  base = __shfl_sync(0xffffffffu, base, leader);
  if (active) {
    a.occ_ent[i] = e;
    a.occ_rank[i] = base + __popc(peers & lanemask_lt());
  } else if (j < n) {
    a.occ_ent[i] = kNoEnt;
  }
  trace_end(kTrCount);
}

constexpr int kAllocIPT = 4;
__global__ void __launch_bounds__(256) k_alloc_flat(BwdArgs a) {
  __shared__ unsigned long long s_scr[33];
  __shared__ unsigned long long s_cursor;
  pdl_wait();
  pdl_launch_dependents();
  trace_begin(kTrAlloc);
  const uint64_t n = a.counts[0];
  const uint64_t b0 = blockIdx.x * uint64_t(256 * kAllocIPT);
  if (b0 >= n) return;
  uint32_t ent[kAllocIPT], len[kAllocIPT];
  unsigned long long mine = 0;
#pragma unroll
  for (int k = 0; k < kAllocIPT; ++k) {
    const uint64_t i = b0 + threadIdx.x * kAllocIPT + k;
    const bool lead = i < n && a.occ_row[i] != a.row_absent && a.occ_rank[i] == 0u;
    ent[k] = lead ? a.occ_ent[i] : kNoEnt;
    len[k] = lead ? __ldcg(&a.bt[ent[k]].y) + 1u : 0u;
    if (len[k] && len[k] <= kChunk) mine += (1ull << 32) | len[k];
  }
  unsigned long long total;
  unsigned long long pos = block_excl_scan<256>(mine, s_scr, &total);
  if (threadIdx.x == 0) s_cursor = total ? atomicAdd(a.short_alloc, total) : 0ull;
  __syncthreads();
  pos += s_cursor;
#pragma unroll
  for (int k = 0; k < kAllocIPT; ++k) {
    const uint64_t i = b0 + threadIdx.x * kAllocIPT + k;
    const bool sh = len[k] && len[k] <= kChunk, lg = len[k] > kChunk;
    if (sh) {
      const uint32_t seg = static_cast<uint32_t>(pos >> 32), first = static_cast<uint32_t>(pos);
      a.short_rec[seg] = make_uint4(a.occ_row[i], first, len[k], ent[k]);
      a.bt[ent[k]].y = first;
      pos += (1ull << 32) | len[k];
    }
    register_long(a, lg, lg ? a.occ_row[i] : 0u, ent[k], len[k], a.long_hist);
  }
  trace_end(kTrAlloc);
}

struct PlaceOp {
  static constexpr int kTrace = kTrPlace;
  BwdArgs a;
  __device__ uint64_t size() const { return a.counts[0]; }
  __device__ uint32_t bag(uint64_t i) const { return a.occ_bag ? a.occ_bag[i] : static_cast<uint32_t>(i); }
  __device__ uint64_t count(uint64_t i) const {
    if (a.occ_row[i] == a.row_absent) return 0;
    const uint32_t loc = __ldcg(&a.bt[a.occ_ent[i]].y);
    if (loc & kLongFlag) return 1;
    a.short_bag[loc + a.occ_rank[i]] = bag(i);
    return 0;
  }
  __device__ void emit(uint64_t i, uint64_t excl, uint64_t c) const {
    if (!c) return;
    a.lkey[excl] = __ldcg(&a.bt[a.occ_ent[i]].y) & ~kLongFlag;
    a.lval[excl] = bag(i);
  }
  __device__ void total(uint64_t t) const { *a.long_occ = t; }
};

// ---- long segments: registration ---------------------------------------------------------
// Nodes above level 1 of a long segment's 32-ary tree (m level-1 chunks).
__device__ __forceinline__ uint32_t higher_nodes(uint32_t m) {
  uint32_t n = 0;
  while (m > 1) {
    m = (m + kChunk - 1) / kChunk;
    n += m;
  }
  return n;
}


// A warp's 32 short segments [u0, u0+32) occupy one contiguous range of the short list:
// load it into shared memory and sort every segment's bags ascending (= canonical order;
// equal bags carry identical gradients, so their relative order is immaterial).
// Sort every segment's bags (already in sbag, range start r0) ascending in place.
__device__ __forceinline__ void sort_short_bags(uint32_t first, uint32_t len, uint32_t r0, uint32_t* sbag) {
  const uint32_t lane = lane_id();
  uint32_t multi = __ballot_sync(0xffffffffu, len >= 2);
  while (multi) {
    const int j = __ffs(multi) - 1;
    multi &= multi - 1;
    const uint32_t jl = __shfl_sync(0xffffffffu, len, j);
    const uint32_t jo = __shfl_sync(0xffffffffu, first, j) - r0;
    const uint32_t b = lane < jl ? sbag[jo + lane] : 0xffffffffu;
    uint32_t rank = 0;
    for (uint32_t q = 0; q < jl; ++q) {
      const uint32_t x = __shfl_sync(0xffffffffu, b, q);
      rank += (x < b || (x == b && q < lane)) ? 1u : 0u;
    }
    __syncwarp();
    if (lane < jl) sbag[jo + rank] = b;
    __syncwarp();
  }
}

// Asynchronous copy (cp.async, 4 B per element) of the bag range of the 32 segments at u0
// (records rec in the lanes) into sbag; lands by cp_async_wait_all().
__device__ __forceinline__ void prefetch_short_bags(const BwdArgs& a, uint64_t S, uint64_t u0, uint32_t first,
                                                    uint32_t len, uint32_t* sbag) {
  const uint32_t lane = lane_id();
  const uint32_t last = static_cast<uint32_t>(min(uint64_t(31), S - 1 - u0));
  const uint32_t r0 = __shfl_sync(0xffffffffu, first, 0);
  const uint32_t r1 = __shfl_sync(0xffffffffu, first + len, last);
  for (uint32_t p = lane; p < r1 - r0; p += 32)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sbag + p)), "l"(a.short_bag + r0 + p)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Returns this lane's segment offset in sbag; sbag receives the 32 segments' contiguous bag
// range (<= 32 * kChunk entries), each segment sorted.
__device__ __forceinline__ uint32_t stage_short_bags(const BwdArgs& a, uint64_t S, uint64_t u0, uint32_t first,
                                                     uint32_t len, uint32_t* sbag) {
  const uint32_t lane = lane_id();
  const uint32_t last = static_cast<uint32_t>(min(uint64_t(31), S - 1 - u0));
  const uint32_t r0 = __shfl_sync(0xffffffffu, first, 0);
  const uint32_t r1 = __shfl_sync(0xffffffffu, first + len, last);
  for (uint32_t p = lane; p < r1 - r0; p += 32) sbag[p] = a.short_bag[r0 + p];
  __syncwarp();
  sort_short_bags(first, len, r0, sbag);
  return first - r0;
}

// ---- row math --------------------------------------------------------------------------
// Row of weights (+ optimizer state): OPT is HPS_OPT_* at compile time, so the loads are
// branch-free and the unused state registers do not exist.
// kOptGrad: no optimizer — the segment's gradient sum is stored into a dense buffer (a.W
// points at it) and a.touched[row] = 1 (hybrid embedding: replicated hot rows are
// all-reduced before the update, hps_gpu_backward_reduce).
constexpr int kOptGrad = 3;
template <int OPT>
constexpr int state_rows() { return OPT == HPS_OPT_ADAGRAD ? 1 : OPT == HPS_OPT_ADAM ? 2 : 0; }

template <int OPT, int VPL>
struct RowState {
  float4 w[VPL], s[state_rows<OPT>() >= 1 ? VPL : 1], q[state_rows<OPT>() >= 2 ? VPL : 1];
};

template <int OPT, int VPL>
__device__ __forceinline__ void load_row(const BwdArgs& a, uint32_t row, uint32_t gl, uint32_t lpr,
                                         RowState<OPT, VPL>& r) {
  const uint32_t nvec = a.dim / 4;
  const uint64_t base = uint64_t(row) * a.dim;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = min(gl + k * lpr, nvec - 1);  // clamped: no branch around the load
    r.w[k] = reinterpret_cast<const float4*>(a.W + base)[v];
    if constexpr (state_rows<OPT>() >= 1) r.s[k] = reinterpret_cast<const float4*>(a.S0 + base)[v];
    if constexpr (state_rows<OPT>() >= 2) r.q[k] = reinterpret_cast<const float4*>(a.S1 + base)[v];
  }
}

// Fused optimizer (operation order identical to the oracle), then store.
template <int OPT, int VPL>
__device__ __forceinline__ void update_store(const BwdArgs& a, uint32_t row, uint32_t gl, uint32_t lpr,
                                             RowState<OPT, VPL>& r, const float4 (&g)[VPL]) {
  const uint32_t nvec = a.dim / 4;
  const uint64_t base = uint64_t(row) * a.dim;
  const float lr = a.opt.lr, eps = a.opt.eps;
  const float lr_t = (OPT == HPS_OPT_ADAM && a.opt.lr_t_device) ? __ldg(a.opt.lr_t_device) : a.opt.lr_t;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = gl + k * lpr;
    if (v >= nvec) continue;
    float* wf = reinterpret_cast<float*>(&r.w[k]);
    float* sf = reinterpret_cast<float*>(&r.s[state_rows<OPT>() >= 1 ? k : 0]);
    float* qf = reinterpret_cast<float*>(&r.q[state_rows<OPT>() >= 2 ? k : 0]);
    const float* gf = reinterpret_cast<const float*>(&g[k]);
    if constexpr (OPT == kOptGrad) {
      reinterpret_cast<float4*>(a.W + base)[v] = g[k];
      if (v == 0 && a.touched) a.touched[row] = 1u;
      continue;
    } else if constexpr (OPT == HPS_OPT_SGD) {
#pragma unroll
      for (int c = 0; c < 4; ++c) wf[c] = __fsub_rn(wf[c], __fmul_rn(lr, gf[c]));
    } else if constexpr (OPT == HPS_OPT_ADAGRAD) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(sf[c], __fmul_rn(gf[c], gf[c]));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(lr, gf[c]), __fadd_rn(__fsqrt_rn(sf[c]), eps)));
      }
      reinterpret_cast<float4*>(a.S0 + base)[v] = r.s[state_rows<OPT>() >= 1 ? k : 0];
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(__fmul_rn(a.opt.beta1, sf[c]), __fmul_rn(a.opt.one_minus_beta1, gf[c]));
        qf[c] = __fadd_rn(__fmul_rn(a.opt.beta2, qf[c]), __fmul_rn(a.opt.one_minus_beta2, __fmul_rn(gf[c], gf[c])));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(lr_t, sf[c]), __fadd_rn(__fsqrt_rn(qf[c]), eps)));
      }
      reinterpret_cast<float4*>(a.S0 + base)[v] = r.s[state_rows<OPT>() >= 1 ? k : 0];
      reinterpret_cast<float4*>(a.S1 + base)[v] = r.q[state_rows<OPT>() >= 2 ? k : 0];
    }
    reinterpret_cast<float4*>(a.W + base)[v] = r.w[k];
  }
}

// Gradient row of one occurrence: d_out[bag] (/ len for mean).
template <int VPL>
__device__ __forceinline__ void load_grad(const BwdArgs& a, uint32_t bag, uint32_t gl, uint32_t lpr, float4 (&x)[VPL]) {
  const uint32_t nvec = a.dim / 4;
  const float4* d = reinterpret_cast<const float4*>(a.dout + uint64_t(bag) * a.dim);
#pragma unroll
  for (int k = 0; k < VPL; ++k) x[k] = __ldg(d + min(gl + k * lpr, nvec - 1));  // clamped, branch-free
}

template <int VPL>
__device__ __forceinline__ void scale_grad(float fl, bool mean, float4 (&x)[VPL]) {
  if (!mean) return;
#pragma unroll
  for (int k = 0; k < VPL; ++k) x[k] = f4_div(x[k], fl);
}

template <int VPL>
__device__ __forceinline__ void add_into(float4 (&acc)[VPL], const float4 (&x)[VPL]) {
#pragma unroll
  for (int k = 0; k < VPL; ++k) acc[k] = f4_add(acc[k], x[k]);
}

// ---- short segments (<= 32 occurrences), register path ----------------------------------
// A warp owns 32 segments — lane l holds segment l's record and first two bags — then its
// lane groups update the segments R at a time (weights/state + gradient rows in flight
// together). The bags come from the warp's sorted shared-memory copy (stage_short_bags).
template <int OPT, int LPR, int VPL>
__device__ __forceinline__ void short_reg(const BwdArgs& a, uint64_t warp, uint64_t n_warps, uint32_t* sbag) {
  constexpr int G = 32 / LPR;  // lane groups (segment streams) per warp
  // segments in flight per group (register budget). Two half-warp groups (dim 64) keep 2 each
  // at 3 CTAs/SM: 4 each needed 128 registers and held the kernel at 2 CTAs/SM (config 3:
  // 0.668 -> 0.602 ms per step, profiles/round2)
  constexpr int R = LPR == 16 ? 2 : (VPL >= 4 ? 1 : 4 / VPL);
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR;
  const uint64_t S = *a.short_alloc >> 32;
  const bool mean = a.bag_len != nullptr;
  for (uint64_t u0 = warp * 32; u0 < S; u0 += n_warps * 32) {
    const uint64_t u = u0 + lane;
    uint32_t first = 0, len = 0, row = 0, b0 = 0, b1 = 0, slot = 0;
    float f0 = 1.f, f1 = 1.f;
    if (u < S) {
      const uint4 rec = a.short_rec[u];
      row = rec.x;
      first = rec.y;
      len = rec.z;
      slot = rec.w;
    }
    const uint32_t off = stage_short_bags(a, S, u0, first, len, sbag);
    if (len) {
      a.bt[slot] = make_uint2(kBtEmpty, 0xffffffffu);  // placement (previous kernels) is done with it
      b0 = sbag[off];
      if (len >= 2) b1 = sbag[off + 1];
      if (mean) {
        f0 = static_cast<float>(a.bag_len[b0]);
        if (len >= 2) f1 = static_cast<float>(a.bag_len[b1]);
      }
    }
    // group g handles segments g, g+G, ... of the 32, R at a time
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += G * R) {
      uint32_t s_len[R], s_off[R], s_row[R], s_b1[R];
      float s_f1[R];
      RowState<OPT, VPL> rs[R];
      float4 g[R][VPL], x[R][VPL];
#pragma unroll
      for (int r = 0; r < R; ++r) {  // every load of the R segments is issued here, unconditionally
        const uint32_t src = j0 + G * r + grp;
        s_len[r] = __shfl_sync(0xffffffffu, len, src);
        s_off[r] = __shfl_sync(0xffffffffu, off, src);
        s_row[r] = __shfl_sync(0xffffffffu, row, src);
        const uint32_t sb0 = __shfl_sync(0xffffffffu, b0, src);
        s_b1[r] = __shfl_sync(0xffffffffu, b1, src);
        const float sf0 = __shfl_sync(0xffffffffu, f0, src);
        s_f1[r] = __shfl_sync(0xffffffffu, f1, src);
        load_row<OPT, VPL>(a, s_len[r] ? s_row[r] : 0u, gl, LPR, rs[r]);
        load_grad<VPL>(a, sb0, gl, LPR, g[r]);
        load_grad<VPL>(a, s_b1[r], gl, LPR, x[r]);
        scale_grad<VPL>(sf0, mean, g[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // (LPR 16: both half-warps stay converged through the lockstep walk below)
        if (LPR != 16 && !s_len[r]) continue;
        if (s_len[r] >= 2) {
          scale_grad<VPL>(s_f1[r], mean, x[r]);
          add_into<VPL>(g[r], x[r]);
        }
        if constexpr (LPR == 32) {  // (narrower groups would diverge across segments of a warp)
          // occurrences 3..32: lane gl holds occurrence 2+gl's bag, then the warp streams the
          // rows 8 in flight, in order.
          const uint32_t rest = s_len[r] > 2 ? s_len[r] - 2 : 0;
          if (rest) {
            const uint32_t bl = gl < rest ? sbag[s_off[r] + 2 + gl] : 0u;
            const float fll = (mean && gl < rest) ? static_cast<float>(a.bag_len[bl]) : 1.f;
            constexpr int KF = VPL >= 8 ? 1 : 8 / VPL;  // rows in flight (register budget)
            for (uint32_t q0 = 0; q0 < rest; q0 += KF) {
              float4 y[KF][VPL];
              float fq[KF];
#pragma unroll
              for (int k = 0; k < KF; ++k) {
                const uint32_t q = q0 + k;
                const int src = static_cast<int>(q % 32);
                const uint32_t vl = __shfl_sync(0xffffffffu, bl, src);
                fq[k] = __shfl_sync(0xffffffffu, fll, src);
                load_grad<VPL>(a, q < rest ? vl : 0u, gl, LPR, y[k]);
              }
#pragma unroll
              for (int k = 0; k < KF; ++k) {
                if (q0 + k < rest) {
                  scale_grad<VPL>(fq[k], mean, y[k]);
                  add_into<VPL>(g[r], y[k]);
                }
              }
            }
          }
        } else if constexpr (LPR == 16) {
          // two segment streams per warp: both half-warps walk occurrences 3..32 in lockstep
          // (to the longer of their two segments, so the warp never diverges), 4 rows in
          // flight per half; lane gl holds occurrences 2+gl and 18+gl of its half's segment
          const uint32_t rest = s_len[r] > 2 ? s_len[r] - 2 : 0;
          const uint32_t rest_max = max(rest, __shfl_xor_sync(0xffffffffu, rest, 16));
          if (rest_max) {
            const uint32_t bl0 = gl < rest ? sbag[s_off[r] + 2 + gl] : 0u;
            const uint32_t bl1 = gl + 16 < rest ? sbag[s_off[r] + 18 + gl] : 0u;
            const float fl0 = (mean && gl < rest) ? static_cast<float>(a.bag_len[bl0]) : 1.f;
            const float fl1 = (mean && gl + 16 < rest) ? static_cast<float>(a.bag_len[bl1]) : 1.f;
            constexpr int KF = VPL >= 4 ? 1 : 4 / VPL;  // rows in flight per half (register budget)
            for (uint32_t q0 = 0; q0 < rest_max; q0 += KF) {
              float4 y[KF][VPL];
              float fq[KF];
#pragma unroll
              for (int k = 0; k < KF; ++k) {
                const uint32_t q = q0 + k;  // warp-uniform
                const int src = static_cast<int>(grp * 16 + (q % 16));
                const uint32_t vl = __shfl_sync(0xffffffffu, q < 16 ? bl0 : bl1, src);
                fq[k] = __shfl_sync(0xffffffffu, q < 16 ? fl0 : fl1, src);
                load_grad<VPL>(a, q < rest ? vl : 0u, gl, LPR, y[k]);
              }
#pragma unroll
              for (int k = 0; k < KF; ++k) {
                if (q0 + k < rest) {
                  scale_grad<VPL>(fq[k], mean, y[k]);
                  add_into<VPL>(g[r], y[k]);
                }
              }
            }
          }
        } else {
          for (uint32_t q = 2; q < s_len[r]; q += 2) {  // narrow rows: two rows in flight
            const uint32_t bq = sbag[s_off[r] + q];
            const bool two = q + 1 < s_len[r];
            const uint32_t bq1 = two ? sbag[s_off[r] + q + 1] : bq;
            float4 y[VPL], z[VPL];
            load_grad<VPL>(a, bq, gl, LPR, y);
            if (two) load_grad<VPL>(a, bq1, gl, LPR, z);
            scale_grad<VPL>(mean ? static_cast<float>(a.bag_len[bq]) : 1.f, mean, y);
            add_into<VPL>(g[r], y);
            if (two) {
              scale_grad<VPL>(mean ? static_cast<float>(a.bag_len[bq1]) : 1.f, mean, z);
              add_into<VPL>(g[r], z);
            }
          }
        }
        if (s_len[r]) update_store<OPT, VPL>(a, s_row[r], gl, LPR, rs[r], g[r]);
      }
    }
    __syncwarp();  // sbag is rewritten by the next iteration
  }
}

// ---- short segments on the bulk-copy engine ----------------------------------------------
// Same work as short_reg, staged through shared memory by cp.async.bulk: a warp takes 32
// segments (lane = segment), packs as many as fit into its smem buffer ("wave": a warp
// prefix sum over rows needed = weight + state rows + one gradient row per occurrence),
// every lane issues the bulk copies of its own segment's rows onto the warp's mbarrier,
// and only then does the warp walk the wave segment by segment (ordered sum from smem,
// fused optimizer, 128-bit stores). Bytes in flight no longer cost registers.
constexpr int kRedWarps = 4;
constexpr int kBagStage = 32 * kChunk;  // sorted bags of a warp's 32 short segments

template <int OPT, int VPL>
__device__ __forceinline__ void short_tma(const BwdArgs& a, uint64_t warp, uint64_t n_warps, float* s_buf,
                                          uint64_t* s_bar) {
  constexpr uint32_t NS = state_rows<OPT>();  // state rows staged with the weight row
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  const uint32_t D = a.dim, nvec = D / 4, row_bytes = D * 4, cap = a.tma_rows;
  float* buf = s_buf + size_t(w) * cap * D;
  float* scale = s_buf + size_t(kRedWarps) * cap * D + size_t(w) * cap;
  // two bag stages per warp: the next 32 segments' bags land (cp.async) while this wave's
  // rows are in flight
  uint32_t* sbag2 = reinterpret_cast<uint32_t*>(s_buf + size_t(kRedWarps) * cap * (D + 1)) + size_t(w) * 2 * kBagStage;
  const bool mean = a.bag_len != nullptr;
  if (lane == 0) {
    mbar_init(&s_bar[w], 1);
    mbar_fence_init();
  }
  __syncwarp();
  uint32_t phase = 0;
  const uint64_t S = *a.short_alloc >> 32;
  const uint64_t stride = n_warps * 32;
  uint4 rec = make_uint4(0, 0, 0, 0);
  if (warp * 32 + lane < S) rec = a.short_rec[warp * 32 + lane];
  if (warp * 32 < S) prefetch_short_bags(a, S, warp * 32, rec.y, rec.z, sbag2);
  uint32_t stage = 0;
  for (uint64_t u0 = warp * 32; u0 < S; u0 += stride, stage ^= 1) {
    const uint32_t row = rec.x, first = rec.y, len = rec.z, slot = rec.w;
    const uint64_t un = u0 + stride;  // the next 32 segments: records now, bags after the first wave's issue
    uint4 nrec = make_uint4(0, 0, 0, 0);
    if (un + lane < S) nrec = a.short_rec[un + lane];
    uint32_t* sbag = sbag2 + stage * kBagStage;
    cp_async_wait_all();
    __syncwarp();
    const uint32_t r0 = __shfl_sync(0xffffffffu, first, 0);
    sort_short_bags(first, len, r0, sbag);
    const uint32_t boff = first - r0;
    bool next_issued = false;
    if (len) a.bt[slot] = make_uint2(kBtEmpty, 0xffffffffu);  // placement (previous kernels) is done with it
    const uint32_t need = len ? 1 + NS + len : 0;
    uint32_t first_lane = 0;  // first lane (segment) of the current wave
    while (first_lane < 32) {
      const uint32_t r = lane >= first_lane ? need : 0u;
      const uint32_t incl = warp_incl_scan(r);
      const bool in_wave = lane >= first_lane && incl <= cap;
      const uint32_t wave_mask = __ballot_sync(0xffffffffu, in_wave);
      const uint32_t last = 31 - __clz(wave_mask);  // wave = lanes [first_lane, last]
      const uint32_t off = incl - r;
      const uint32_t total_rows = __shfl_sync(0xffffffffu, incl, last);
      if (lane == 0) mbar_arrive_expect_tx(&s_bar[w], total_rows * row_bytes);
      __syncwarp();
      if (in_wave && len) {
        float* dst = buf + size_t(off) * D;
        bulk_g2s(dst, a.W + uint64_t(row) * D, row_bytes, &s_bar[w]);
        if constexpr (NS >= 1) bulk_g2s(dst + D, a.S0 + uint64_t(row) * D, row_bytes, &s_bar[w]);
        if constexpr (NS >= 2) bulk_g2s(dst + 2 * D, a.S1 + uint64_t(row) * D, row_bytes, &s_bar[w]);
        for (uint32_t q = 0; q < len; ++q) {
          const uint32_t bq = sbag[boff + q];
          bulk_g2s(dst + (1 + NS + q) * D, a.dout + uint64_t(bq) * D, row_bytes, &s_bar[w]);
          if (mean) scale[off + 1 + NS + q] = static_cast<float>(a.bag_len[bq]);
        }
      }
      if (!next_issued) {  // the other stage was last read by the previous iteration (done)
        next_issued = true;
        if (un < S) prefetch_short_bags(a, S, un, nrec.y, nrec.z, sbag2 + (stage ^ 1) * kBagStage);
      }
      mbar_wait(&s_bar[w], phase);
      phase ^= 1;
      __syncwarp();  // the scale[] writes of other lanes
      // walk the wave in segment order
      for (uint32_t j = first_lane; j <= last; ++j) {
        const uint32_t jl = __shfl_sync(0xffffffffu, len, j);
        const uint32_t jo = __shfl_sync(0xffffffffu, off, j);
        const uint32_t jr = __shfl_sync(0xffffffffu, row, j);
        if (!jl) continue;
        const float4* seg = reinterpret_cast<const float4*>(buf + size_t(jo) * D);
        RowState<OPT, VPL> rs;
        float4 g[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const uint32_t v = min(lane + 32u * k, nvec - 1);
          rs.w[k] = seg[v];
          if constexpr (NS >= 1) rs.s[k] = seg[nvec + v];
          if constexpr (NS >= 2) rs.q[k] = seg[2 * nvec + v];
          g[k] = seg[(1 + NS) * nvec + v];
          if (mean) g[k] = f4_div(g[k], scale[jo + 1 + NS]);
        }
        for (uint32_t q = 1; q < jl; ++q) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const uint32_t v = min(lane + 32u * k, nvec - 1);
            float4 x = seg[(1 + NS + q) * nvec + v];
            if (mean) x = f4_div(x, scale[jo + 1 + NS + q]);
            g[k] = f4_add(g[k], x);
          }
        }
        update_store<OPT, VPL>(a, jr, lane, 32, rs, g);
      }
      __syncwarp();  // every lane is done reading the buffer before the next wave overwrites it
      first_lane = last + 1;
    }
    rec = nrec;
  }
}

// ---- short segments, register row stream -------------------------------------------------
// A warp takes 32 segments (lane j = segment j) and flattens their rows into ONE stream:
// segment j contributes [weight row, state rows, gradient rows in canonical order]. The
// stream is cut into sub-lists of <= kPipeList entries (whole segments), each built in a
// small shared-memory list (the gradient rows' bags are read from the segment CSR and
// sorted into canonical order on the way in; every entry carries its row's address, computed
// once by the lane that builds it — per-issue address arithmetic by the whole warp was 15% of
// the kernel's instructions). The warp then walks its sub-list U rows at a
// time: U 128-bit row loads in flight (lane l owns float4s l, l+32, ...: fully coalesced),
// then the ordered sums, the fused optimizer at each segment's last row, 128-bit stores.
// Latency is hidden by occupancy (small register and shared-memory footprint), not by a
// deep per-warp pipeline: a fully unrolled ring overflows the instruction cache.
constexpr uint32_t kPipeList = 128;  // entries per sub-list (>= 3 + kChunk: one whole segment)
static_assert(kPipeList >= 3 + kChunk, "a sub-list holds at least one whole short segment");


__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_sh(uint32_t smem_dst, const void* gsrc, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gsrc), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// A sub-list entry: the row's global address (computed once, by the lane that builds the
// entry, not per issue by the whole warp), its kind and flags, and an operand: the table row
// of a weight entry (the update's store target), the bag length of a gradient (mean).
struct PipeEntry {
  uint32_t lo, hi;   // source address
  uint32_t flags;    // kind (0 weight, 1/2 optimizer state, 3 gradient) | 4: segment's last row
  uint32_t aux;      // weight: row id; gradient: mean divisor (1 for sum)
};
__device__ __forceinline__ PipeEntry pipe_entry(const float* base, uint32_t row, uint32_t dim, uint32_t flags,
                                                uint32_t aux) {
  const uint64_t p = reinterpret_cast<uint64_t>(base + uint64_t(row) * dim);
  return PipeEntry{static_cast<uint32_t>(p), static_cast<uint32_t>(p >> 32), flags, aux};
}

// U rows per chunk, two chunk buffers per warp: chunk c+1's rows land (per-lane cp.async,
// 16 B each, 128-bit coalesced) while chunk c is summed from shared memory.
template <int OPT, int VPL, int U>
__device__ __forceinline__ void short_pipe(const BwdArgs& a, uint64_t warp, uint64_t n_warps, PipeEntry* list,
                                           float4* buf) {
  constexpr uint32_t NS = state_rows<OPT>();
  constexpr uint32_t HDR = 1u + NS;  // weight (gradient-only: the row id, nothing loaded) + state rows
  const uint32_t lane = lane_id();
  const uint32_t D = a.dim, nvec = D / 4;
  const bool mean = a.bag_len != nullptr;
  const uint32_t sbuf = smem_u32(buf) + lane * 16u;  // this lane's float4 of chunk buffer 0, row 0
  const uint64_t efp = l2_policy_evict_first();
  const uint64_t S = *a.short_alloc >> 32;
  // segments per warp pass: the whole list spread over every warp of the grid (a fixed 32
  // left a third of the warps idle on config 2 and the rest with 32-segment chains)
  const uint64_t spread = (S + n_warps - 1) / n_warps;
  const uint32_t per = spread < 1 ? 1u : spread > 32 ? 32u : static_cast<uint32_t>(spread);
  for (uint64_t u0 = warp * per; u0 < S; u0 += n_warps * per) {
    uint4 rec = make_uint4(0, 0, 0, 0);
    if (lane < per && u0 + lane < S) rec = a.short_rec[u0 + lane];
    const uint32_t row = rec.x, first = rec.y, len = rec.z, slot = rec.w;
    if (len) a.bt[slot] = make_uint2(kBtEmpty, 0xffffffffu);  // placement (previous kernels) is done with it
    uint32_t bag0 = len ? a.short_bag[first] : 0u;
    const uint32_t c = len ? HDR + len : 0u;
    const uint32_t incl = warp_incl_scan(c), excl = incl - c;
    uint32_t done = 0;  // lanes (segments) already streamed
    while (done < 32) {
      const uint32_t base = __shfl_sync(0xffffffffu, excl, done);
      const bool in = lane >= done && incl - base <= kPipeList;
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      const uint32_t j1 = 31 - __clz(m);
      const uint32_t T = __shfl_sync(0xffffffffu, incl, j1) - base;
      // build the sub-list: header rows + single gradients by their own lane ...
      if (in && len) {
        const uint32_t o = excl - base;
        list[o] = pipe_entry(a.W, row, D, 0u, row);
        if constexpr (NS >= 1) list[o + 1] = pipe_entry(a.S0, row, D, 1u, row);
        if constexpr (NS >= 2) list[o + 2] = pipe_entry(a.S1, row, D, 2u, row);
        if (len == 1) list[o + HDR] = pipe_entry(a.dout, bag0, D, 3u | 4u, mean ? a.bag_len[bag0] : 1u);
      }
      // ... longer segments' bags sorted into canonical order by the whole warp
      uint32_t multi = __ballot_sync(0xffffffffu, in && len >= 2);
      while (multi) {
        const int j = __ffs(multi) - 1;
        multi &= multi - 1;
        const uint32_t jl = __shfl_sync(0xffffffffu, len, j);
        const uint32_t jf = __shfl_sync(0xffffffffu, first, j);
        const uint32_t jo = __shfl_sync(0xffffffffu, excl, j) - base + HDR;
        const uint32_t b = lane < jl ? a.short_bag[jf + lane] : 0xffffffffu;
        uint32_t rank = 0;
        for (uint32_t q = 0; q < jl; ++q) {
          const uint32_t x = __shfl_sync(0xffffffffu, b, q);
          rank += (x < b || (x == b && q < lane)) ? 1u : 0u;
        }
        if (lane < jl)
          list[jo + rank] = pipe_entry(a.dout, b, D, 3u | (rank + 1 == jl ? 4u : 0u), mean ? a.bag_len[b] : 1u);
      }
      __syncwarp();
      auto issue_chunk = [&](uint32_t ch) {
        const uint32_t dst = sbuf + (ch & 1u) * (U * nvec * 16u);
        const uint32_t t0 = ch * U, n = min(uint32_t(U), T - t0);
        for (uint32_t k = 0; k < n; ++k) {
          const PipeEntry e = list[t0 + k];
          if (OPT == kOptGrad && (e.flags & 3u) == 0) continue;  // gradient-only: the row is written, never read
          const char* src = reinterpret_cast<const char*>((uint64_t(e.hi) << 32) | e.lo) + lane * 16u;
          const bool ef = a.grad_once && (e.flags & 3u) == 3u;
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (lane + 32u * v < nvec) {
              if (ef) cp_async16_sh(dst + k * nvec * 16u + v * 512u, src + v * 512, efp);
              else cp_async16_s(dst + k * nvec * 16u + v * 512u, src + v * 512);
            }
        }
        cp_async_commit();
      };
      const uint32_t nch = (T + U - 1) / U;
      issue_chunk(0);
      RowState<OPT, VPL> rs;
      float4 g[VPL];
      bool g0 = true;  // the next gradient row starts its segment's sum
      uint32_t cur_row = 0;
      for (uint32_t ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) {
          issue_chunk(ch + 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        const float4* xb = buf + (ch & 1u) * U * nvec;
        const uint32_t t0 = ch * U, n = min(uint32_t(U), T - t0);
        for (uint32_t k = 0; k < n; ++k) {
          const uint32_t flags = list[t0 + k].flags, aux = list[t0 + k].aux;
          const uint32_t kind = flags & 3u;
          float4 x[VPL];
#pragma unroll
          for (int v = 0; v < VPL; ++v) x[v] = xb[k * nvec + min(lane + 32u * v, nvec - 1)];
          if (kind == 0) {
            cur_row = aux;
#pragma unroll
            for (int v = 0; v < VPL; ++v) rs.w[v] = x[v];
          } else if (kind == 1) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) rs.s[state_rows<OPT>() >= 1 ? v : 0] = x[v];
          } else if (kind == 2) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) rs.q[state_rows<OPT>() >= 2 ? v : 0] = x[v];
          } else {
            const float f = static_cast<float>(aux);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              const float4 gx = mean ? f4_div(x[v], f) : x[v];
              g[v] = g0 ? gx : f4_add(g[v], gx);
            }
            g0 = false;
            if (flags & 4u) {
              update_store<OPT, VPL>(a, cur_row, lane, 32, rs, g);
              g0 = true;
            }
          }
        }
        __syncwarp();  // this buffer is refilled two chunks from now
      }
      done = j1 + 1;
    }
  }
}

// ---- long segments: the tree above level 1 ----------------------------------------------
// Level-1 chunk c of segment j is complete in partial[base_j + c]. The warp counts itself
// into its parent node; the last of the parent's (<= 32) children sums them in order into
// the parent, and so on up: the root's sum goes through the optimizer. Counters reset
// themselves when their node completes, so they are zero at the start of every call.
template <int OPT, int VW>
__device__ __forceinline__ void climb(const BwdArgs& a, uint32_t j, uint32_t c, uint32_t m, uint32_t row) {
  const uint32_t lane = lane_id(), nvec = a.dim / 4;
  const float* level = a.partial + uint64_t(__ldcg(a.long_base + j)) * a.dim;
  const uint32_t hb = __ldcg(a.long_hbase + j);
  uint32_t off = 0, idx = c, lm = m;
  while (true) {
    const uint32_t parent = idx / kChunk, nm = (lm + kChunk - 1) / kChunk;
    const uint32_t nch = min(static_cast<uint32_t>(kChunk), lm - parent * kChunk);
    // Arrival: __syncwarp orders every lane's partial stores before lane 0's acq_rel atomic
    // (release, cumulative); the last arriver's acquire + __syncwarp makes the siblings'
    // partials visible to the whole warp.
    __syncwarp();
    uint32_t old = 0;
    if (lane == 0) {
      uint32_t* cnt = a.node_cnt + hb + off + parent;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
      if (old == nch - 1) *cnt = 0;  // node complete: reset for the next call
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    __syncwarp();
    if (old != nch - 1) return;
    const float4* ch = reinterpret_cast<const float4*>(level) + uint64_t(parent) * kChunk * nvec;
    float4 g[VW];
#pragma unroll
    for (int k = 0; k < VW; ++k) {
      const uint32_t v = lane + 32u * k;
      g[k] = v < nvec ? __ldcg(ch + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    constexpr int RB = VW >= 4 ? 1 : 4 / VW;
    for (uint32_t q0 = 1; q0 < nch; q0 += RB) {
      float4 x[RB][VW];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const uint32_t v = lane + 32u * k;
          x[r][k] = (q0 + r < nch && v < nvec) ? __ldcg(ch + uint64_t(q0 + r) * nvec + v)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (q0 + r >= nch) break;
#pragma unroll
        for (int k = 0; k < VW; ++k) g[k] = f4_add(g[k], x[r][k]);
      }
    }
    if (nm == 1) {  // root: the segment's gradient
      RowState<OPT, VW> rs;
      load_row<OPT, VW>(a, row, lane, 32, rs);
      update_store<OPT, VW>(a, row, lane, 32, rs, g);
      return;
    }
    float4* dst = reinterpret_cast<float4*>(a.partial2 + uint64_t(hb + off + parent) * a.dim);
#pragma unroll
    for (int k = 0; k < VW; ++k) {
      const uint32_t v = lane + 32u * k;
      if (v < nvec) __stcg(dst + v, g[k]);
    }
    level = a.partial2 + uint64_t(hb + off) * a.dim;
    off += nm;
    idx = parent;
    lm = nm;
  }
}

// ---- long segments: level-1 chunk partials -----------------------------------------------
// One warp per 32-occurrence chunk; its bags are loaded in one coalesced access, then the
// rows stream through G lane groups (G rows per instruction, RB instructions in flight) and
// are added in order (row q lives in group q % G; the running sum is kept replicated in
// every group). Runs after the grid barrier: the task lists are complete.
template <int OPT, int LPR, int VPL>
__device__ __forceinline__ void long_phase(const BwdArgs& a, uint64_t warp, uint64_t n_warps) {
  constexpr int G = 32 / LPR;
  // x G rows in flight (occupancy does the rest); full-warp rows of 128 floats keep 8
  constexpr int RB = VPL >= 4 ? 1 : (VPL == 2 ? 2 : (G == 1 ? 8 : 4));
  constexpr int VW = LPR == 32 ? VPL : 1;  // warp-wide layout of the same row (LPR < 32 <=> nvec <= 32)
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = a.dim / 4;
  const bool mean = a.bag_len != nullptr;
  const uint64_t T = *a.long_chunks;
  const uint32_t* lbag = (radix_passes_run(*a.n_long, a.long_passes) & 1) ? a.lval_b : a.lval;
  for (uint64_t t = warp; t < T; t += n_warps) {
    const uint32_t j = a.task_long[t];
    const uint32_t c = static_cast<uint32_t>(t) - a.long_base[j];
    if (c == 0 && lane == 0) a.bt[a.long_ent[j]] = make_uint2(kBtEmpty, 0xffffffffu);  // the entry's last reader
    const uint32_t s0 = a.long_start[j], e = s0 + a.long_len[j];
    const uint32_t s = s0 + c * kChunk;
    const uint32_t n = min(static_cast<uint32_t>(kChunk), e - s);
    const uint32_t my_bag = lane < n ? lbag[s + lane] : 0u;
    const float my_f = (mean && lane < n) ? static_cast<float>(a.bag_len[my_bag]) : 1.f;
    float4 acc[VPL];
    for (uint32_t q0 = 0; q0 < n; q0 += G * RB) {  // n is warp-uniform
      float4 x[RB][VPL];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const uint32_t q = q0 + r * G + grp;
        const uint32_t b = __shfl_sync(0xffffffffu, my_bag, q & 31);
        const float f = __shfl_sync(0xffffffffu, my_f, q & 31);
        if (q < n) {
          load_grad<VPL>(a, b, gl, LPR, x[r]);
          scale_grad<VPL>(f, mean, x[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const uint32_t q = q0 + r * G + h;
          if (q >= n) break;
          float4 y[VPL];
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            if (G == 1) {
              y[k] = x[r][k];
            } else {
              const int srcl = h * LPR + gl;
              y[k].x = __shfl_sync(0xffffffffu, x[r][k].x, srcl);
              y[k].y = __shfl_sync(0xffffffffu, x[r][k].y, srcl);
              y[k].z = __shfl_sync(0xffffffffu, x[r][k].z, srcl);
              y[k].w = __shfl_sync(0xffffffffu, x[r][k].w, srcl);
            }
            acc[k] = (q == 0) ? y[k] : f4_add(acc[k], y[k]);
          }
        }
      }
    }
    if (grp == 0) {
      float4* p = reinterpret_cast<float4*>(a.partial + t * a.dim);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const uint32_t v = gl + k * LPR;
        if (v < nvec) __stcg(p + v, acc[k]);
      }
    }
    climb<OPT, VW>(a, j, c, (e - s0 + kChunk - 1) / kChunk, a.long_row[j]);
  }
}

// ---- kernels ------------------------------------------------------------------------------
// Short segments reduced + updated.
template <int OPT, int LPR, int VPL, bool TMA>
__global__ void __launch_bounds__(TMA ? kRedWarps * 32 : 256,
                                  TMA ? 1 : (OPT == HPS_OPT_ADAM ? 2 : 3))
    k_reduce_short(BwdArgs a) {
  extern __shared__ __align__(128) float s_dyn[];  // TMA: [kRedWarps][cap][dim] rows, scales, bags
  __shared__ __align__(8) uint64_t s_bar[kRedWarps];
  pdl_wait();
  pdl_launch_dependents();
  // the short segments' batch-table entries are reset by this kernel: the slot no longer holds
  // an unconsumed record (counts[5], set by k_dedup / k_count_flat, read by their resets)
  if (blockIdx.x == 0 && threadIdx.x == 0) const_cast<uint64_t*>(a.counts)[5] = 0;
  const uint64_t wpb = blockDim.x >> 5;
  const uint64_t warp = uint64_t(blockIdx.x) * wpb + (threadIdx.x >> 5);
  const uint64_t n_warps = uint64_t(gridDim.x) * wpb;
  trace_begin(kTrReduce);
  if constexpr (TMA) {
    short_tma<OPT, VPL>(a, warp, n_warps, s_dyn, s_bar);
  } else {
    short_reg<OPT, LPR, VPL>(a, warp, n_warps, reinterpret_cast<uint32_t*>(s_dyn) + (threadIdx.x >> 5) * kBagStage);
  }
  trace_end(kTrReduce);
}

// Short segments reduced + updated through the register-pipelined row stream (dim 128..256).
constexpr int kPipeBlock = 256;
template <int OPT, int VPL, int U>
__global__ void __launch_bounds__(kPipeBlock, VPL >= 2 ? 2 : (OPT == HPS_OPT_SGD ? 4 : 3)) k_reduce_pipe(BwdArgs a) {
  extern __shared__ __align__(16) float4 s_rows[];  // per warp: 2 chunk buffers of U rows
  __shared__ PipeEntry s_list[kPipeBlock / 32][kPipeList];
  pdl_wait();
  pdl_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x == 0) const_cast<uint64_t*>(a.counts)[5] = 0;  // (as k_reduce_short)
  const uint64_t wpb = blockDim.x >> 5;
  const uint64_t warp = uint64_t(blockIdx.x) * wpb + (threadIdx.x >> 5);
  const uint64_t n_warps = uint64_t(gridDim.x) * wpb;
  const uint32_t w = threadIdx.x >> 5;
  trace_begin(kTrReduce);
  short_pipe<OPT, VPL, U>(a, warp, n_warps, s_list[w], s_rows + size_t(w) * 2 * U * (a.dim / 4));
  trace_end(kTrReduce);
}

// Long segments: chunk partials + the last-arriver tree + optimizer, at full occupancy
// (this part is a latency-bound gather stream).
template <int OPT, int LPR, int VPL>
__global__ void __launch_bounds__(256, VPL >= 4 ? 2 : (LPR == 32 ? 3 : 4)) k_long(BwdArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  trace_begin(kTrLong);
  long_phase<OPT, LPR, VPL>(a, warp, n_warps);
  trace_end(kTrLong);
}

__global__ void k_bt_used(const uint2* bt, uint64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    c += (bt[i].x != kBtEmpty || bt[i].y != 0xffffffffu) ? 1ull : 0ull;
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

__global__ void k_copy_counted(const uint32_t* __restrict__ src, const uint64_t* count, uint32_t* __restrict__ dst) {
  const uint64_t n = *count;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_unique_count(const unsigned long long* short_alloc, const uint32_t* n_long, uint64_t* count_out) {
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) *count_out = (*short_alloc >> 32) + *n_long;
}

// Rows updated by the last backward (short + long segments), unsorted; count -> *count_out.
__global__ void k_unique_rows(const uint4* short_rec, const unsigned long long* short_alloc, const uint32_t* long_row,
                              const uint32_t* n_long, uint32_t* out, uint64_t* count_out) {
  const uint64_t S = *short_alloc >> 32, L = *n_long;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_out = S + L;
  for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < S + L; u += uint64_t(gridDim.x) * blockDim.x)
    out[u] = u < S ? short_rec[u].x : long_row[u - S];
}

// Short segments on `st` (main), long segments on `side` — disjoint rows, run side by side.
template <int OPT, int LPR, int VPL, bool TMA>
int launch_backward_v(const BwdArgs& a, cudaStream_t st, cudaStream_t side, size_t smem, int grid, int long_grid) {
  auto kern = k_reduce_short<OPT, LPR, VPL, TMA>;
  constexpr int block = TMA ? kRedWarps * 32 : 256;
  static std::atomic<uint64_t> attr{0};
  HPSG_CUDA(once_per_device(attr, [&]() -> cudaError_t {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) return e;
    if (cudaError_t e = prefer_max_smem(kern)) return e;
    return prefer_max_smem(k_long<OPT, LPR, VPL>);
  }));
  HPSG_CUDA(launch_k(false, k_long<OPT, LPR, VPL>, long_grid, 256, 0, side, a));  // first after a join
  HPSG_CUDA(launch_k(false, kern, grid, block, smem, st, a));
  return HPS_GPU_OK;
}

template <int OPT, int VPL, int U>
int launch_backward_pipe(const BwdArgs& a, cudaStream_t st, cudaStream_t side, int long_grid, uint64_t nk) {
  auto kern = k_reduce_pipe<OPT, VPL, U>;
  static std::atomic<uint64_t> attr{0};
  const size_t smem = size_t(kPipeBlock / 32) * 2 * U * a.dim * sizeof(float);
  HPSG_CUDA(once_per_device(attr, [&]() -> cudaError_t {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024)) return e;
    if (cudaError_t e = prefer_max_smem(kern)) return e;
    return prefer_max_smem(k_long<OPT, 32, VPL>);
  }));
  int per_sm = 0;
  HPSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPipeBlock, smem));
  if (const char* e = std::getenv("HPS_GPU_PIPE_CTAS")) per_sm = std::max(1, std::atoi(e));  // A/B knob
  const int grid = static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>((nk + kPipeBlock - 1) / kPipeBlock, uint64_t(kNumSMs) * std::max(1, per_sm))));
  HPSG_CUDA(launch_k(false, k_long<OPT, 32, VPL>, long_grid, 256, 0, side, a));  // first after a join
  HPSG_CUDA(launch_k(false, kern, grid, kPipeBlock, smem, st, a));
  return HPS_GPU_OK;
}

// Lanes per row stream so that a lane holds VPL = ceil(nvec / LPR) float4 of a row.
template <int OPT>
int launch_backward(const BwdArgs& a, cudaStream_t st, cudaStream_t side, bool tma, size_t smem, int g, int lg,
                    uint32_t nvec) {
  if (tma) {
    if (nvec > 32) return launch_backward_v<OPT, 32, 2, true>(a, st, side, smem, g, lg);
    return launch_backward_v<OPT, 32, 1, true>(a, st, side, smem, g, lg);
  }
  if (nvec > 128) return launch_backward_v<OPT, 32, 8, false>(a, st, side, smem, g, lg);
  if (nvec > 64) return launch_backward_v<OPT, 32, 4, false>(a, st, side, smem, g, lg);
  if (nvec > 32) return launch_backward_v<OPT, 32, 2, false>(a, st, side, smem, g, lg);
  if (nvec == 32) return launch_backward_v<OPT, 32, 1, false>(a, st, side, smem, g, lg);
  if (nvec > 16) return launch_backward_v<OPT, 16, 2, false>(a, st, side, smem, g, lg);
  if (nvec == 16) return launch_backward_v<OPT, 16, 1, false>(a, st, side, smem, g, lg);
  if (nvec > 8) return launch_backward_v<OPT, 8, 2, false>(a, st, side, smem, g, lg);
  if (nvec == 8) return launch_backward_v<OPT, 8, 1, false>(a, st, side, smem, g, lg);
  if (nvec > 4) return launch_backward_v<OPT, 4, 2, false>(a, st, side, smem, g, lg);
  if (nvec == 4) return launch_backward_v<OPT, 4, 1, false>(a, st, side, smem, g, lg);
  if (nvec > 2) return launch_backward_v<OPT, 2, 2, false>(a, st, side, smem, g, lg);
  if (nvec == 2) return launch_backward_v<OPT, 2, 1, false>(a, st, side, smem, g, lg);
  return launch_backward_v<OPT, 1, 1, false>(a, st, side, smem, g, lg);
}

BwdArgs base_args(hps_gpu_table t) {
  const BwdZero zl = bwd_zero_layout(t->last_n_keys_host);
  uint32_t* z = t->ws_zero;
  BwdArgs a{};
  a.counts = t->ws_counts;
  a.occ_row = t->ws_rows_a;
  a.occ_rank = t->ws_rank;
  a.lead = t->ws_lead;
  a.occ_bag = t->last_multi ? t->ws_occ_bag : nullptr;
  a.occ_ent = t->ws_occ_ent;
  a.bt = t->ws_bt;
  a.bt_mask = t->bt_mask;
  a.row_absent = t->row_absent;
  a.short_alloc = reinterpret_cast<unsigned long long*>(z);
  a.short_rec = t->ws_short_rec;
  a.short_bag = t->ws_short_bag;
  a.long_alloc = reinterpret_cast<unsigned long long*>(z + 8);
  a.n_long = z + 9;
  a.higher_total = z + 3;
  a.long_occ = reinterpret_cast<unsigned long long*>(z + 4);
  a.long_chunks = reinterpret_cast<unsigned long long*>(z + 6);
  a.long_row = t->ws_long_row;
  a.long_ent = t->ws_long_ent;
  a.long_len = t->ws_long_len;
  a.long_start = t->ws_long_start;
  a.long_hist = z + zl.sort;  // (radix_sort workspace layout: the histograms come first)
  a.long_passes = bwd_long_passes(t->last_n_keys_host);
  a.lkey = t->ws_lkey_a;
  a.lval = t->ws_lval_a;
  a.lval_b = t->ws_lval_b;
  a.bag_len = (t->last_multi && t->last_combiner == HPS_COMBINER_MEAN) ? t->ws_bag_len : nullptr;
  a.dim = t->dim;
  a.n_slots = t->n_slots;
  a.long_base = t->ws_long_base;
  a.task_long = t->ws_task_long;
  a.partial = t->ws_partial;
  a.partial2 = t->ws_partial2;
  a.long_hbase = t->ws_long_hbase;
  a.node_cnt = t->ws_node_cnt;
  a.grad_once = !t->last_multi;
  (void)zl;
  return a;
}

}  // namespace

namespace {
std::atomic<uint64_t> g_dedup_attr{0};
cudaError_t dedup_attributes() {
  return once_per_device(g_dedup_attr, []() -> cudaError_t {
    for (auto kern : {k_dedup<512, 8>, k_dedup<1024, 4>})
      if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kDedupHash * 4))
        return e;
    for (cudaError_t e : {prefer_max_smem(k_dedup<512, 8>), prefer_max_smem(k_dedup<1024, 4>),
                          prefer_max_smem(k_count_flat), prefer_max_smem(k_alloc_flat),
                          prefer_max_smem(k_scan<PlaceOp>), prefer_max_smem(k_radix_hist), prefer_max_smem(k_radix_pass)})
      if (e) return e;
    return cudaSuccess;
  });
}
}  // namespace

// Which dedup a table runs: the persistent kernel (one CTA per SM, shared-memory
// aggregation per CTA chunk: Zipf-hot rows take one global atomic per CTA) when one of its
// CTAs fits every SM of this device, else the flat three-kernel dedup (no grid barrier, so
// no co-residency requirement: MIG slices, smaller parts). HPS_GPU_DEDUP=flat|persistent
// forces one (A/B). Measured on config 2/3/5 (profiles/round2): persistent <= flat on every
// config; config 3 (Zipf multi-hot) 0.66 vs 0.70 ms.
int hpsg::choose_dedup(bool* flat_out) {
  HPSG_CUDA(dedup_attributes());
  int per_sm = 0;
  int per_sm_wide = 0;
  HPSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dedup<512, 8>, 512, size_t(2) * kDedupHash * 4));
  HPSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_wide, k_dedup<1024, 4>, 1024,
                                                          size_t(2) * kDedupHash * 4));
  per_sm = std::min(per_sm, per_sm_wide);
  bool flat = per_sm < 1;
  if (const char* e = std::getenv("HPS_GPU_DEDUP")) {
    if (std::strcmp(e, "flat") == 0) flat = true;
    if (std::strcmp(e, "persistent") == 0) {
      if (per_sm < 1) {
        set_last_error("k_dedup (persistent, grid barriers) cannot keep one CTA resident per SM on this device");
        return HPS_GPU_E_NO_DEVICE;
      }
      flat = false;
    }
  }
  *flat_out = flat;
  return HPS_GPU_OK;
}

// K4a-K4d on the table's side stream, right after the training probe (table.cu
// fork_dedup): they need only the occurrence record, so they overlap the pooling.
int hpsg::launch_dedup(hps_gpu_table t, cudaStream_t st) {
  const bool pdl = t->ctx->pdl;
  const uint64_t nk = t->last_n_keys_host;
  const BwdZero zl = bwd_zero_layout(nk);
  uint32_t* z = t->ws_zero;
  const BwdArgs a = base_args(t);
  // K4a-c: counts, allocation, placement (first on this stream after the fork: a plain launch)
  if (t->flat_dedup) {
    HPSG_CUDA(dedup_attributes());
    const uint64_t tiles = std::max<uint64_t>(1, scan_tiles(nk));
    HPSG_CUDA(launch_k(false, k_count_flat, grid_for(nk, 256, 1 << 30), 256, 0, st, a));
    HPSG_CUDA(launch_k(pdl, k_alloc_flat, grid_for((nk + kAllocIPT - 1) / kAllocIPT, 256, 1 << 30), 256, 0, st, a));
    uint64_t* status = reinterpret_cast<uint64_t*>(z + zl.place);
    HPSG_CUDA(launch_k(pdl, k_scan<PlaceOp>, static_cast<unsigned>(tiles), kScanBlock, 0, st, PlaceOp{a}, status,
                       reinterpret_cast<uint32_t*>(status + tiles)));
  } else {
    HPSG_CUDA(dedup_attributes());

    uint64_t per_cta = 256;  // occurrences per CTA below a full grid (more CTAs: shorter chains; cfg1 64.9 -> 63.4 us)
    if (const char* e = std::getenv("HPS_GPU_DEDUP_PER_CTA")) per_cta = std::max(64, std::atoi(e));  // A/B knob
    // at most one CTA per SM of THIS device (a MIG slice or a smaller part has fewer): the
    // grid barriers need every CTA resident, which one per SM guarantees (table create
    // checked that one k_dedup CTA fits an SM)
    const uint64_t sms = static_cast<uint64_t>(t->ctx->num_sms);
    const int g = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(sms, (nk + per_cta - 1) / per_cta)));
    // A plain launch (a cooperative one would not start beside the pooling): co-residency of
    // the grid barriers holds by construction — at most one CTA per SM, and every kernel it
    // can share the SMs with (the pooling) runs to completion without waiting on it.
    // shape: one-hot batches 1024 x 4 (short per-CTA chunks: more warps in flight), multi-hot
    // 512 x 8 (long chunks); HPS_GPU_DEDUP_SHAPE=512|1024 forces one (A/B)
    bool wide = !t->last_multi;
    if (const char* e = std::getenv("HPS_GPU_DEDUP_SHAPE")) wide = std::atoi(e) == 1024;
    if (wide)
      HPSG_CUDA(launch_k(false, k_dedup<1024, 4>, g, 1024, size_t(2) * kDedupHash * 4, st, a, z + zl.coop));
    else
      HPSG_CUDA(launch_k(false, k_dedup<512, 8>, g, 512, size_t(2) * kDedupHash * 4, st, a, z + zl.coop));
  }
  // the short segments are complete: the short reduce may start (backward_update joins here);
  // the long segments' sort and registration continue on this stream
  if (st == t->side) HPSG_CUDA(cudaEventRecord(t->ev_join, st));
  // K4c: stable sort of the long list by segment id (canonical order within each segment)
  {
    const int passes = bwd_long_passes(nk);
    const uint64_t stiles = sort_tiles(nk);
    uint32_t* hist = z + zl.sort;
    uint32_t* stick = hist + 4 * 256;
    uint32_t* status = stick + 4;
    const auto* d_n = reinterpret_cast<const uint64_t*>(a.long_occ);
    // (the digit histograms were counted at allocation: register_long)
    const uint32_t* kin = t->ws_lkey_a;
    const uint32_t* vin = t->ws_lval_a;
    bool in_b = false;
    for (int p = 0; p < passes; ++p) {
      uint32_t* kout = in_b ? t->ws_lkey_a : t->ws_lkey_b;
      uint32_t* vout = in_b ? t->ws_lval_a : t->ws_lval_b;
      HPSG_CUDA(launch_k(pdl, k_radix_pass, static_cast<unsigned>(stiles), kSortBlock, 0, st, kin, vin, kout, vout, d_n,
                         8 * p, static_cast<const uint32_t*>(hist + 256 * p), status + size_t(p) * stiles * 256,
                         stick + p, static_cast<const uint32_t*>(a.n_long)));  // keys: segment ids < n_long
      kin = kout;
      vin = vout;
      in_b = !in_b;
    }
  }
  HPSG_CHECK_LAUNCH("backward dedup");
  return HPS_GPU_OK;
}

namespace {
// Mean combiner: each bag's gradient row divided by the bag's length ONCE (IEEE division,
// the oracle's g / len), instead of once per occurrence inside the reduces — on multi-hot
// batches every bag is read by ~hots segments, and the correctly rounded divide (reciprocal,
// refinement, range check) was a third of the long reduce's instructions on config 3.
__global__ void __launch_bounds__(256) k_scale_dout(const float4* __restrict__ dout, const uint32_t* __restrict__ bag_len,
                                                    uint64_t n_bags, uint32_t nvec, float4* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  trace_begin(kTrScale);
  // a streaming pass: four float4 loads (and their bags' lengths) in flight per thread
  constexpr int K = 4;
  const uint32_t sh = (nvec & (nvec - 1)) == 0 ? static_cast<uint32_t>(__ffs(nvec) - 1) : 32u;
  const uint64_t n = n_bags * nvec;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < n; b += K * stride) {
    float4 x[K];
    uint32_t len[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = b + k * stride;
      if (i < n) {
        x[k] = __ldg(dout + i);
        len[k] = __ldg(bag_len + (sh < 32 ? (i >> sh) : i / nvec));
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = b + k * stride;
      if (i < n) out[i] = f4_div(x[k], static_cast<float>(len[k]));
    }
  }
  trace_end(kTrScale);
}

// grads_out != nullptr: gradient-only mode (kOptGrad) — per-row sums into grads_out
// [total_rows x dim] (rows not in the batch untouched) and touched_out[row] = 1.
int backward_impl(hps_gpu_table t, const float* d_out, const hps_opt_params* opt, float* grads_out,
                  uint32_t* touched_out) {
  if (!t->have_train) {
    set_last_error("backward_update: no preceding lookup_pooled with HPS_LOOKUP_TRAIN");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!d_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const uint64_t nk = t->last_n_keys_host;
  // join the dedup forked by the training lookup; the long reduce runs on the side stream
  // (after this point of the main stream: the pooling has read the rows, d_out is ready)
  if (t->dedup_deferred) {
    if (int s = launch_dedup(t, st)) return s;
    t->dedup_deferred = false;
  }
  BwdArgs a = base_args(t);
  a.dout = d_out;
  if (a.bag_len) {  // mean: the scaled gradient rows, once per bag (the workspace is allocated on
                    // the first such backward outside stream capture; inside one, the reduces divide)
    if (!t->ws_dscale && capture_id(st) == 0) HPSG_CUDA(cudaMalloc(&t->ws_dscale, t->max_bags * t->dim * sizeof(float)));
    if (t->ws_dscale) {
      const uint32_t nv = t->dim / 4;
      HPSG_CUDA(launch_k(t->ctx->pdl, k_scale_dout, grid_for(uint64_t(t->pre_n_bags) * nv / 4, 256, kNumSMs * 8), 256, 0,
                         st, reinterpret_cast<const float4*>(d_out), static_cast<const uint32_t*>(a.bag_len),
                         uint64_t(t->pre_n_bags), nv, reinterpret_cast<float4*>(t->ws_dscale)));
      a.dout = t->ws_dscale;
      a.bag_len = nullptr;  // (the reduces now sum rows as given)
    }
  }
  HPSG_CUDA(cudaEventRecord(t->ev_bwd, st));
  HPSG_CUDA(cudaStreamWaitEvent(t->side, t->ev_bwd, 0));
  if (t->dedup_pending) {
    HPSG_CUDA(wait_recorded(st, t->ev_join, t->pre_capture));
    t->dedup_pending = false;
  }
  const bool grad_only = grads_out != nullptr;
  a.W = grad_only ? grads_out : t->d_w;
  a.S0 = grad_only ? nullptr : t->d_s0;
  a.S1 = grad_only ? nullptr : t->d_s1;
  a.touched = touched_out;
  a.optimizer = t->optimizer;
  if (opt) a.opt = *opt;

  const uint32_t nvec = t->dim / 4;
  // K4e + K5: short segments (reduce fused with the optimizer), then the long segments'
  // chunk partials + tree + optimizer.
  uint32_t tma_min_dim = 128;
  if (const char* e = std::getenv("HPS_GPU_TMA_MIN_DIM")) tma_min_dim = std::max(16, std::atoi(e));  // A/B knob
  const bool tma = t->dim >= tma_min_dim && t->dim <= 256 && !t->no_tma;  // narrower rows: the register path wins
  size_t smem = 0;
  int grid = 0;
  if (tma) {
    a.tma_rows = 38;  // 2 CTAs/SM (rows + two bag stages per warp) with room for the long chain beside them
    if (const char* e = std::getenv("HPS_GPU_TMA_ROWS")) a.tma_rows = std::max(36, std::atoi(e));  // A/B knob
    smem = size_t(kRedWarps) * a.tma_rows * (t->dim + 1) * sizeof(float) + size_t(kRedWarps) * 2 * kBagStage * 4;
    int waves = 2;  // CTAs per SM of the grid (2 resident per SM): 2 = a single resident wave
    if (const char* e = std::getenv("HPS_GPU_RED_WAVES")) waves = std::max(1, std::atoi(e));  // A/B knob
    grid = static_cast<int>(
        std::max<uint64_t>(1, std::min<uint64_t>((nk + 32 * kRedWarps - 1) / (32 * kRedWarps), kNumSMs * waves)));
  } else {
    smem = size_t(8) * kBagStage * 4;
    grid = grid_for((nk + 31) / 32 * 32, 256, kNumSMs * 16);
  }
  const int long_grid = grid_for((nk / kChunk + 2) * 32, 256, kNumSMs * 16);
  int s = HPS_GPU_OK;
  int red_mode = 2;  // 0 register path, 1 bulk-copy waves, 2 register-pipelined row stream
  if (const char* e = std::getenv("HPS_GPU_RED_MODE")) red_mode = std::atoi(e);  // A/B knob
  if (tma && red_mode == 2) {
    const bool two = nvec > 32;
    auto pipe = [&](auto opt_tag) -> int {
      constexpr int O = decltype(opt_tag)::value;
      static const int uu = std::getenv("HPS_GPU_PIPE_U") ? std::atoi(std::getenv("HPS_GPU_PIPE_U")) : 4;  // A/B knob
      if (two) return uu == 16 ? launch_backward_pipe<O, 2, 8>(a, st, t->side, long_grid, nk)
                                : launch_backward_pipe<O, 2, 4>(a, st, t->side, long_grid, nk);
      if (uu == 16) return launch_backward_pipe<O, 1, 16>(a, st, t->side, long_grid, nk);
      if (uu == 4) return launch_backward_pipe<O, 1, 4>(a, st, t->side, long_grid, nk);
      return launch_backward_pipe<O, 1, 8>(a, st, t->side, long_grid, nk);
    };
    if (grad_only) s = pipe(std::integral_constant<int, kOptGrad>{});
    else if (t->optimizer == HPS_OPT_SGD) s = pipe(std::integral_constant<int, HPS_OPT_SGD>{});
    else if (t->optimizer == HPS_OPT_ADAGRAD) s = pipe(std::integral_constant<int, HPS_OPT_ADAGRAD>{});
    else s = pipe(std::integral_constant<int, HPS_OPT_ADAM>{});
    if (s) return s;
    HPSG_CHECK_LAUNCH("backward");
    HPSG_CUDA(cudaEventRecord(t->ev_join2, t->side));
    HPSG_CUDA(cudaStreamWaitEvent(st, t->ev_join2, 0));
    t->have_train = false;
    t->have_unique = true;
    return HPS_GPU_OK;
  }
  if (grad_only) s = launch_backward<kOptGrad>(a, st, t->side, tma, smem, grid, long_grid, nvec);
  else if (t->optimizer == HPS_OPT_SGD) s = launch_backward<HPS_OPT_SGD>(a, st, t->side, tma, smem, grid, long_grid, nvec);
  else if (t->optimizer == HPS_OPT_ADAGRAD)
    s = launch_backward<HPS_OPT_ADAGRAD>(a, st, t->side, tma, smem, grid, long_grid, nvec);
  else s = launch_backward<HPS_OPT_ADAM>(a, st, t->side, tma, smem, grid, long_grid, nvec);
  if (s) return s;
  HPSG_CHECK_LAUNCH("backward");
  HPSG_CUDA(cudaEventRecord(t->ev_join2, t->side));
  HPSG_CUDA(cudaStreamWaitEvent(st, t->ev_join2, 0));
  t->have_train = false;  // one backward per training lookup (its zeroed workspace is now used)
  t->have_unique = true;
  return HPS_GPU_OK;
}

// Dense apply: warp per row, rows with touched[r] take the optimizer with grads[r].
template <int OPT, int VPL>
__global__ void __launch_bounds__(256) k_apply_grads(BwdArgs a, const float* __restrict__ grads,
                                                     const uint32_t* __restrict__ touched, uint64_t n_rows) {
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t lane = lane_id(), nvec = a.dim / 4;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = warp; r < n_rows; r += n_warps) {
    if (!touched[r]) continue;
    float4 g[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      g[k] = reinterpret_cast<const float4*>(grads + r * a.dim)[min(lane + 32u * k, nvec - 1)];
    RowState<OPT, VPL> rs;
    load_row<OPT, VPL>(a, static_cast<uint32_t>(r), lane, 32, rs);
    update_store<OPT, VPL>(a, static_cast<uint32_t>(r), lane, 32, rs, g);
  }
}

template <int OPT>
void launch_apply(const BwdArgs& a, cudaStream_t st, bool pdl, const float* grads, const uint32_t* touched,
                  uint64_t n_rows, uint32_t nvec) {
  const int grid = grid_for(n_rows * 32, 256, kNumSMs * 16);
  if (nvec > 128) launch_k(pdl, k_apply_grads<OPT, 8>, grid, 256, 0, st, a, grads, touched, n_rows);
  else if (nvec > 64) launch_k(pdl, k_apply_grads<OPT, 4>, grid, 256, 0, st, a, grads, touched, n_rows);
  else if (nvec > 32) launch_k(pdl, k_apply_grads<OPT, 2>, grid, 256, 0, st, a, grads, touched, n_rows);
  else launch_k(pdl, k_apply_grads<OPT, 1>, grid, 256, 0, st, a, grads, touched, n_rows);
}
}  // namespace

extern "C" {

int hps_gpu_backward_update(hps_gpu_table t, const float* d_out, const hps_opt_params* opt) {
  if (!t || !opt) return HPS_GPU_E_INVALID_ARGUMENT;
  if (t->dim != t->dim_io && d_out && t->have_train) {  // padded rows: widen the gradients first
    if (rows_widen(t->ws_io, t->dim, d_out, t->dim_io, t->pre_n_bags, t->ctx->stream) != cudaSuccess)
      return HPS_GPU_E_CUDA;
    d_out = t->ws_io;
  }
  return backward_impl(t, d_out, opt, nullptr, nullptr);
}

int hps_gpu_backward_reduce(hps_gpu_table t, const float* d_out, float* grads_out, uint32_t* touched_out) {
  if (t && t->dim != t->dim_io) {
    set_last_error("hybrid gradient path: needs dim % 4 == 0 (rows of this table are padded)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!t || !grads_out || !touched_out) return HPS_GPU_E_INVALID_ARGUMENT;
  return backward_impl(t, d_out, nullptr, grads_out, touched_out);
}

int hps_gpu_apply_grads(hps_gpu_table t, const float* grads, const uint32_t* touched, const hps_opt_params* opt) {
  if (t && t->dim != t->dim_io) {
    set_last_error("hybrid gradient path: needs dim % 4 == 0 (rows of this table are padded)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!t || !grads || !touched || !opt) return HPS_GPU_E_INVALID_ARGUMENT;
  if (t->f16) return HPS_GPU_E_DTYPE_MISMATCH;  // an F16 table is an inference table
  BwdArgs a{};
  a.dim = t->dim;
  a.W = t->d_w;
  a.S0 = t->d_s0;
  a.S1 = t->d_s1;
  a.optimizer = t->optimizer;
  a.opt = *opt;
  const uint32_t nvec = t->dim / 4;
  cudaStream_t st = t->ctx->stream;
  if (t->optimizer == HPS_OPT_SGD) launch_apply<HPS_OPT_SGD>(a, st, t->ctx->pdl, grads, touched, t->total_rows, nvec);
  else if (t->optimizer == HPS_OPT_ADAGRAD)
    launch_apply<HPS_OPT_ADAGRAD>(a, st, t->ctx->pdl, grads, touched, t->total_rows, nvec);
  else launch_apply<HPS_OPT_ADAM>(a, st, t->ctx->pdl, grads, touched, t->total_rows, nvec);
  HPSG_CHECK_LAUNCH("k_apply_grads");
  return HPS_GPU_OK;
}

// In-graph kernel timeline of the training step. mode 1: attach a zeroed
// trace buffer; 2: copy the kTraceSlots x {start_ns, end_ns} records to trace_host
// (2 * kTraceSlots u64; start = UINT64_MAX when the kernel did not run) and re-arm;
// 0: detach. Synchronises the device.
}  // extern "C"

namespace {
__global__ void k_stamp(int id) {
  trace_begin(id);
  trace_end(id);
}
}  // namespace

extern "C" {

int hps_gpu_debug_stamp(void* stream, int id) {
  if (id < 0 || id >= kTraceSlots) return HPS_GPU_E_INVALID_ARGUMENT;
  k_stamp<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(id);
  HPSG_CHECK_LAUNCH("k_stamp");
  return HPS_GPU_OK;
}

int hps_gpu_debug_trace(int mode, uint64_t* trace_host) {
  static TraceRec* buf = nullptr;
  constexpr size_t kRecs = size_t(kTraceSlots) * kTraceSMs;
  auto arm = [&]() -> cudaError_t {
    std::vector<TraceRec> init(kRecs, TraceRec{~0ull, 0ull});
    return cudaMemcpy(buf, init.data(), kRecs * sizeof(TraceRec), cudaMemcpyHostToDevice);
  };
  if (mode == 1) {
    if (!buf) HPSG_CUDA(cudaMalloc(&buf, kRecs * sizeof(TraceRec)));
    HPSG_CUDA(arm());
    HPSG_CUDA(trace_attach_tu(buf));
    HPSG_CUDA(hpsg::trace_attach_table(buf));
    return HPS_GPU_OK;
  }
  if (mode == 2) {
    if (!buf || !trace_host) return HPS_GPU_E_INVALID_ARGUMENT;
    HPSG_CUDA(cudaDeviceSynchronize());
    std::vector<TraceRec> per_sm(kRecs);
    HPSG_CUDA(cudaMemcpy(per_sm.data(), buf, kRecs * sizeof(TraceRec), cudaMemcpyDeviceToHost));
    for (int id = 0; id < kTraceSlots; ++id) {
      TraceRec r{~0ull, 0ull};
      for (int m = 0; m < kTraceSMs; ++m) {
        r.start = std::min(r.start, per_sm[size_t(id) * kTraceSMs + m].start);
        r.end = std::max(r.end, per_sm[size_t(id) * kTraceSMs + m].end);
      }
      trace_host[2 * id] = r.start;
      trace_host[2 * id + 1] = r.end;
    }
    HPSG_CUDA(arm());
    return HPS_GPU_OK;
  }
  if (mode == 0) {
    HPSG_CUDA(trace_attach_tu(nullptr));
    HPSG_CUDA(hpsg::trace_attach_table(nullptr));
    return HPS_GPU_OK;
  }
  return HPS_GPU_E_INVALID_ARGUMENT;
}

// Invariant check (tests): batch-table entries in use. Zero whenever no training record is
// pending (every backward and every counter reset empties what it used). Synchronises.
int hps_gpu_debug_batch_table_used(hps_gpu_table t, uint64_t* used_host) {
  if (!t || !used_host) return HPS_GPU_E_INVALID_ARGUMENT;
  unsigned long long* d = nullptr;
  HPSG_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  HPSG_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), t->ctx->stream));
  for (uint32_t k = 0; k < t->parked.size(); ++k) {  // every batch slot's table
    const BatchSlot& b = k == t->cur ? static_cast<const BatchSlot&>(*t) : t->parked[k];
    HPSG_CUDA(cudaStreamSynchronize(b.side));
    k_bt_used<<<grid_for(t->bt_mask + 1, 256, kNumSMs * 8), 256, 0, t->ctx->stream>>>(b.ws_bt, t->bt_mask + 1, d);
    HPSG_CHECK_LAUNCH("k_bt_used");
  }
  HPSG_CUDA(cudaStreamSynchronize(t->ctx->stream));
  unsigned long long v = 0;
  HPSG_CUDA(cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost));
  cudaFree(d);
  *used_host = v;
  return HPS_GPU_OK;
}

int hps_gpu_table_last_unique(hps_gpu_table t, uint64_t* count_out, uint32_t* unique_rows_out) {
  if (!t || !count_out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!t->have_unique) {
    set_last_error("last_unique: no backward since the last training lookup");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  cudaStream_t st = t->ctx->stream;
  const uint64_t nk = t->last_n_keys_host;
  const BwdArgs a = base_args(t);
  if (!unique_rows_out) {  // the count alone (the end-to-end step's result): one thread
    HPSG_CUDA(launch_k(true, k_unique_count, 1, 32, 0, st, static_cast<const unsigned long long*>(a.short_alloc),
                       static_cast<const uint32_t*>(a.n_long), count_out));
    return HPS_GPU_OK;
  }
  // unsorted rows into the (now free) long-list buffers, then an ascending radix sort
  k_unique_rows<<<grid_for(nk, 256, kNumSMs * 8), 256, 0, st>>>(t->ws_short_rec, a.short_alloc, t->ws_long_row,
                                                               a.n_long, t->ws_lkey_a, count_out);
  HPSG_CHECK_LAUNCH("k_unique_rows");
  if (!unique_rows_out) return HPS_GPU_OK;
  cudaError_t err = cudaSuccess;
  const bool in_b = radix_sort_pairs(st, t->ws_lkey_a, nullptr, t->ws_lval_a, t->ws_lkey_b, t->ws_lval_b, count_out,
                                     nk, t->sort_bits, t->ws_zero, &err);
  if (err != cudaSuccess) return cuda_status(err, "last_unique sort");
  // only the *count_out unique rows: the caller's buffer may be sized to the unique count
  k_copy_counted<<<grid_for(nk, 256, kNumSMs * 8), 256, 0, st>>>(in_b ? t->ws_lkey_b : t->ws_lkey_a, count_out,
                                                                  unique_rows_out);
  HPSG_CHECK_LAUNCH("k_copy_counted");
  return HPS_GPU_OK;
}

}  // extern "C"
