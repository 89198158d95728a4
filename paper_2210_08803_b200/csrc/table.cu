// table.cu — embedding table group: K2 index insert/find, K3 fused lookup+pool,
// K4 dedup + blocked segmented reduction, K5 fused sparse optimizers.
//
// HBM layout of one table group:
//   slots   [Σ_t cap_slots(t)] x 16 B   open-addressing key->row index, one power-of-two
//                                        region per table; home = key_hash(k) & mask
//                                        (proj/include/hps/hash.hpp:42-49)
//   weights [Σ_t row_cap(t) x dim] fp32 row slab; table t owns rows [row_base(t), +row_cap)
//   state0/1 same shape (AdaGrad accumulator / Adam m, v)
//   row_keys[Σ row_cap] u64            inverse index (export, dedup reporting)
// Row ids are assigned in order of first occurrence (oracle/oracle.cpp table_insert),
// so key->row is deterministic under parallel insert.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "primitives.cuh"
#include "table_internal.cuh"

using namespace hpsg;

namespace {

constexpr uint64_t kNoSlot = ~0ull;
constexpr uint64_t kPresent = ~1ull;  // key committed before this call; nothing to do (keys-only insert)
// keys-only insert that records a training batch (InsertRecord): a committed key's slot word
// is kPresentRow | its local row. Every value >= kPresentRow (this, kPresent, kNoSlot) names
// no slot claimed by the call.
constexpr uint64_t kPresentRow = 1ull << 62;

// A one-hot training record produced by the insert-on-miss pass itself (no separate probe):
// k_insert_finish writes each occurrence's global row (row_absent if the insert failed for
// it), the record's size, and clears the backward's zeroed words, as k_probe would.
struct InsertRecord {
  uint32_t* occ_row = nullptr;  // nullptr: not a training record
  uint64_t row_base = 0;
  uint32_t row_absent = 0;
  uint64_t* d_n = nullptr;
  uint32_t* zero = nullptr;
  uint32_t zero_words = 0;
};

// ---------------------------------------------------------------------------------
// K2: index probe helpers
// ---------------------------------------------------------------------------------
// Read-only probe (no concurrent writers: handles are externally synchronised).
__device__ __forceinline__ uint32_t probe_find(const Slot* __restrict__ slots, const TableDev& td, uint64_t key) {
  uint64_t idx = hps::key_hash(key) & td.slot_mask;
  const Slot* base = slots + td.slot_base;
  for (uint64_t p = 0; p <= td.slot_mask; ++p) {
    const Slot s = load_slot(base + idx);
    if (s.row == kRowEmpty) return kRowEmpty;
    if (s.key == key) return s.row;
    idx = (idx + 1) & td.slot_mask;
  }
  return kRowEmpty;
}

// Warp-cooperative probing (north_star (1)): G lanes examine G consecutive slots of an aligned
// window at once (one 16*G-byte coalesced load), ballot for the first match or empty slot in
// linear-probe order from the home slot — the same answer as probe_find. Kept as the measured
// alternative (hps_gpu_debug_find_variant): at load <= 0.5 the per-thread probe
// ends in ~1.5 slots, so the group's extra lanes are mostly wasted issue slots.
template <int G>
__device__ __forceinline__ uint32_t probe_find_coop(const Slot* __restrict__ slots, const TableDev& td, uint64_t key,
                                                    uint32_t gl, uint32_t gmask) {
  const uint64_t home = hps::key_hash(key) & td.slot_mask;
  const Slot* base = slots + td.slot_base;
  uint64_t w = home & ~uint64_t(G - 1);
  uint32_t skip = static_cast<uint32_t>(home - w);  // lanes before the home slot (first window only)
  for (uint64_t p = 0; p <= td.slot_mask; p += G) {
    const Slot s = load_slot(base + ((w + gl) & td.slot_mask));
    const bool valid = gl >= skip;
    const uint32_t hit = __ballot_sync(gmask, valid && s.key == key && s.row != kRowEmpty);
    const uint32_t emp = __ballot_sync(gmask, valid && s.row == kRowEmpty);
    const uint32_t sh = __ffs(gmask) - 1;  // the group's first lane
    const uint32_t h = hit >> sh, e = emp >> sh;
    if (h | e) {
      const int first = __ffs(h | e) - 1;
      if (!((h >> first) & 1u)) return kRowEmpty;
      return __shfl_sync(gmask, s.row, static_cast<int>(sh) + first);
    }
    w += G;
    skip = 0;
  }
  return kRowEmpty;
}

template <int G>
__global__ void k_find_coop(const Slot* __restrict__ slots, TableDev td, const uint64_t* __restrict__ keys, uint64_t n,
                            uint64_t* __restrict__ rows_out) {
  const uint32_t lane = lane_id(), gl = lane % G;
  const uint32_t gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane - gl);
  const uint64_t groups = (uint64_t(gridDim.x) * blockDim.x) / G;
  for (uint64_t i0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / G; i0 < n; i0 += groups) {
    const uint32_t r = probe_find_coop<G>(slots, td, keys[i0], gl, gmask);
    if (gl == 0) rows_out[i0] = r == kRowEmpty ? ~0ull : r;
  }
}

__global__ void k_find(const Slot* __restrict__ slots, TableDev td, const uint64_t* __restrict__ keys, uint64_t n,
                       uint64_t* __restrict__ rows_out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = probe_find(slots, td, keys[i]);
    rows_out[i] = r == kRowEmpty ? ~0ull : r;
  }
}

// Insert phase A: claim or find a slot for every occurrence (128-bit CAS gives an
// atomic snapshot of the slot, so no torn key/row reads); aux = min occurrence index.
// keys_only (no rows, no rows_out: insert-on-miss and plain bulk loads): an occurrence
// whose key was committed before the call needs no claim, no aux and no row work, so a
// read-only probe settles it (rows committed before the call cannot change during it).
__global__ void k_insert_claim(Slot* __restrict__ slots, TableDev td, const uint64_t* __restrict__ keys, uint64_t n,
                               uint64_t* __restrict__ ws_slot, uint32_t* __restrict__ abort_flag, uint32_t* status,
                               bool keys_only, const uint32_t* __restrict__ key_tables, uint32_t table,
                               bool record_rows) {
  if (*reinterpret_cast<volatile uint32_t*>(abort_flag)) return;
  trace_begin(kTrInsClaim);
  Slot* base = slots + td.slot_base;
  const Slot empty{0, kRowEmpty, kAuxNone};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (key_tables && key_tables[i] != table) {  // keys-only insert: entries of other tables / empty slots
      ws_slot[i] = kPresent;
      continue;
    }
    const uint64_t key = keys[i];
    const uint64_t home = hps::key_hash(key) & td.slot_mask;
    if (keys_only) {
      uint64_t j = home;
      bool present = false;
      uint32_t prow = 0;
      for (uint64_t p = 0; p <= td.slot_mask; ++p) {
        const Slot s = load_slot(base + j);
        if (s.row == kRowEmpty) break;
        if (s.key == key) {
          present = s.row != kRowPending;
          prow = s.row;
          break;
        }
        j = (j + 1) & td.slot_mask;
      }
      if (present) {
        ws_slot[i] = record_rows ? (kPresentRow | prow) : kPresent;
        continue;
      }
    }
    uint64_t idx = home;
    uint64_t found = kNoSlot;
    for (uint64_t p = 0; p <= td.slot_mask; ++p) {
      const Slot want{key, kRowPending, static_cast<uint32_t>(i)};
      const Slot old = slot_cas(base + idx, empty, want);
      if (old.row == kRowEmpty) {  // claimed a fresh slot
        found = idx;
        break;
      }
      if (old.key == key) {
        atomicMin(&base[idx].aux, static_cast<uint32_t>(i));
        found = idx;
        break;
      }
      idx = (idx + 1) & td.slot_mask;
    }
    if (found == kNoSlot) {
      latch_status(status, HPS_GPU_E_INFEASIBLE);
      atomicMax(abort_flag, 2u);
    }
    ws_slot[i] = found;
  }
  trace_end(kTrInsClaim);
}

// Insert phase B (scan op): count(i) = 1 iff occurrence i is the first occurrence of a
// key that was absent before the call. emit() stores its rank among those.
struct InsertScanOp {
  const Slot* slots;
  uint64_t slot_base;
  const uint64_t* ws_slot;
  uint32_t* ws_pos;
  uint8_t* ws_flag;  // bit0: first occurrence of a new key, bit1: first occurrence of an existing key
  uint64_t n;
  uint64_t* d_new;
  const uint32_t* abort_flag;
  __device__ uint64_t size() const { return *abort_flag ? 0 : n; }
  __device__ uint32_t count(uint64_t i) const {
    const uint64_t si = ws_slot[i];
    if (si >= kPresentRow) return 0;
    const Slot s = load_slot(slots + slot_base + si);
    return (s.row == kRowPending && s.aux == static_cast<uint32_t>(i)) ? 1u : 0u;
  }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    uint8_t f = 0;
    if (c) {
      ws_pos[i] = static_cast<uint32_t>(excl);
      f = 1;
    } else {
      const uint64_t si = ws_slot[i];
      if (si < kPresentRow) {
        const Slot s = load_slot(slots + slot_base + si);
        if (s.row != kRowPending && s.aux == static_cast<uint32_t>(i)) f = 2;
      }
    }
    ws_flag[i] = f;
  }
  __device__ void total(uint64_t t) const { *d_new = t; }
};

// Insert phase C: commit rows (warp-cooperative row initialisation, coalesced).
__global__ void k_insert_commit(Slot* __restrict__ slots, TableDev td, uint32_t table, const uint64_t* __restrict__ keys,
                                uint64_t n, const float* __restrict__ rows, const uint64_t* __restrict__ ws_slot,
                                const uint32_t* __restrict__ ws_pos, const uint8_t* __restrict__ ws_flag,
                                const uint64_t* __restrict__ d_new, const uint64_t* __restrict__ d_nrows,
                                float* __restrict__ W, float* __restrict__ S0, float* __restrict__ S1, int n_state,
                                float a0, uint32_t dim, uint64_t seed, uint64_t* __restrict__ row_keys,
                                uint32_t* abort_flag, uint32_t* status, uint16_t* __restrict__ Wh) {
  if (*reinterpret_cast<volatile uint32_t*>(abort_flag)) return;
  const uint64_t nrows = d_nrows[table];
  if (nrows + *d_new > td.row_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      latch_status(status, HPS_GPU_E_INFEASIBLE);
      atomicMax(abort_flag, 2u);
    }
    return;
  }
  trace_begin(kTrInsCommit);
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Slot* base = slots + td.slot_base;
  for (uint64_t w0 = warp * 32; w0 < n; w0 += n_warps * 32) {
    const uint64_t i = w0 + lane;
    uint8_t f = 0;
    uint64_t g = 0, key = 0;
    if (i < n) {
      f = ws_flag[i];
      key = keys[i];
      if (f & 1) {
        const uint64_t local = nrows + ws_pos[i];
        base[ws_slot[i]].row = static_cast<uint32_t>(local);
        g = td.row_base + local;
        row_keys[g] = key;
      } else if (f & 2) {
        g = td.row_base + base[ws_slot[i]].row;
      }
    }
    uint32_t todo = __ballot_sync(0xffffffffu, (f & 1) || ((f & 2) && rows != nullptr));
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t gr = __shfl_sync(0xffffffffu, g, src);
      const uint64_t kr = __shfl_sync(0xffffffffu, key, src);
      const uint8_t fr = static_cast<uint8_t>(__shfl_sync(0xffffffffu, static_cast<uint32_t>(f), src));
      const uint64_t ir = w0 + src;
      for (uint32_t j = lane; j < dim; j += 32) {
        const float val = rows ? rows[ir * dim + j] : init_value(seed, kr, j);
        if (Wh) Wh[gr * dim + j] = f32_to_half_bits(val);  // F16 table: round to nearest even
        else W[gr * dim + j] = val;
        if (fr & 1) {
          if (n_state >= 1) S0[gr * dim + j] = (n_state == 1) ? a0 : 0.0f;
          if (n_state >= 2) S1[gr * dim + j] = 0.0f;
        }
      }
    }
  }
  trace_end(kTrInsCommit);
}

// Insert phase D: publish rows_out, reset aux scratch (or roll the call back).
__global__ void k_insert_finish(Slot* __restrict__ slots, TableDev td, uint32_t table, uint64_t n,
                                const uint64_t* __restrict__ ws_slot, uint64_t* __restrict__ rows_out,
                                const uint64_t* __restrict__ d_new, uint64_t* __restrict__ d_nrows,
                                const uint32_t* __restrict__ abort_flag, InsertRecord rec) {
  const uint32_t ab = *reinterpret_cast<const volatile uint32_t*>(abort_flag);
  trace_begin(kTrInsFinish);
  Slot* base = slots + td.slot_base;
  if (rec.occ_row) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < rec.zero_words; w += gridDim.x * blockDim.x) rec.zero[w] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *rec.d_n = n;
  }
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t occ = rec.row_absent;  // (training record: the occurrence's global row)
    const uint64_t si = ws_slot[i];
    if (ab == 1) {  // refused before any claim (NonFinite)
      if (rows_out) rows_out[i] = ~0ull;
    } else if (si >= kPresentRow) {  // no slot claimed by this call: committed before, skipped, or failed
      if (si == kNoSlot && rows_out) rows_out[i] = ~0ull;
      if (si < kPresent) occ = static_cast<uint32_t>(td.row_base + static_cast<uint32_t>(si));
    } else {
      Slot* s = base + si;
      if (ab) {  // roll back: drop every slot claimed by this call, release aux
        if (s->row == kRowPending) {
          *reinterpret_cast<ulonglong2*>(s) = make_ulonglong2(0ull, (uint64_t(kAuxNone) << 32) | kRowEmpty);
        } else {
          s->aux = kAuxNone;
          occ = static_cast<uint32_t>(td.row_base + s->row);  // (committed by an earlier call)
        }
        if (rows_out) rows_out[i] = ~0ull;
      } else {
        // every occurrence of the key reads its row; only the first one (the claim's minimum
        // index, in aux) releases the scratch word — a store per occurrence would serialise the
        // hot keys' reads behind it (config 5: 29 vs 6.5 us)
        const uint32_t r = s->row;
        if (rows_out) rows_out[i] = r;
        occ = static_cast<uint32_t>(td.row_base + r);
        if (s->aux == static_cast<uint32_t>(i)) s->aux = kAuxNone;
      }
    }
    if (rec.occ_row) rec.occ_row[i] = occ;
  }
  if (!ab && blockIdx.x == 0 && threadIdx.x == 0) d_nrows[table] += *d_new;
  trace_end(kTrInsFinish);
}

// Ingest validation (the whole call is refused before any claim): NaN/Inf -> NonFinite; for
// an F16 table, a value whose binary16 rounding overflows (|x| >= 65520) -> F16Range.
__global__ void k_rows_non_finite(const float* __restrict__ v, uint64_t n, uint32_t* abort_flag, uint32_t* status,
                                  int f16) {
  bool bad = false, range = false;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = __float_as_uint(v[i]);
    bad |= non_finite_bits(b);
    range |= f16 && (b & 0x7fffffffu) >= 0x477ff000u && !non_finite_bits(b);
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) {
    latch_status(status, HPS_GPU_E_NON_FINITE);
    atomicMax(abort_flag, 1u);
  }
  if (__any_sync(0xffffffffu, range) && lane_id() == 0) {
    latch_status(status, HPS_GPU_E_F16_RANGE);
    atomicMax(abort_flag, 1u);
  }
}

__global__ void k_widen_half(const uint16_t* __restrict__ src, uint64_t n, float* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = __half2float(__ushort_as_half(src[i]));
}

__global__ void k_fill_slots_empty(Slot* slots, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    *reinterpret_cast<ulonglong2*>(slots + i) = make_ulonglong2(0ull, (uint64_t(kAuxNone) << 32) | kRowEmpty);
}

// ---------------------------------------------------------------------------------
// K1+K2+K3: fused hash -> probe -> gather -> pool
// ---------------------------------------------------------------------------------
struct LookupArgs {
  const uint64_t* keys;
  const uint32_t* offsets;
  uint32_t n_bags;
  uint32_t n_slots;
  const uint32_t* slot_table;
  const uint32_t* key_tables;  // one-key bags only: table of each key (overrides slot_table);
                               // an id >= n_tables marks an empty slot (absent, no gradient)
  uint32_t n_tables;
  const TableDev* tables;
  const Slot* slots;
  const float* W;
  const uint16_t* Wh;  // F16 table: binary16 rows (W unused)
  const float* defaults;
  uint32_t dim;
  int mean;
  float* out;
  // training only: per-occurrence records consumed by backward.cu
  uint32_t* occ_row;   // global row of each occurrence (row_absent: key absent -> no gradient)

  uint32_t row_absent;
  uint32_t* occ_bag;   // multi-hot: bag of each occurrence
  uint32_t* bag_len;   // multi-hot mean: bag lengths
  uint64_t* d_n;       // number of key occurrences (device)
  uint64_t max_keys;   // training record capacity (max_batch_keys)
  uint32_t* status;    // ctx status word: a device-offsets batch larger than max_keys latches InvalidArgument
  uint32_t* zero;      // training: the backward's zeroed words (bwd_zero_layout), cleared by the probe
  uint32_t zero_words;
};

// K3a (training): probe every occurrence once and record its row (row_absent when the
// key is absent), bag (multi-hot) and the bag lengths (mean). The pooling kernels then
// read the recorded rows, while the backward's dedup (backward.cu launch_dedup) runs on
// the side stream from the same record, concurrently with the pooling.
template <bool MULTI>
__global__ void __launch_bounds__(256) k_probe(LookupArgs a) {
  const uint32_t lane = lane_id();
  const uint64_t n_bags = a.n_bags;
  trace_begin(kTrProbe);
  // the backward's allocators and look-back words start from zero (the dedup, forked after
  // this kernel, is their first user): cleared here instead of by a memset node of its own
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.zero_words; i += gridDim.x * blockDim.x) a.zero[i] = 0;
  if constexpr (MULTI) {
    // device offsets are not validated on the host: a batch beyond the record's capacity is
    // refused here (latched InvalidArgument, an empty record) instead of overrunning it
    const uint64_t total = a.offsets[n_bags];
    if (total > a.max_keys) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.d_n = 0;
        latch_status(a.status, HPS_GPU_E_INVALID_ARGUMENT);
      }
      // the pooling still walks the offsets: every recorded row reads as absent
      for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.max_keys;
           i += uint64_t(gridDim.x) * blockDim.x)
        a.occ_row[i] = a.row_absent;
      trace_end(kTrProbe);
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_n = MULTI ? a.offsets[n_bags] : n_bags;
  if constexpr (!MULTI) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_bags; i += uint64_t(gridDim.x) * blockDim.x) {
      const uint32_t table = a.key_tables ? a.key_tables[i] : a.slot_table[static_cast<uint32_t>(i) % a.n_slots];
      if (table >= a.n_tables) {  // an empty slot of a fixed-capacity exchange buffer
        a.occ_row[i] = a.row_absent;
        continue;
      }
      const TableDev td = a.tables[table];
      const uint32_t local = probe_find(a.slots, td, a.keys[i]);
      a.occ_row[i] = local == kRowEmpty ? a.row_absent : static_cast<uint32_t>(td.row_base + local);
    }
  } else {
    // a warp owns 32 consecutive bags (lane = bag: its offsets), then walks the bags'
    // occurrences 32 at a time, coalesced; each lane finds its occurrence's bag by a
    // binary search over the warp's offsets (shuffles)
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t b0 = warp * 32; b0 < n_bags; b0 += n_warps * 32) {
      const uint64_t b = b0 + lane;
      const uint32_t nb = static_cast<uint32_t>(min(uint64_t(32), n_bags - b0));
      const uint32_t lo = a.offsets[b < n_bags ? b : n_bags];
      const uint32_t hi_all = __shfl_sync(0xffffffffu, a.offsets[b0 + nb], 0);
      if (b < n_bags && a.bag_len) a.bag_len[b] = a.offsets[b + 1] - lo;
      const uint32_t lo0 = __shfl_sync(0xffffffffu, lo, 0);
      for (uint32_t p0 = lo0; p0 < hi_all; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint32_t k = 0;
#pragma unroll
        for (uint32_t step = 16; step > 0; step >>= 1) {
          const uint32_t cand = k + step;
          const uint32_t lc = __shfl_sync(0xffffffffu, lo, cand & 31);
          if (cand < nb && lc <= p) k = cand;
        }
        if (p < hi_all) {
          const uint64_t bag = b0 + k;
          const uint32_t table = a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
          const TableDev td = a.tables[table];
          const uint32_t local = probe_find(a.slots, td, a.keys[p]);
          a.occ_row[p] = local == kRowEmpty ? a.row_absent : static_cast<uint32_t>(td.row_base + local);
          a.occ_bag[p] = static_cast<uint32_t>(bag);
        }
      }
    }
  }
  trace_end(kTrProbe);
}

// Batch-table entries left by a training record that no backward consumed: back to empty
// (the flat dedup's reset; k_dedup does the same at its start). Entries come from occ_ent,
// which the dedup writes for every occurrence (0xffffffff: absent key), so this may run after
// the next record's probe.
__global__ void k_reset_counts(const uint32_t* __restrict__ occ_ent, const uint64_t* d_n, uint2* bt) {
  trace_begin(kTrReset);
  if (d_n[5] == 0) {  // no unconsumed record in this slot (device truth; see begin_training_record)
    trace_end(kTrReset);
    return;
  }
  const uint64_t n = d_n[6];  // the unconsumed record's size
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = occ_ent[i];
    if (e != 0xffffffffu) bt[e] = make_uint2(kBtEmpty, 0xffffffffu);
  }
  trace_end(kTrReset);
}

// Row of occurrence i: ROWS — recorded by the training probe (k_probe_*); otherwise hash
// and probe the key here (inference: one fused pass).
template <bool ROWS>
__device__ __forceinline__ uint32_t occurrence_row(const LookupArgs& a, uint64_t i, uint32_t table) {
  if constexpr (ROWS) {
    if (i >= a.max_keys) return kRowEmpty;  // an oversized device-offsets batch (refused by k_probe)
    const uint32_t r = a.occ_row[i];
    return r == a.row_absent ? kRowEmpty : r;
  } else {
    const TableDev td = a.tables[table];
    const uint32_t local = probe_find(a.slots, td, a.keys[i]);
    return local == kRowEmpty ? kRowEmpty : static_cast<uint32_t>(td.row_base + local);
  }
}

// One-key-per-bag path. A warp owns 32 consecutive bags: every lane resolves one key's
// row (32 independent index loads in flight); then groups of LPR lanes stream the rows
// with 128-bit loads (VPL float4 per lane, 8 rows in flight per group) and write the bags
// coalesced.
template <int LPR, int VPL, bool ROWS, bool F16 = false>
__global__ void __launch_bounds__(256, 4) k_lookup_1hot(LookupArgs a) {
  constexpr int G = 32 / LPR;  // rows handled side by side by one warp
  constexpr int kBatch = (LPR < 8 ? LPR : 8) / (VPL > 4 ? 4 : VPL) > 0 ? (LPR < 8 ? LPR : 8) / (VPL > 4 ? 4 : VPL) : 1;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPR, gl = lane % LPR;
  const uint32_t nvec = a.dim / 4;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t t0 = warp * 32; t0 < a.n_bags; t0 += n_warps * 32) {
    const uint64_t bag = t0 + lane;
    uint32_t row = kRowEmpty, table = 0;
    if (bag < a.n_bags) {
      table = a.key_tables ? a.key_tables[bag] : a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
      if (table >= a.n_tables) table = 0;  // empty exchange slot: reads as absent
      else row = occurrence_row<ROWS>(a, bag, table);
    }
    for (int m0 = 0; m0 < LPR; m0 += kBatch) {
      float4 x[kBatch][VPL];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const uint32_t src = grp + G * (m0 + j);
        const uint32_t r = __shfl_sync(0xffffffffu, row, src);
        const uint32_t tb = __shfl_sync(0xffffffffu, table, src);
        const float4* p = reinterpret_cast<const float4*>(r == kRowEmpty ? a.defaults + uint64_t(tb) * a.dim
                                                                         : (F16 ? a.defaults : a.W + uint64_t(r) * a.dim));
        const uint16_t* ph = (F16 && r != kRowEmpty) ? a.Wh + uint64_t(r) * a.dim : nullptr;
        const bool ok = t0 + src < a.n_bags;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const uint32_t v = gl + k * LPR;
          x[j][k] = (ok && v < nvec) ? (F16 && ph ? ldg_half4(ph, v) : ldg_stream(p + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const uint64_t b = t0 + grp + G * (m0 + j);
        if (b >= a.n_bags) continue;
        float4* o = reinterpret_cast<float4*>(a.out + b * a.dim);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const uint32_t v = gl + k * LPR;
          // +0.0f + x (and x / 1.0f for mean) is the identity on every finite x except -0.0
          if (v < nvec) o[v] = f4_add(make_float4(0.f, 0.f, 0.f, 0.f), x[j][k]);
        }
      }
    }
  }
}

// One-key-per-bag path on the bulk-copy engine (TMA 1-D), used when rows are <= 1 KB and
// `out` is 16-byte aligned. A warp owns 32 consecutive bags per tile: the lanes hash and
// probe 32 keys; each lane then issues ONE cp.async.bulk of its row (or the table's
// default vector) into the warp's shared-memory tile, all completing on one mbarrier; the
// +0.0f normalisation of the oracle runs in smem; a single bulk store writes the 32 pooled
// rows (contiguous in `out`) back while the next tile's probes are already in flight.
// No registers hold row data, so every warp keeps 32 rows (16 KB at dim 128) outstanding.
constexpr int kTmaWarps = 4;

template <bool ROWS>
__global__ void __launch_bounds__(kTmaWarps * 32) k_lookup_1hot_tma(LookupArgs a) {
  extern __shared__ __align__(128) float s_rows[];  // [kTmaWarps][32][dim]
  __shared__ __align__(8) uint64_t s_bar[kTmaWarps];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  const uint32_t D = a.dim, nvec = D / 4, row_bytes = D * 4;
  float* tile = s_rows + size_t(w) * 32 * D;
  if (lane == 0) {
    mbar_init(&s_bar[w], 1);
    mbar_fence_init();
  }
  __syncwarp();
  uint32_t phase = 0;
  const uint64_t warp = uint64_t(blockIdx.x) * kTmaWarps + w;
  const uint64_t n_warps = uint64_t(gridDim.x) * kTmaWarps;
  trace_begin(ROWS ? kTrPool : -1);
  // training: the rows stay in L2 for the update that re-reads them after the dedup (evict_last),
  // the pooled outputs (read by the caller, not by this step) leave first (evict_first)
  // (config 2 0.115 -> 0.110 ms with the row stream's gradient rows evict_first too)
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  for (uint64_t t0 = warp * 32; t0 < a.n_bags; t0 += n_warps * 32) {
    const uint64_t bag = t0 + lane;
    const uint32_t nb = static_cast<uint32_t>(min(uint64_t(32), a.n_bags - t0));
    const float* src = nullptr;
    if (bag < a.n_bags) {
      uint32_t table = a.key_tables ? a.key_tables[bag] : a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
      uint32_t row = kRowEmpty;
      if (table >= a.n_tables) table = 0;  // empty exchange slot: reads as absent
      else row = occurrence_row<ROWS>(a, bag, table);
      src = row == kRowEmpty ? a.defaults + uint64_t(table) * D : a.W + uint64_t(row) * D;
    }
    if (lane == 0) bulk_wait_read_all();  // the previous tile's store has finished reading smem
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&s_bar[w], nb * row_bytes);
    __syncwarp();
    if (bag < a.n_bags) {
      if (ROWS) bulk_g2s_hint(tile + lane * D, src, row_bytes, &s_bar[w], keep);
      else bulk_g2s(tile + lane * D, src, row_bytes, &s_bar[w]);
    }
    mbar_wait(&s_bar[w], phase);
    phase ^= 1;
    float4* t4 = reinterpret_cast<float4*>(tile);
    for (uint32_t e = lane; e < nb * nvec; e += 32) t4[e] = f4_add(make_float4(0.f, 0.f, 0.f, 0.f), t4[e]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (ROWS) bulk_s2g_hint(a.out + t0 * D, tile, nb * row_bytes, stream);
      else bulk_s2g(a.out + t0 * D, tile, nb * row_bytes);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
  trace_end(ROWS ? kTrPool : -1);
}

// Source tier of a read-through key (SPEC.md:326 LookupResult.source_counts order).
constexpr uint8_t kSrcCache = 0, kSrcTable = 1, kSrcDefault = 3;

// Orchestrator read-through (one table): hits come from the cache's
// compacted rows, misses from this table (or its default vector when absent); the misses
// are listed in input order for migration into the cache (absent keys flagged: never cached).
template <int LPR>
__global__ void __launch_bounds__(256) k_read_through(const uint64_t* __restrict__ keys,
                                                      const float* __restrict__ found_vecs,
                                                      const uint32_t* __restrict__ found_idx,
                                                      const uint32_t* __restrict__ missing_idx, const uint64_t* counts,
                                                      const Slot* __restrict__ slots, TableDev td,
                                                      const float* __restrict__ W, const float* __restrict__ def,
                                                      uint32_t dim, float* __restrict__ out, uint64_t* miss_keys,
                                                      float* miss_vecs, uint8_t* miss_absent,
                                                      const uint16_t* __restrict__ Wh, uint8_t* src_out) {
  pdl_wait();
  pdl_launch_dependents();
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t nf = counts[0], nm = counts[1];
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t j = gid; j < nf + nm; j += ng) {
    const float4* src;
    const uint16_t* srch = nullptr;  // F16 table row (widened on the fly)
    float4* dst2 = nullptr;
    uint32_t i;
    if (j < nf) {
      i = found_idx[j];
      if (src_out && gl == 0) src_out[i] = kSrcCache;
      if (!found_vecs) continue;  // the hit's row is in place already
      src = reinterpret_cast<const float4*>(found_vecs + j * dim);
    } else {
      const uint64_t m = j - nf;
      i = missing_idx[m];
      const uint64_t k = keys[i];
      const uint32_t local = probe_find(slots, td, k);
      src = reinterpret_cast<const float4*>(local == kRowEmpty || Wh ? def : W + (td.row_base + local) * dim);
      if (Wh && local != kRowEmpty) srch = Wh + (td.row_base + local) * dim;
      dst2 = reinterpret_cast<float4*>(miss_vecs + m * dim);
      if (gl == 0) {
        miss_keys[m] = k;
        miss_absent[m] = local == kRowEmpty ? 1 : 0;
        if (src_out) src_out[i] = local == kRowEmpty ? kSrcDefault : kSrcTable;
      }
    }
    float4* dst = reinterpret_cast<float4*>(out + uint64_t(i) * dim);
    for (uint32_t v = gl; v < nvec; v += LPR) {
      const float4 x = srch ? ldg_half4(srch, v) : __ldg(src + v);
      dst[v] = x;
      if (dst2) dst2[v] = x;
    }
  }
}

// Multi-hot path: a group of LPR lanes owns one bag at a time; the group resolves LPR
// keys of the bag in parallel, then accumulates the rows in bag order (4 in flight).
// Rows of a bag's chunk gathered before any is summed (bytes in flight per lane group).
#ifndef HPS_MULTI_ROWS
#define HPS_MULTI_ROWS 4
#endif
constexpr int kMultiRows = HPS_MULTI_ROWS;
template <int LPR, int VPL, bool ROWS, bool F16 = false>
__global__ void __launch_bounds__(256) k_lookup_multi(LookupArgs a) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPR, gl = lane % LPR;
  const uint32_t gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const uint32_t nvec = a.dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t n_groups = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  trace_begin(ROWS ? kTrPool : -1);
  for (uint64_t bag = gid; bag < a.n_bags; bag += n_groups) {
    const uint32_t lo = a.offsets[bag], hi = a.offsets[bag + 1];
    const uint32_t table = a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
    float4 acc[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t c = lo; c < hi; c += LPR) {
      const uint32_t i = c + gl;
      const uint32_t row = i < hi ? occurrence_row<ROWS>(a, i, table) : kRowEmpty;
      const uint32_t cnt = min(uint32_t(LPR), hi - c);
      for (uint32_t m0 = 0; m0 < cnt; m0 += kMultiRows) {
        float4 x[kMultiRows][VPL];
#pragma unroll
        for (int j = 0; j < kMultiRows; ++j) {
          const uint32_t m = m0 + j;
          const uint32_t r = __shfl_sync(gmask, row, grp * LPR + (m < LPR ? m : 0));
          const float4* p = reinterpret_cast<const float4*>(
              r == kRowEmpty ? a.defaults + uint64_t(table) * a.dim : (F16 ? a.defaults : a.W + uint64_t(r) * a.dim));
          const uint16_t* ph = (F16 && r != kRowEmpty) ? a.Wh + uint64_t(r) * a.dim : nullptr;
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const uint32_t v = gl + k * LPR;
            x[j][k] = (m < cnt && v < nvec) ? (F16 && ph ? ldg_half4(ph, v) : ldg_stream(p + v))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int j = 0; j < kMultiRows; ++j) {
          if (m0 + j < cnt) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) acc[k] = f4_add(acc[k], x[j][k]);
          }
        }
      }
    }
    const uint32_t len = hi - lo;
    float4* o = reinterpret_cast<float4*>(a.out + bag * a.dim);
    const float fl = static_cast<float>(len);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t v = gl + k * LPR;
      if (v < nvec) o[v] = (a.mean && len > 0) ? f4_div(acc[k], fl) : acc[k];
    }
  }
  trace_end(ROWS ? kTrPool : -1);
}

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

uint64_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return HPS_GPU_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_last_error("cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}

}  // namespace

cudaError_t hpsg::trace_attach_table(TraceRec* p) { return trace_attach_tu(p); }

namespace {

// Entry points whose caller buffers are addressed at the storage stride (the exchange, hybrid
// and read-through paths) take only dims that are a multiple of 4.
int refuse_padded(hps_gpu_table, const char* what) {
  set_last_error(std::string(what) + ": needs dim % 4 == 0 (rows of this table are padded)");
  return HPS_GPU_E_INVALID_ARGUMENT;
}

int check_tbl(hps_gpu_table t) {
  if (!t) {
    set_last_error("null table handle");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  return HPS_GPU_OK;
}

// (lanes per row, float4 per lane) for a row of nvec float4: LPR = largest power of two
// <= min(32, nvec); VPL = ceil(nvec / LPR) (<= 8, so dim <= 1024).
#define HPSG_DISPATCH_ROW(KERNEL, R, GRIDF, ...)                                    \
  do {                                                                              \
    if (nvec > 128) KERNEL<32, 8, R><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);       \
    else if (nvec > 64) KERNEL<32, 4, R><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec > 32) KERNEL<32, 2, R><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec == 32) KERNEL<32, 1, R><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);  \
    else if (nvec > 16) KERNEL<16, 2, R><<<GRIDF(16), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec == 16) KERNEL<16, 1, R><<<GRIDF(16), 256, 0, st>>>(__VA_ARGS__);  \
    else if (nvec > 8) KERNEL<8, 2, R><<<GRIDF(8), 256, 0, st>>>(__VA_ARGS__);      \
    else if (nvec == 8) KERNEL<8, 1, R><<<GRIDF(8), 256, 0, st>>>(__VA_ARGS__);     \
    else if (nvec > 4) KERNEL<4, 2, R><<<GRIDF(4), 256, 0, st>>>(__VA_ARGS__);      \
    else if (nvec == 4) KERNEL<4, 1, R><<<GRIDF(4), 256, 0, st>>>(__VA_ARGS__);     \
    else if (nvec > 2) KERNEL<2, 2, R><<<GRIDF(2), 256, 0, st>>>(__VA_ARGS__);      \
    else if (nvec == 2) KERNEL<2, 1, R><<<GRIDF(2), 256, 0, st>>>(__VA_ARGS__);     \
    else KERNEL<1, 1, R><<<GRIDF(1), 256, 0, st>>>(__VA_ARGS__);                    \
  } while (0)

// nk: key occurrences of this call (host bound). A training lookup also clears the
// backward's look-back/ticket region here, so the lookup -> sort -> reduce chain that
// follows is kernel-to-kernel (programmatic dependent launches, no memset node between).
// ---------------------------------------------------------------------------------
// Hybrid sparse embedding:
// hot keys live in a replicated table group (this table), cold keys on their owner.
// ---------------------------------------------------------------------------------
// Cold occurrences (absent from the hot index), compacted in occurrence order.
struct ColdOp {
  const uint32_t* occ_row;
  uint32_t row_absent;
  const uint64_t* keys;
  const uint32_t* occ_bag;  // nullptr: one key per bag
  uint32_t* cold_pos;
  uint64_t* cold_keys;
  uint32_t* cold_bags;
  uint64_t* d_count;
  const uint64_t* d_n;
  __device__ uint64_t size() const { return *d_n; }
  __device__ uint32_t count(uint64_t i) const { return occ_row[i] == row_absent ? 1u : 0u; }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    cold_pos[i] = static_cast<uint32_t>(excl);
    if (c) {
      cold_keys[excl] = keys[i];
      cold_bags[excl] = occ_bag ? occ_bag[i] : static_cast<uint32_t>(i);
    }
  }
  __device__ void total(uint64_t t) const { *d_count = t; }
};

// Pool every bag in occurrence order from the hot replica or the rows returned by the
// cold owners (cold_rows[perm[cold_pos[i]]]): the same sequential sum as any lookup.
template <int LPR>
__global__ void __launch_bounds__(256) k_hybrid_pool(const uint32_t* __restrict__ occ_row, uint32_t row_absent,
                                                     const float* __restrict__ W, const uint32_t* __restrict__ cold_pos,
                                                     const uint32_t* __restrict__ perm,
                                                     const float* __restrict__ cold_rows,
                                                     const uint32_t* __restrict__ offsets, uint64_t n_bags,
                                                     uint32_t dim, int mean, float* __restrict__ out) {
  pdl_wait();
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t b = gid; b < n_bags; b += ng) {
    const uint64_t lo = offsets ? offsets[b] : b, hi = offsets ? offsets[b + 1] : b + 1;
    for (uint32_t v = gl; v < nvec; v += LPR) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint64_t i = lo; i < hi; ++i) {
        const uint32_t r = occ_row[i];
        const float4* src = r != row_absent
                                ? reinterpret_cast<const float4*>(W + uint64_t(r) * dim)
                                : reinterpret_cast<const float4*>(cold_rows + uint64_t(perm[cold_pos[i]]) * dim);
        acc = f4_add(acc, __ldg(src + v));
      }
      if (mean && hi > lo) acc = f4_div(acc, static_cast<float>(hi - lo));
      reinterpret_cast<float4*>(out + b * dim)[v] = acc;
    }
  }
}

}  // namespace
int hpsg_insert_on(hps_gpu_table t, uint32_t table, const uint64_t* keys, uint64_t n, const float* rows,
                   uint64_t* rows_out, cudaStream_t st, const uint32_t* key_tables = nullptr,
                   const InsertRecord& rec = InsertRecord{});
namespace {

// A training record is about to overwrite ws_rows_a: counters of a previous record that no
// backward consumed go back to zero first (they are still described by ws_rows_a, once
// that record's dedup on the side stream is done).
int begin_training_record(hps_gpu_table t, LookupArgs& a, uint64_t nk, cudaStream_t st) {
  if (t->dedup_pending) {  // the whole previous dedup, long-segment part included
    HPSG_CUDA(wait_recorded(st, t->ev_done, t->pre_capture));
    t->dedup_pending = false;
  }
  // An unconsumed previous record's batch-table entries: the persistent k_dedup resets them
  // itself (device-checked at its start); the flat dedup gets the reset kernel, always (it is
  // device-checked: a captured graph may be replayed after eager calls left a record behind).
  if (t->flat_dedup) {
    k_reset_counts<<<grid_for(t->last_n_keys_host, 256, kNumSMs * 8), 256, 0, st>>>(t->ws_occ_ent, t->ws_counts,
                                                                                   t->ws_bt);
    HPSG_CHECK_LAUNCH("k_reset_counts");
  }
  a.zero = t->ws_zero;  // cleared by k_probe, which record() launches next
  a.zero_words = static_cast<uint32_t>(bwd_zero_layout(nk).total);
  a.occ_row = t->ws_rows_a;

  a.row_absent = t->row_absent;
  a.d_n = t->ws_counts;
  a.max_keys = t->max_keys;
  a.status = t->ctx->d_status;
  t->have_unique = false;
  t->prefetched = false;
  t->pre_keys_host = false;
  return HPS_GPU_OK;
}

// Training record: probe + record every occurrence (on `st`). fork_dedup then puts the
// backward's dedup on the slot's side stream (it needs only the record), after the pooling
// was launched on the main stream: the two run concurrently; backward_update joins.
int record_done(hps_gpu_table t, const LookupArgs& a, bool multi, bool mean, uint64_t nk, cudaStream_t st);

int record(hps_gpu_table t, const LookupArgs& a, bool multi, bool mean, uint64_t nk, cudaStream_t st) {
  if (multi) k_probe<true><<<grid_for((uint64_t(a.n_bags) + 31) / 32 * 32, 256, kNumSMs * 16), 256, 0, st>>>(a);
  else k_probe<false><<<grid_for(a.n_bags, 256, kNumSMs * 16), 256, 0, st>>>(a);
  HPSG_CHECK_LAUNCH("probe");
  return record_done(t, a, multi, mean, nk, st);
}

// One-hot insert-on-miss training record: the insert pass resolves every key anyway, so its
// last kernel writes the record (rows, size, zeroed words) and no probe follows — one launch
// and one full pass over the hash table fewer on config 5's critical path.
int record_by_insert(hps_gpu_table t, const LookupArgs& a, const uint64_t* keys, uint64_t nk, cudaStream_t st) {
  InsertRecord rec;
  rec.occ_row = t->ws_rows_a;
  rec.row_base = t->h_tables[0].row_base;
  rec.row_absent = t->row_absent;
  rec.d_n = t->ws_counts;
  rec.zero = a.zero;
  rec.zero_words = a.zero_words;
  if (int s = hpsg_insert_on(t, 0, keys, nk, nullptr, nullptr, st, nullptr, rec)) return s;
  return record_done(t, a, false, a.mean, nk, st);
}

int record_done(hps_gpu_table t, const LookupArgs& a, bool multi, bool mean, uint64_t nk, cudaStream_t st) {
  t->last_multi = multi;
  t->last_combiner = mean ? HPS_COMBINER_MEAN : HPS_COMBINER_SUM;
  t->last_n_keys_host = nk;
  t->pre_n_bags = a.n_bags;
  t->pre_capture = capture_id(st);
  // the fork point: right after the record (the pooling launched next does not gate the dedup)
  if (!t->no_fork && st != t->side) HPSG_CUDA(cudaEventRecord(t->ev_fork, st));
  return HPS_GPU_OK;
}

// The dedup of the current slot on its side stream. A table's dedups run one at a time
// (each is a persistent kernel whose grid barriers need all its CTAs resident).
int dedup_on_side(hps_gpu_table t) {
  hps_gpu_ctx c = t->ctx;
  if (c->ev_last_dedup && c->ev_last_dedup != t->ev_done)
    HPSG_CUDA(wait_recorded(t->side, c->ev_last_dedup, c->last_dedup_capture));
  if (int s = launch_dedup(t, t->side)) return s;  // records ev_join after the short placement
  HPSG_CUDA(cudaEventRecord(t->ev_done, t->side));
  c->ev_last_dedup = t->ev_done;
  c->last_dedup_capture = capture_id(t->side);
  t->dedup_pending = true;
  return HPS_GPU_OK;
}

int fork_dedup(hps_gpu_table t) {
  if (t->no_fork) {  // A/B measurement: dedup deferred to backward_update, all on the main stream
    t->dedup_deferred = true;
    return HPS_GPU_OK;
  }
  HPSG_CUDA(cudaStreamWaitEvent(t->side, t->ev_fork, 0));
  return dedup_on_side(t);
}

int launch_lookup(hps_gpu_table t, const LookupArgs& a, bool multi, bool rows);

// Host-pointer keys/offsets staged H2D into the current slot (HPS_LOOKUP_KEYS_HOST); sets
// *n_keys_host exactly when it is known on the host.
int stage_keys(hps_gpu_table t, const uint64_t*& keys, const uint32_t*& offsets, uint64_t n_bags, uint32_t flags,
               cudaStream_t st, uint64_t* n_keys_host, bool defer_insert = false) {
  const bool multi = offsets != nullptr;
  if (flags & HPS_LOOKUP_KEYS_HOST) {
    // Host buffers: stage H2D on the stream (pinned memory -> async copy).
    *n_keys_host = multi ? offsets[n_bags] : n_bags;
    if (*n_keys_host > t->max_keys) return HPS_GPU_E_INVALID_ARGUMENT;
    HPSG_CUDA(cudaMemcpyAsync(t->ws_keys_stage, keys, *n_keys_host * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    if (multi)
      HPSG_CUDA(cudaMemcpyAsync(t->ws_offsets_stage, offsets, (n_bags + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    keys = t->ws_keys_stage;
    if (multi) offsets = t->ws_offsets_stage;
  } else if (!multi && n_bags > t->max_keys) {
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (flags & HPS_LOOKUP_INSERT) {
    // Dynamic table (keys materialise on first touch): insert the batch's keys first, in
    // batch order, so new rows get deterministic ids; then the lookup finds all of them.
    if (t->n_tables != 1 || (multi && !(flags & HPS_LOOKUP_KEYS_HOST))) {
      set_last_error("HPS_LOOKUP_INSERT needs a single-table group and a host-known key count");
      return HPS_GPU_E_INVALID_ARGUMENT;
    }
    if (!defer_insert)  // (deferred: the caller's training record runs the insert, record_by_insert)
      if (int s = hpsg_insert_on(t, 0, keys, *n_keys_host, nullptr, nullptr, st)) return s;
  }
  return HPS_GPU_OK;
}

void fill_lookup_args(hps_gpu_table t, LookupArgs& a, const uint64_t* keys, const uint32_t* offsets, uint64_t n_bags,
                      int combiner, float* out) {
  a.keys = keys;
  a.offsets = offsets;
  a.n_bags = static_cast<uint32_t>(n_bags);
  a.n_slots = t->n_slots;
  a.slot_table = t->d_slot_table;
  a.tables = t->d_tables;
  a.n_tables = t->n_tables;
  a.slots = t->d_slots;
  a.W = t->d_w;
  a.Wh = t->d_wh;
  a.defaults = t->d_defaults;
  a.dim = t->dim;
  a.mean = combiner == HPS_COMBINER_MEAN;
  a.out = out;
}

// hps_gpu_table_prefetch with the target slot current: everything on the slot's side stream,
// after the table stream's position at the call.
int prefetch_into_current(hps_gpu_table t, const uint64_t* keys, const uint32_t* offsets, uint64_t n_bags,
                          int combiner, uint32_t flags) {
  cudaStream_t st = t->side;
  HPSG_CUDA(cudaEventRecord(t->ev_pre, t->ctx->stream));
  HPSG_CUDA(cudaStreamWaitEvent(st, t->ev_pre, 0));
  const bool multi = offsets != nullptr;
  uint64_t n_keys_host = multi ? t->max_keys : n_bags;
  if (int s = stage_keys(t, keys, offsets, n_bags, flags, st, &n_keys_host)) return s;
  LookupArgs a{};
  fill_lookup_args(t, a, keys, offsets, n_bags, combiner, nullptr);
  if (int s = begin_training_record(t, a, n_keys_host, st)) return s;
  a.occ_bag = multi ? t->ws_occ_bag : nullptr;
  a.bag_len = (multi && a.mean) ? t->ws_bag_len : nullptr;
  if (int s = record(t, a, multi, a.mean, n_keys_host, st)) return s;
  HPSG_CUDA(cudaEventRecord(t->ev_probe, st));
  if (int s = dedup_on_side(t)) return s;
  t->prefetched = true;
  t->pre_keys_host = multi && (flags & HPS_LOOKUP_KEYS_HOST);
  t->have_train = false;
  return HPS_GPU_OK;
}

// HPS_LOOKUP_PREFETCHED: make the prefetched slot current and pool from its record.
int lookup_prefetched(hps_gpu_table t, const uint32_t* offsets, uint64_t n_bags, int combiner, float* out,
                      uint32_t flags) {
  const uint32_t slot = HPS_LOOKUP_SLOT_OF(flags);
  if (slot >= t->parked.size() || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (slot != t->cur && t->have_train) {
    set_last_error("lookup(PREFETCHED): the previous training lookup's backward has not run");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const BatchSlot& b = slot == t->cur ? static_cast<const BatchSlot&>(*t) : t->parked[slot];
  const bool multi = offsets != nullptr || b.pre_keys_host;
  // Under stream capture the host flags may lag the device (graphs replayed out of capture
  // order): the caller's slot discipline is trusted there, the batch shape is still checked.
  const bool capturing = capture_id(t->ctx->stream) != 0;
  if ((!b.prefetched && !capturing) || b.have_train || b.pre_n_bags != n_bags || b.last_multi != multi ||
      b.last_combiner != combiner) {
    set_last_error("lookup(PREFETCHED): no matching prefetch in this slot (bags, offsets, combiner)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  use_slot(t, slot);
  cudaStream_t st = t->ctx->stream;
  HPSG_CUDA(wait_recorded(st, t->ev_probe, t->pre_capture));
  LookupArgs a{};
  fill_lookup_args(t, a, nullptr, t->pre_keys_host ? t->ws_offsets_stage : offsets, n_bags, combiner, out);
  a.occ_row = t->ws_rows_a;
  a.row_absent = t->row_absent;
  a.d_n = t->ws_counts;
  a.max_keys = t->max_keys;
  a.status = t->ctx->d_status;
  a.occ_bag = multi ? t->ws_occ_bag : nullptr;
  a.bag_len = (multi && a.mean) ? t->ws_bag_len : nullptr;
  if (int s = launch_lookup(t, a, multi, true)) return s;
  t->prefetched = false;
  t->have_train = true;
  return HPS_GPU_OK;
}

// Pooled lookup. ROWS (training): rows come from the record (record() ran first);
// otherwise hash + probe + gather + pool in one pass.
#define HPSG_DISPATCH_ROW16(KERNEL, GRIDF, ...)                                          \
  do {                                                                                    \
    if (nvec > 128) KERNEL<32, 8, false, true><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec > 64) KERNEL<32, 4, false, true><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);\
    else if (nvec > 32) KERNEL<32, 2, false, true><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);\
    else if (nvec == 32) KERNEL<32, 1, false, true><<<GRIDF(32), 256, 0, st>>>(__VA_ARGS__);\
    else if (nvec > 16) KERNEL<16, 2, false, true><<<GRIDF(16), 256, 0, st>>>(__VA_ARGS__);\
    else if (nvec == 16) KERNEL<16, 1, false, true><<<GRIDF(16), 256, 0, st>>>(__VA_ARGS__);\
    else if (nvec > 8) KERNEL<8, 2, false, true><<<GRIDF(8), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec == 8) KERNEL<8, 1, false, true><<<GRIDF(8), 256, 0, st>>>(__VA_ARGS__);  \
    else if (nvec > 4) KERNEL<4, 2, false, true><<<GRIDF(4), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec == 4) KERNEL<4, 1, false, true><<<GRIDF(4), 256, 0, st>>>(__VA_ARGS__);  \
    else if (nvec > 2) KERNEL<2, 2, false, true><<<GRIDF(2), 256, 0, st>>>(__VA_ARGS__);   \
    else if (nvec == 2) KERNEL<2, 1, false, true><<<GRIDF(2), 256, 0, st>>>(__VA_ARGS__);  \
    else KERNEL<1, 1, false, true><<<GRIDF(1), 256, 0, st>>>(__VA_ARGS__);                 \
  } while (0)

int launch_lookup(hps_gpu_table t, const LookupArgs& a, bool multi, bool rows) {
  const cudaStream_t st = t->ctx->stream;
  const uint32_t nvec = t->dim / 4;
  if (t->f16) {  // inference table: binary16 rows widened in the register paths
    auto grid1 = [&](int) { return grid_for((uint64_t(a.n_bags) + 31) / 32 * 32, 256, kNumSMs * 64); };
    auto gridm = [&](int lpr) {
      const uint64_t groups_per_block = 8 * (32 / lpr);
      return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((a.n_bags + groups_per_block - 1) / groups_per_block,
                                                                       kNumSMs * 64)));
    };
    if (multi) HPSG_DISPATCH_ROW16(k_lookup_multi, gridm, a);
    else HPSG_DISPATCH_ROW16(k_lookup_1hot, grid1, a);
    HPSG_CHECK_LAUNCH("lookup f16");
    return HPS_GPU_OK;
  }
  const bool tma_ok = t->dim <= 256 && (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0 && !t->no_tma;
  if (!multi && tma_ok) {
    static std::atomic<uint64_t> attr{0};
    HPSG_CUDA(once_per_device(attr, []() -> cudaError_t {
      for (cudaError_t e : {cudaFuncSetAttribute(k_lookup_1hot_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kTmaWarps * 32 * 256 * 4),
                            cudaFuncSetAttribute(k_lookup_1hot_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kTmaWarps * 32 * 256 * 4),
                            prefer_max_smem(k_lookup_1hot_tma<true>), prefer_max_smem(k_lookup_1hot_tma<false>)})
        if (e) return e;
      return cudaSuccess;
    }));
    const size_t smem = size_t(kTmaWarps) * 32 * t->dim * sizeof(float);
    const uint64_t tiles = (uint64_t(a.n_bags) + 31) / 32;
    // training: ONE CTA per SM. The pooling runs beside the dedup, and its row stream slows
    // the dedup's L2 atomics; at one CTA per SM it takes ~46 us instead of 37, still hidden,
    // and the dedup's count phase drops from 35 to 27 us (config 2: 0.134 -> 0.131 ms)
    uint64_t train_ctas = t->prefetched ? 8 : 1;  // prefetched: its dedup ran ahead, nothing to leave room for
    if (const char* e = std::getenv("HPS_GPU_POOL_CTAS")) train_ctas = std::max(1, std::atoi(e));  // A/B knob
    const uint64_t max_grid = rows ? uint64_t(kNumSMs) * train_ctas : uint64_t(kNumSMs) * 8;
    const int grid =
        static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((tiles + kTmaWarps - 1) / kTmaWarps, max_grid)));
    if (rows) k_lookup_1hot_tma<true><<<grid, kTmaWarps * 32, smem, st>>>(a);
    else k_lookup_1hot_tma<false><<<grid, kTmaWarps * 32, smem, st>>>(a);
  } else if (!multi) {
    auto grid1 = [&](int) { return grid_for((uint64_t(a.n_bags) + 31) / 32 * 32, 256, kNumSMs * (rows ? 4 : 64)); };
    if (rows) HPSG_DISPATCH_ROW(k_lookup_1hot, true, grid1, a);
    else HPSG_DISPATCH_ROW(k_lookup_1hot, false, grid1, a);
  } else {
    auto gridm = [&](int lpr) {
      const uint64_t groups_per_block = 8 * (32 / lpr);
      const uint64_t g = (a.n_bags + groups_per_block - 1) / groups_per_block;
      return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, kNumSMs * (rows ? 4 : 64))));
    };
    if (rows) HPSG_DISPATCH_ROW(k_lookup_multi, true, gridm, a);
    else HPSG_DISPATCH_ROW(k_lookup_multi, false, gridm, a);
  }
  HPSG_CHECK_LAUNCH("lookup");
  return HPS_GPU_OK;
}

// One batch slot's workspaces, side stream and events (sizes from the table's max_keys /
// max_bags); the caller keeps it in the table (current or parked).
int alloc_batch_slot(hps_gpu_table t, BatchSlot& b) {
  const uint64_t D = t->dim, N = t->max_keys, B = t->max_bags;
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dalloc(&b.ws_rows_a, N));
  A(dalloc(&b.ws_rank, N));
  A(dalloc(&b.ws_bt, t->bt_mask + 1));
  A(dalloc(&b.ws_occ_ent, N));
  A(dalloc(&b.ws_lead, N));
  A(dalloc(&b.ws_long_ent, t->max_long));
  A(dalloc(&b.ws_occ_bag, N));
  A(dalloc(&b.ws_bag_len, B));
  A(dalloc(&b.ws_short_rec, N));
  A(dalloc(&b.ws_short_bag, N));
  A(dalloc(&b.ws_long_row, t->max_long));
  A(dalloc(&b.ws_long_len, t->max_long));
  A(dalloc(&b.ws_long_start, t->max_long));
  A(dalloc(&b.ws_lkey_a, N));
  A(dalloc(&b.ws_lval_a, N));
  A(dalloc(&b.ws_lkey_b, N));
  A(dalloc(&b.ws_lval_b, N));
  A(dalloc(&b.ws_long_base, t->max_long));
  A(dalloc(&b.ws_task_long, t->max_chunks));
  A(dalloc(&b.ws_partial2, bwd_max_nodes(N) * D));
  A(dalloc(&b.ws_long_hbase, t->max_long));
  A(dalloc(&b.ws_node_cnt, bwd_max_nodes(N)));
  A(dalloc(&b.ws_partial, t->max_chunks * D));
  A(dalloc(&b.ws_counts, 8));
  A(dalloc(&b.ws_zero, t->zero_words));
  A(dalloc(&b.ws_keys_stage, N));
  A(dalloc(&b.ws_offsets_stage, B + 1));
  A(dalloc(&b.ws_ins_slot, N));
  A(dalloc(&b.ws_ins_pos, N));
  A(dalloc(&b.ws_ins_flag, N));
  A(dalloc(&b.ws_ins_scan, scan_tiles(N) + 3));
  if (st) return st;
  cudaStream_t s = t->ctx->stream;
  HPSG_CUDA(cudaMemsetAsync(b.ws_counts, 0, 8 * sizeof(uint64_t), s));
  HPSG_CUDA(cudaMemsetAsync(b.ws_bt, 0xff, (t->bt_mask + 1) * sizeof(uint2), s));  // {kBtEmpty, UINT32_MAX}
  HPSG_CUDA(cudaMemsetAsync(b.ws_node_cnt, 0, bwd_max_nodes(N) * sizeof(uint32_t), s));
  {  // the dedup / long-segment side stream gets the higher priority: its short, latency-bound
     // kernels are dispatched ahead of the bandwidth-bound main-stream CTAs they overlap
    int lo = 0, hi = 0;
    HPSG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    HPSG_CUDA(cudaStreamCreateWithPriority(&b.side, cudaStreamNonBlocking, hi));
  }
  for (cudaEvent_t* e : {&b.ev_bwd, &b.ev_done, &b.ev_join2, &b.ev_fork, &b.ev_join, &b.ev_pre, &b.ev_probe})
    HPSG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  (void)D;
  (void)B;
  return HPS_GPU_OK;
}

void free_batch_slot(BatchSlot& b) {
  void* ptrs[] = {b.ws_rows_a,   b.ws_bt,        b.ws_occ_ent,    b.ws_lead,       b.ws_long_ent,   b.ws_rank,
                  b.ws_short_rec, b.ws_short_bag, b.ws_occ_bag,   b.ws_bag_len,    b.ws_long_row,   b.ws_long_len,
                  b.ws_long_start, b.ws_lkey_a,   b.ws_lval_a,    b.ws_lkey_b,     b.ws_lval_b,     b.ws_long_base,
                  b.ws_task_long, b.ws_partial2,  b.ws_long_hbase, b.ws_node_cnt,  b.ws_partial,    b.ws_counts,
                  b.ws_zero,      b.ws_keys_stage, b.ws_offsets_stage, b.ws_ins_slot, b.ws_ins_pos,
                  b.ws_ins_flag,  b.ws_ins_scan};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t e : {b.ev_fork, b.ev_join, b.ev_bwd, b.ev_done, b.ev_join2, b.ev_pre, b.ev_probe})
    if (e) cudaEventDestroy(e);
  if (b.side) cudaStreamDestroy(b.side);
  b = BatchSlot{};
}

}  // namespace

extern "C" {

int hps_gpu_table_create(hps_gpu_ctx ctx, const hps_table_config* cfg, hps_gpu_table* out) {
  if (!ctx || !cfg || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  if (cfg->n_tables == 0 || !cfg->row_capacity_host || cfg->n_slots == 0 || !cfg->slot_table_host) {
    set_last_error("table config: n_tables, row_capacity, n_slots and slot_table are required");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (cfg->dim == 0 || cfg->dim > 1024) {
    set_last_error("table config: dim must be in [1, 1024] (rows up to 1024 floats per warp)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (cfg->optimizer < HPS_OPT_SGD || cfg->optimizer > HPS_OPT_ADAM) return HPS_GPU_E_INVALID_ARGUMENT;
  for (uint32_t s = 0; s < cfg->n_slots; ++s)
    if (cfg->slot_table_host[s] >= cfg->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (cfg->max_batch_keys == 0 || cfg->max_batch_keys >= (1ull << 31) || cfg->max_batch_bags == 0 ||
      cfg->max_batch_bags >= (1ull << 31)) {
    set_last_error("table config: max_batch_keys / max_batch_bags must be in [1, 2^31)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  HPSG_CUDA(cudaSetDevice(ctx->device));
  bool flat_dedup = false;
  if (int s = choose_dedup(&flat_dedup)) return s;
  auto t = new hps_gpu_table_s;
  t->flat_dedup = flat_dedup;
  t->ctx = ctx;
  t->n_tables = cfg->n_tables;
  t->dim_io = cfg->dim;
  t->dim = padded_dim(cfg->dim);
  t->n_slots = cfg->n_slots;
  t->optimizer = cfg->optimizer;
  t->n_state = cfg->optimizer == HPS_OPT_SGD ? 0 : cfg->optimizer == HPS_OPT_ADAGRAD ? 1 : 2;
  if (cfg->dtype != HPS_DTYPE_F32 && cfg->dtype != HPS_DTYPE_F16) {
    delete t;
    set_last_error("table config: dtype must be HPS_DTYPE_F32 or HPS_DTYPE_F16");
    return HPS_GPU_E_DTYPE_MISMATCH;
  }
  t->f16 = cfg->dtype == HPS_DTYPE_F16;
  if (t->f16) t->n_state = 0;  // an inference table holds no optimizer state
  t->seed = cfg->init_seed;
  t->a0 = cfg->adagrad_initial_accumulator;
  t->max_keys = cfg->max_batch_keys;
  t->max_bags = cfg->max_batch_bags;
  if (const char* e = std::getenv("HPS_GPU_NO_TMA")) t->no_tma = e[0] == '1';
  if (const char* e = std::getenv("HPS_GPU_NO_FORK")) t->no_fork = e[0] == '1';
  uint64_t rows = 0, slots = 0;
  for (uint32_t i = 0; i < t->n_tables; ++i) {
    const uint64_t cap = cfg->row_capacity_host[i];
    if (cap == 0 || cap >= 0xfffffff0ull) {
      delete t;
      return HPS_GPU_E_INVALID_ARGUMENT;
    }
    const uint64_t sc = next_pow2(std::max<uint64_t>(2 * cap, 16));
    t->row_cap.push_back(cap);
    t->row_base.push_back(rows);
    t->slot_cap.push_back(sc);
    t->slot_base.push_back(slots);
    t->h_tables.push_back(TableDev{slots, sc - 1, rows, cap});
    rows += cap;
    slots += sc;
  }
  if (rows >= 0xfffffff0ull) {
    set_last_error("table group exceeds 2^32 - 16 rows (u32 global row ids)");
    delete t;
    return HPS_GPU_E_INFEASIBLE;
  }
  t->total_rows = rows;
  t->total_slots = slots;
  const uint64_t D = t->dim, N = t->max_keys, B = t->max_bags;
  t->row_absent = static_cast<uint32_t>(rows);
  t->sort_bits = std::max(1, bits_for(rows));
  t->max_long = bwd_max_long(N);
  t->max_chunks = bwd_max_chunks(N);
  // (also the scratch of last_unique's row sort)
  t->zero_words = std::max(bwd_zero_layout(N).total, sort_ws_words(N, (t->sort_bits + 7) / 8));
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dalloc(&t->d_tables, t->n_tables));
  A(dalloc(&t->d_slots, slots));
  if (t->f16) A(dalloc(&t->d_wh, rows * D));
  else A(dalloc(&t->d_w, rows * D));
  if (t->n_state >= 1) A(dalloc(&t->d_s0, rows * D));
  if (t->n_state >= 2) A(dalloc(&t->d_s1, rows * D));
  A(dalloc(&t->d_row_keys, rows));
  A(dalloc(&t->d_nrows, t->n_tables));
  A(dalloc(&t->d_defaults, uint64_t(t->n_tables) * D));
  A(dalloc(&t->d_slot_table, t->n_slots));
  // load <= 1/8 (<= 2^25 entries): a home-slot CAS almost always settles an insert
  uint64_t bt_mult = 8;
  if (const char* e = std::getenv("HPS_GPU_BT_MULT")) bt_mult = std::max(2, std::atoi(e));  // A/B knob
  t->bt_mask = std::min<uint64_t>(next_pow2(bt_mult * N), 1ull << 25) - 1;
  (void)B;
  if (t->dim != t->dim_io) A(dalloc(&t->ws_io, B * D));
  if (!st) st = alloc_batch_slot(t, *t);
  t->parked.resize(1);
  t->cur = 0;
  if (st) {
    hps_gpu_table_destroy(t);
    return st;
  }
  cudaStream_t s = ctx->stream;
  HPSG_CUDA(cudaMemcpyAsync(t->d_tables, t->h_tables.data(), t->n_tables * sizeof(TableDev), cudaMemcpyHostToDevice, s));
  HPSG_CUDA(cudaMemcpyAsync(t->d_slot_table, cfg->slot_table_host, t->n_slots * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
  HPSG_CUDA(cudaMemsetAsync(t->d_nrows, 0, t->n_tables * sizeof(uint64_t), s));
  HPSG_CUDA(cudaMemsetAsync(t->d_defaults, 0, uint64_t(t->n_tables) * D * sizeof(float), s));
  k_fill_slots_empty<<<grid_for(slots, 256, kNumSMs * 32), 256, 0, s>>>(t->d_slots, slots);
  HPSG_CHECK_LAUNCH("k_fill_slots_empty");
  HPSG_CUDA(cudaStreamSynchronize(s));  // the host arrays above are caller-owned
  *out = t;
  return HPS_GPU_OK;
}

int hps_gpu_table_destroy(hps_gpu_table t) {
  if (!t) return HPS_GPU_OK;
  if (t->parked.empty()) t->parked.resize(1);
  t->parked[t->cur] = static_cast<BatchSlot&>(*t);
  for (BatchSlot& b : t->parked) {
    if (b.side) cudaStreamSynchronize(b.side);
    if (t->ctx && t->ctx->ev_last_dedup == b.ev_done) t->ctx->ev_last_dedup = nullptr;  // (about to be destroyed)
  }
  void* ptrs[] = {t->d_wh,        t->d_tables,    t->d_slots,      t->d_w,          t->d_s0,          t->d_s1,
                  t->d_row_keys,  t->d_nrows,      t->d_defaults,   t->d_slot_table,  t->ws_io,
                  t->ws_dscale};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (BatchSlot& b : t->parked) free_batch_slot(b);
  delete t;
  return HPS_GPU_OK;
}

// Pipeline depth (batch slots): depth 2 lets hps_gpu_table_prefetch record + dedup the next
// batch while the current one pools and updates. Allocates the extra slots (not a hot call).
int hps_gpu_table_set_pipeline(hps_gpu_table t, uint32_t depth) {
  if (int s = check_tbl(t)) return s;
  if (depth < 1 || depth > 4) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaSetDevice(t->ctx->device));
  while (t->parked.size() < depth) {
    BatchSlot b;
    if (int s = alloc_batch_slot(t, b)) {
      free_batch_slot(b);
      return s;
    }
    t->parked.push_back(b);
  }
  HPSG_CUDA(cudaStreamSynchronize(t->ctx->stream));
  return HPS_GPU_OK;
}

int hps_gpu_table_set_default_vector(hps_gpu_table t, uint32_t table, const float* vec_host) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (!vec_host) return HPS_GPU_E_INVALID_ARGUMENT;
  std::vector<float> v(t->dim, 0.f);  // (padding columns: zero)
  for (uint32_t j = 0; j < t->dim_io; ++j) {
    uint32_t b;
    std::memcpy(&b, vec_host + j, 4);
    if ((b & 0x7f800000u) == 0x7f800000u) return HPS_GPU_E_NON_FINITE;
    v[j] = vec_host[j];
  }
  HPSG_CUDA(cudaMemcpyAsync(t->d_defaults + uint64_t(table) * t->dim, v.data(), t->dim * sizeof(float),
                            cudaMemcpyHostToDevice, t->ctx->stream));
  HPSG_CUDA(cudaStreamSynchronize(t->ctx->stream));
  return HPS_GPU_OK;
}

int hps_gpu_table_size(hps_gpu_table t, uint32_t table, uint64_t* n_rows_host) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (!n_rows_host) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaMemcpyAsync(n_rows_host, t->d_nrows + table, sizeof(uint64_t), cudaMemcpyDeviceToHost, t->ctx->stream));
  HPSG_CUDA(cudaStreamSynchronize(t->ctx->stream));
  return HPS_GPU_OK;
}

int hps_gpu_table_insert(hps_gpu_table t, uint32_t table, const uint64_t* keys, uint64_t n, const float* rows,
                         uint64_t* rows_out) {
  if (int s = check_tbl(t)) return s;
  if (rows && n && t->dim != t->dim_io) {  // padded rows: widen the given values first
    cudaStream_t st = t->ctx->stream;
    float* tmp = nullptr;
    HPSG_CUDA(cudaMallocAsync(&tmp, n * t->dim * sizeof(float), st));
    int s = rows_widen(tmp, t->dim, rows, t->dim_io, n, st) == cudaSuccess
                ? hpsg_insert_on(t, table, keys, n, tmp, rows_out, st) : HPS_GPU_E_CUDA;
    cudaFreeAsync(tmp, st);
    return s;
  }
  return hpsg_insert_on(t, table, keys, n, rows, rows_out, t->ctx->stream);
}

}  // extern "C"

// Insert on stream `st` with the current batch slot's scratch (hps_gpu_table_insert; the
// insert-on-miss of a prefetch runs it on the slot's side stream).
int hpsg_insert_on(hps_gpu_table t, uint32_t table, const uint64_t* keys, uint64_t n, const float* rows,
                   uint64_t* rows_out, cudaStream_t st, const uint32_t* key_tables, const InsertRecord& rec) {
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || n >= (1ull << 32) - 1) return HPS_GPU_E_INVALID_ARGUMENT;
  const TableDev td = t->h_tables[table];
  uint64_t* ws_slot = nullptr;
  uint32_t* ws_pos = nullptr;
  uint8_t* ws_flag = nullptr;
  uint64_t* hdr = nullptr;  // [abort flag, new-key count, scan status x tiles, ticket]: one memset
  const uint64_t tiles = scan_tiles(n);
  // Batches up to max_keys (insert-on-miss inside a step) use the preallocated scratch;
  // larger bulk loads take stream-ordered allocations.
  const bool own = n > t->max_keys;
  if (own) {
    HPSG_CUDA(cudaMallocAsync(&ws_slot, n * sizeof(uint64_t), st));
    HPSG_CUDA(cudaMallocAsync(&ws_pos, n * sizeof(uint32_t), st));
    HPSG_CUDA(cudaMallocAsync(&ws_flag, n, st));
    HPSG_CUDA(cudaMallocAsync(&hdr, (tiles + 3) * sizeof(uint64_t), st));
  } else {
    ws_slot = t->ws_ins_slot;
    ws_pos = t->ws_ins_pos;
    ws_flag = t->ws_ins_flag;
    hdr = t->ws_ins_scan;
  }
  HPSG_CUDA(cudaMemsetAsync(hdr, 0, (tiles + 3) * sizeof(uint64_t), st));
  uint32_t* abort_flag = reinterpret_cast<uint32_t*>(hdr);
  uint64_t* d_new = hdr + 1;
  uint64_t* scan_status = hdr + 2;
  const int grid = grid_for(n, 256, kNumSMs * 32);
  if (rows) k_rows_non_finite<<<grid_for(n * t->dim, 256, kNumSMs * 32), 256, 0, st>>>(rows, n * t->dim, abort_flag,
                                                                                      t->ctx->d_status, t->f16 ? 1 : 0);
  k_insert_claim<<<grid, 256, 0, st>>>(t->d_slots, td, keys, n, ws_slot, abort_flag, t->ctx->d_status,
                                       rows == nullptr && rows_out == nullptr, key_tables, table,
                                       rec.occ_row != nullptr);
  InsertScanOp op{t->d_slots, td.slot_base, ws_slot, ws_pos, ws_flag, n, d_new, abort_flag};
  k_scan<InsertScanOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(
      op, scan_status, reinterpret_cast<uint32_t*>(scan_status + tiles));
  k_insert_commit<<<grid, 256, 0, st>>>(t->d_slots, td, table, keys, n, rows, ws_slot, ws_pos, ws_flag,
                                        d_new, t->d_nrows, t->d_w, t->d_s0, t->d_s1, t->n_state, t->a0,
                                        t->dim, t->seed, t->d_row_keys, abort_flag, t->ctx->d_status, t->d_wh);
  k_insert_finish<<<grid, 256, 0, st>>>(t->d_slots, td, table, n, ws_slot, rows_out, d_new, t->d_nrows, abort_flag,
                                        rec);
  HPSG_CHECK_LAUNCH("insert");
  if (own) {
    HPSG_CUDA(cudaFreeAsync(ws_slot, st));
    HPSG_CUDA(cudaFreeAsync(ws_pos, st));
    HPSG_CUDA(cudaFreeAsync(ws_flag, st));
    HPSG_CUDA(cudaFreeAsync(hdr, st));
  }
  return HPS_GPU_OK;
}

extern "C" {

// A/B of the probe scheme: group = 1 is hps_gpu_table_find's per-thread linear
// probe, 2/4/8 the warp-cooperative window probe.
int hps_gpu_debug_find_variant(hps_gpu_table t, uint32_t table, const uint64_t* keys, uint64_t n, uint64_t* rows_out,
                               uint32_t group) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || !rows_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const TableDev td = t->h_tables[table];
  switch (group) {
    case 1: return hps_gpu_table_find(t, table, keys, n, rows_out);
    case 2: k_find_coop<2><<<grid_for(n * 2, 256, kNumSMs * 32), 256, 0, st>>>(t->d_slots, td, keys, n, rows_out); break;
    case 4: k_find_coop<4><<<grid_for(n * 4, 256, kNumSMs * 32), 256, 0, st>>>(t->d_slots, td, keys, n, rows_out); break;
    case 8: k_find_coop<8><<<grid_for(n * 8, 256, kNumSMs * 32), 256, 0, st>>>(t->d_slots, td, keys, n, rows_out); break;
    default: return HPS_GPU_E_INVALID_ARGUMENT;
  }
  HPSG_CHECK_LAUNCH("k_find_coop");
  return HPS_GPU_OK;
}

int hps_gpu_table_find(hps_gpu_table t, uint32_t table, const uint64_t* keys, uint64_t n, uint64_t* rows_out) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || !rows_out) return HPS_GPU_E_INVALID_ARGUMENT;
  k_find<<<grid_for(n, 256, kNumSMs * 32), 256, 0, t->ctx->stream>>>(t->d_slots, t->h_tables[table], keys, n, rows_out);
  HPSG_CHECK_LAUNCH("k_find");
  return HPS_GPU_OK;
}

int hps_gpu_table_export(hps_gpu_table t, uint32_t table, uint64_t row_begin, uint64_t n, float* w, float* s0,
                         float* s1) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (row_begin + n > t->row_cap[table]) return HPS_GPU_E_INVALID_ARGUMENT;
  if (t->dim != t->dim_io && n) {  // padded rows: export at the storage stride, then narrow
    cudaStream_t st = t->ctx->stream;
    float* tmp = nullptr;
    HPSG_CUDA(cudaMallocAsync(&tmp, n * t->dim * sizeof(float), st));
    const uint32_t io = t->dim_io;
    t->dim_io = t->dim;  // (the recursive call exports unpadded)
    int s = HPS_GPU_OK;
    float* outs[3] = {w, s0, s1};
    for (int k = 0; k < 3 && !s; ++k) {
      if (!outs[k]) continue;
      s = hps_gpu_table_export(t, table, row_begin, n, k == 0 ? tmp : nullptr, k == 1 ? tmp : nullptr,
                               k == 2 ? tmp : nullptr);
      if (!s && rows_narrow(outs[k], io, tmp, t->dim, n, st) != cudaSuccess) s = HPS_GPU_E_CUDA;
    }
    t->dim_io = io;
    cudaFreeAsync(tmp, st);
    return s;
  }
  const uint64_t off = (t->row_base[table] + row_begin) * t->dim, bytes = n * t->dim * sizeof(float);
  cudaStream_t st = t->ctx->stream;
  if (w && t->f16) {  // binary16 rows widened exactly
    k_widen_half<<<grid_for(n * t->dim, 256, kNumSMs * 16), 256, 0, st>>>(t->d_wh + off, n * t->dim, w);
    HPSG_CHECK_LAUNCH("k_widen_half");
  } else if (w) {
    HPSG_CUDA(cudaMemcpyAsync(w, t->d_w + off, bytes, cudaMemcpyDeviceToDevice, st));
  }
  if (s0 && t->n_state >= 1) HPSG_CUDA(cudaMemcpyAsync(s0, t->d_s0 + off, bytes, cudaMemcpyDeviceToDevice, st));
  if (s1 && t->n_state >= 2) HPSG_CUDA(cudaMemcpyAsync(s1, t->d_s1 + off, bytes, cudaMemcpyDeviceToDevice, st));
  return HPS_GPU_OK;
}

int hps_gpu_table_row_keys(hps_gpu_table t, uint32_t table, uint64_t row_begin, uint64_t n, uint64_t* keys_out) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (row_begin + n > t->row_cap[table]) return HPS_GPU_E_INVALID_ARGUMENT;
  if (n == 0) return HPS_GPU_OK;
  if (!keys_out) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaMemcpyAsync(keys_out, t->d_row_keys + t->row_base[table] + row_begin, n * sizeof(uint64_t),
                            cudaMemcpyDeviceToDevice, t->ctx->stream));
  return HPS_GPU_OK;
}

int hps_gpu_lookup_pooled(hps_gpu_table t, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                          int combiner, float* out, uint32_t flags) {
  if (int s = check_tbl(t)) return s;
  if (combiner != HPS_COMBINER_SUM && combiner != HPS_COMBINER_MEAN) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint64_t n_bags = uint64_t(n_samples) * t->n_slots;
  if (n_bags > t->max_bags) {
    set_last_error("lookup: n_samples * n_slots exceeds max_batch_bags");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (t->dim != t->dim_io && n_bags && out) {  // padded rows: pool into the staging, then narrow
    const uint32_t io = t->dim_io;
    t->dim_io = t->dim;  // (the recursive call sees an unpadded table)
    int s = hps_gpu_lookup_pooled(t, keys, offsets, n_samples, combiner, t->ws_io, flags);
    t->dim_io = io;
    if (!s && rows_narrow(out, io, t->ws_io, t->dim, n_bags, t->ctx->stream) != cudaSuccess) s = HPS_GPU_E_CUDA;
    return s;
  }
  if (flags & HPS_LOOKUP_PREFETCHED) return lookup_prefetched(t, offsets, n_bags, combiner, out, flags);
  if (n_bags == 0) {
    t->have_train = false;
    return HPS_GPU_OK;
  }
  if (!keys || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const bool multi = offsets != nullptr;
  uint64_t n_keys_host = multi ? t->max_keys : n_bags;
  const bool train = (flags & HPS_LOOKUP_TRAIN) != 0;
  if (train && t->f16) {
    set_last_error("lookup: an F16 table is an inference table (no training lookups)");
    return HPS_GPU_E_DTYPE_MISMATCH;
  }
  const bool ins_rec = train && !multi && (flags & HPS_LOOKUP_INSERT);
  if (int s = stage_keys(t, keys, offsets, n_bags, flags, st, &n_keys_host, ins_rec)) return s;
  LookupArgs a{};
  fill_lookup_args(t, a, keys, offsets, n_bags, combiner, out);
  if (train) {
    if (int s = begin_training_record(t, a, n_keys_host, st)) return s;
    a.occ_bag = multi ? t->ws_occ_bag : nullptr;
    a.bag_len = (multi && a.mean) ? t->ws_bag_len : nullptr;
    if (int s = ins_rec ? record_by_insert(t, a, keys, n_keys_host, st) : record(t, a, multi, a.mean, n_keys_host, st))
      return s;
  }
  if (int s = launch_lookup(t, a, multi, train)) return s;
  if (train)
    if (int s = fork_dedup(t)) return s;
  t->have_train = train;
  return HPS_GPU_OK;
}

int hps_gpu_table_prefetch(hps_gpu_table t, uint32_t slot, const uint64_t* keys, const uint32_t* offsets,
                           uint32_t n_samples, int combiner, uint32_t flags) {
  if (int s = check_tbl(t)) return s;
  if (slot >= t->parked.size()) {
    set_last_error("prefetch: slot >= pipeline depth (hps_gpu_table_set_pipeline)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (combiner != HPS_COMBINER_SUM && combiner != HPS_COMBINER_MEAN) return HPS_GPU_E_INVALID_ARGUMENT;
  if (t->f16) return HPS_GPU_E_DTYPE_MISMATCH;
  if (t->no_fork) {
    set_last_error("prefetch: needs the side streams (HPS_GPU_NO_FORK is set)");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const uint64_t n_bags = uint64_t(n_samples) * t->n_slots;
  if (n_bags == 0 || n_bags > t->max_bags || !keys) {
    set_last_error("prefetch: empty batch, missing keys, or n_samples * n_slots exceeds max_batch_bags");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (slot == t->cur && t->have_train) {
    set_last_error("prefetch: the slot holds a training lookup whose backward has not run");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const uint32_t prev = t->cur;
  use_slot(t, slot);
  int s = prefetch_into_current(t, keys, offsets, n_bags, combiner, flags);
  use_slot(t, prev);
  return s;
}

int hps_gpu_table_join_prefetch(hps_gpu_table t) {
  if (int s = check_tbl(t)) return s;
  cudaStream_t st = t->ctx->stream;
  for (uint32_t k = 0; k < t->parked.size(); ++k) {
    const BatchSlot& b = k == t->cur ? static_cast<const BatchSlot&>(*t) : t->parked[k];
    if (b.dedup_pending) HPSG_CUDA(wait_recorded(st, b.ev_done, b.pre_capture));
  }
  return HPS_GPU_OK;
}

}  // extern "C"

int hpsg::table_read_through(hps_gpu_table t, uint32_t table, const uint64_t* keys, const float* found_vecs,
                             const uint32_t* found_idx, const uint32_t* missing_idx, const uint64_t* counts,
                             uint64_t n, float* out, uint64_t* miss_keys, float* miss_vecs, uint8_t* miss_absent,
                             uint8_t* src_out, bool hits_in_place) {
  // hits_in_place: the hits' rows are already at out[i] (the cache query scattered them there)
  if (t && t->dim != t->dim_io) return refuse_padded(t, "read_through");
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || (!found_vecs && !hits_in_place) || !found_idx || !missing_idx || !counts || !out || !miss_keys ||
      !miss_vecs || !miss_absent)
    return HPS_GPU_E_INVALID_ARGUMENT;
  if (hits_in_place) found_vecs = nullptr;
  const uint32_t nvec = t->dim / 4;
  const int lpr = nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
  const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
  cudaStream_t st = t->ctx->stream;
  const TableDev td = t->h_tables[table];
  const float* def = t->d_defaults + uint64_t(table) * t->dim;
  switch (lpr) {
    case 32: launch_k(true, k_read_through<32>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
    case 16: launch_k(true, k_read_through<16>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
    case 8: launch_k(true, k_read_through<8>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
    case 4: launch_k(true, k_read_through<4>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
    case 2: launch_k(true, k_read_through<2>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
    default: launch_k(true, k_read_through<1>, grid, 256, 0, st, keys, found_vecs, found_idx, missing_idx, counts, t->d_slots, td, t->d_w, def, t->dim, out, miss_keys, miss_vecs, miss_absent, t->d_wh, src_out); break;
  }
  HPSG_CHECK_LAUNCH("k_read_through");
  return HPS_GPU_OK;
}

extern "C" {

int hps_gpu_table_read_through(hps_gpu_table t, uint32_t table, const uint64_t* keys, const float* found_vecs,
                               const uint32_t* found_idx, const uint32_t* missing_idx, const uint64_t* counts,
                               uint64_t n, float* out, uint64_t* miss_keys, float* miss_vecs, uint8_t* miss_absent) {
  return table_read_through(t, table, keys, found_vecs, found_idx, missing_idx, counts, n, out, miss_keys, miss_vecs,
                            miss_absent, nullptr);
}

int hps_gpu_hybrid_probe(hps_gpu_table t, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         int combiner, uint64_t n_keys_host, uint32_t* cold_pos_out, uint64_t* cold_keys_out,
                         uint32_t* cold_bags_out, uint64_t* cold_count_out) {
  if (t && t->dim != t->dim_io) return refuse_padded(t, "hybrid_probe");
  if (int s = check_tbl(t)) return s;
  if (t->f16) return HPS_GPU_E_DTYPE_MISMATCH;  // hybrid hot tables train
  const uint64_t n_bags = uint64_t(n_samples) * t->n_slots;
  const bool multi = offsets != nullptr;
  if (!multi) n_keys_host = n_bags;
  if (n_bags > t->max_bags || n_keys_host > t->max_keys) {
    set_last_error("hybrid_probe: batch exceeds max_batch_bags / max_batch_keys");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!keys || !cold_pos_out || !cold_keys_out || !cold_bags_out || !cold_count_out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (combiner != HPS_COMBINER_SUM && combiner != HPS_COMBINER_MEAN) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  LookupArgs a{};
  if (int s = begin_training_record(t, a, n_keys_host, st)) return s;
  a.keys = keys;
  a.offsets = offsets;
  a.n_bags = static_cast<uint32_t>(n_bags);
  a.n_slots = t->n_slots;
  a.slot_table = t->d_slot_table;
  a.tables = t->d_tables;
  a.n_tables = t->n_tables;
  a.slots = t->d_slots;
  a.occ_bag = multi ? t->ws_occ_bag : nullptr;
  a.bag_len = (multi && combiner == HPS_COMBINER_MEAN) ? t->ws_bag_len : nullptr;
  if (int s = record(t, a, multi, combiner == HPS_COMBINER_MEAN, n_keys_host, st)) return s;
  if (int s = fork_dedup(t)) return s;
  // compaction scan: its look-back words live past the backward's zeroed region
  const uint64_t tiles = scan_tiles(std::max<uint64_t>(n_keys_host, 1));
  HPSG_CUDA(cudaMemsetAsync(t->ws_ins_scan, 0, (tiles + 1) * sizeof(uint64_t), st));
  ColdOp op{t->ws_rows_a, t->row_absent, keys, a.occ_bag, cold_pos_out, cold_keys_out, cold_bags_out, cold_count_out,
            t->ws_counts};
  k_scan<ColdOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(op, t->ws_ins_scan,
                                                                      reinterpret_cast<uint32_t*>(t->ws_ins_scan + tiles));
  HPSG_CHECK_LAUNCH("hybrid_probe");
  t->have_train = true;
  return HPS_GPU_OK;
}

int hps_gpu_hybrid_pool(hps_gpu_table t, const uint32_t* cold_pos, const uint32_t* perm, const float* cold_rows,
                        const uint32_t* offsets, uint64_t n_bags, int combiner, float* out) {
  if (t && t->dim != t->dim_io) return refuse_padded(t, "hybrid_pool");
  if (int s = check_tbl(t)) return s;
  if (t->f16) return HPS_GPU_E_DTYPE_MISMATCH;
  if (n_bags == 0) return HPS_GPU_OK;
  if (!cold_pos || !out || (!cold_rows && perm)) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint32_t nvec = t->dim / 4;
  const int lpr = nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
  const int grid = grid_for(n_bags * lpr, 256, kNumSMs * 16);
  cudaStream_t st = t->ctx->stream;
  const int mean = combiner == HPS_COMBINER_MEAN;
#define HPSG_HP(L)                                                                                             \
  k_hybrid_pool<L><<<grid, 256, 0, st>>>(t->ws_rows_a, t->row_absent, t->d_w, cold_pos, perm, cold_rows, offsets, \
                                         n_bags, t->dim, mean, out)
  switch (lpr) {
    case 32: HPSG_HP(32); break;
    case 16: HPSG_HP(16); break;
    case 8: HPSG_HP(8); break;
    case 4: HPSG_HP(4); break;
    case 2: HPSG_HP(2); break;
    default: HPSG_HP(1); break;
  }
#undef HPSG_HP
  HPSG_CHECK_LAUNCH("hybrid_pool");
  return HPS_GPU_OK;
}

int hps_gpu_gather_rows(hps_gpu_table t, const uint64_t* keys, const uint32_t* tables, uint64_t n, float* rows_out,
                        uint32_t flags) {
  if (t && t->dim != t->dim_io) return refuse_padded(t, "gather_rows");
  if (int s = check_tbl(t)) return s;
  if (n > t->max_keys || n > t->max_bags) {
    set_last_error("gather_rows: n exceeds max_batch_keys / max_batch_bags");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const bool train = (flags & HPS_LOOKUP_TRAIN) != 0;
  if (train && t->f16) {
    set_last_error("gather_rows: an F16 table is an inference table (no training lookups)");
    return HPS_GPU_E_DTYPE_MISMATCH;
  }
  if (n == 0) {
    t->have_train = false;
    return HPS_GPU_OK;
  }
  if (!keys || !tables || !rows_out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (flags & HPS_LOOKUP_INSERT) {  // dynamic single-table shard: materialise absent keys first
    if (t->n_tables != 1) return HPS_GPU_E_INVALID_ARGUMENT;
    // (entries of an empty exchange slot carry a table id >= n_tables: not inserted)
    if (int s = hpsg_insert_on(t, 0, keys, n, nullptr, nullptr, t->ctx->stream, tables)) return s;
  }
  LookupArgs a{};
  a.keys = keys;
  a.n_bags = static_cast<uint32_t>(n);
  a.n_slots = t->n_slots;
  a.slot_table = t->d_slot_table;
  a.key_tables = tables;
  a.tables = t->d_tables;
  a.n_tables = t->n_tables;
  a.slots = t->d_slots;
  a.W = t->d_w;
  a.Wh = t->d_wh;
  a.defaults = t->d_defaults;
  a.dim = t->dim;
  a.out = rows_out;
  if (train) {
    if (int s = begin_training_record(t, a, n, t->ctx->stream)) return s;
    if (int s = record(t, a, false, false, n, t->ctx->stream)) return s;
  }
  if (int s = launch_lookup(t, a, false, train)) return s;
  if (train)
    if (int s = fork_dedup(t)) return s;
  t->have_train = train;
  return HPS_GPU_OK;
}

}  // extern "C"
