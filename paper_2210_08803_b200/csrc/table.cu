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

using namespace hpsg;

namespace {

constexpr uint32_t kChunk = 32;  // blocked reduction width
constexpr uint64_t kNoSlot = ~0ull;

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

__global__ void k_find(const Slot* __restrict__ slots, TableDev td, const uint64_t* __restrict__ keys, uint64_t n,
                       uint64_t* __restrict__ rows_out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = probe_find(slots, td, keys[i]);
    rows_out[i] = r == kRowEmpty ? ~0ull : r;
  }
}

// Insert phase A: claim or find a slot for every occurrence (128-bit CAS gives an
// atomic snapshot of the slot, so no torn key/row reads); aux = min occurrence index.
__global__ void k_insert_claim(Slot* __restrict__ slots, TableDev td, const uint64_t* __restrict__ keys, uint64_t n,
                               uint64_t* __restrict__ ws_slot, uint32_t* __restrict__ abort_flag, uint32_t* status) {
  if (*reinterpret_cast<volatile uint32_t*>(abort_flag)) return;
  Slot* base = slots + td.slot_base;
  const Slot empty{0, kRowEmpty, kAuxNone};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[i];
    uint64_t idx = hps::key_hash(key) & td.slot_mask;
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
    if (si == kNoSlot) return 0;
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
      if (si != kNoSlot) {
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
                                uint32_t* abort_flag, uint32_t* status) {
  if (*reinterpret_cast<volatile uint32_t*>(abort_flag)) return;
  const uint64_t nrows = d_nrows[table];
  if (nrows + *d_new > td.row_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      latch_status(status, HPS_GPU_E_INFEASIBLE);
      atomicMax(abort_flag, 2u);
    }
    return;
  }
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
      float* wr = W + gr * dim;
      for (uint32_t j = lane; j < dim; j += 32) {
        wr[j] = rows ? rows[ir * dim + j] : init_value(seed, kr, j);
        if (fr & 1) {
          if (n_state >= 1) S0[gr * dim + j] = (n_state == 1) ? a0 : 0.0f;
          if (n_state >= 2) S1[gr * dim + j] = 0.0f;
        }
      }
    }
  }
}

// Insert phase D: publish rows_out, reset aux scratch (or roll the call back).
__global__ void k_insert_finish(Slot* __restrict__ slots, TableDev td, uint32_t table, uint64_t n,
                                const uint64_t* __restrict__ ws_slot, uint64_t* __restrict__ rows_out,
                                const uint64_t* __restrict__ d_new, uint64_t* __restrict__ d_nrows,
                                const uint32_t* __restrict__ abort_flag) {
  const uint32_t ab = *reinterpret_cast<const volatile uint32_t*>(abort_flag);
  Slot* base = slots + td.slot_base;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (ab == 1) {  // refused before any claim (NonFinite)
      if (rows_out) rows_out[i] = ~0ull;
      continue;
    }
    const uint64_t si = ws_slot[i];
    if (si == kNoSlot) {
      if (rows_out) rows_out[i] = ~0ull;
      continue;
    }
    Slot* s = base + si;
    if (ab) {  // roll back: drop every slot claimed by this call, release aux
      if (s->row == kRowPending) {
        *reinterpret_cast<ulonglong2*>(s) = make_ulonglong2(0ull, (uint64_t(kAuxNone) << 32) | kRowEmpty);
      } else {
        s->aux = kAuxNone;
      }
      if (rows_out) rows_out[i] = ~0ull;
    } else {
      if (rows_out) rows_out[i] = s->row;
      s->aux = kAuxNone;
    }
  }
  if (!ab && blockIdx.x == 0 && threadIdx.x == 0) d_nrows[table] += *d_new;
}

__global__ void k_rows_non_finite(const float* __restrict__ v, uint64_t n, uint32_t* abort_flag, uint32_t* status) {
  bool bad = false;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    bad |= non_finite_bits(__float_as_uint(v[i]));
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) {
    latch_status(status, HPS_GPU_E_NON_FINITE);
    atomicMax(abort_flag, 1u);
  }
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
  const TableDev* tables;
  const Slot* slots;
  const float* W;
  const float* defaults;
  uint32_t dim;
  int mean;
  float* out;
  uint32_t* occ_row;   // train: global row per key occurrence (row_absent for misses)
  uint32_t* occ_bag;   // train, multi-hot: bag of each occurrence
  uint32_t* bag_len;   // train, multi-hot mean: bag lengths
  uint32_t row_absent;
  uint64_t* d_n;       // train: number of key occurrences (device)
};

// One-key-per-bag path. A warp owns 32 consecutive bags: every lane hashes and probes
// one key (32 independent index loads in flight), then groups of LPR lanes stream the
// rows with 128-bit loads (VPL float4 per lane) and write the bag outputs coalesced.
template <int LPR>
__global__ void __launch_bounds__(256) k_lookup_1hot(LookupArgs a) {
  constexpr int G = 32 / LPR;  // rows handled side by side by one warp
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPR, gl = lane % LPR;
  const uint32_t nvec = a.dim / 4;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  if (a.d_n && warp == 0 && lane == 0) *a.d_n = a.n_bags;
  for (uint64_t t0 = warp * 32; t0 < a.n_bags; t0 += n_warps * 32) {
    const uint64_t bag = t0 + lane;
    uint32_t row = kRowEmpty, table = 0;
    if (bag < a.n_bags) {
      const uint64_t key = a.keys[bag];
      table = a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
      const TableDev td = a.tables[table];
      const uint32_t local = probe_find(a.slots, td, key);
      row = local == kRowEmpty ? kRowEmpty : static_cast<uint32_t>(td.row_base + local);
      if (a.occ_row) a.occ_row[bag] = local == kRowEmpty ? a.row_absent : row;
    }
#pragma unroll 4
    for (int m = 0; m < LPR; ++m) {
      const uint32_t src = grp + G * m;
      const uint32_t r = __shfl_sync(0xffffffffu, row, src);
      const uint32_t tb = __shfl_sync(0xffffffffu, table, src);
      const uint64_t b = t0 + src;
      if (b >= a.n_bags) continue;
      const float4* p = reinterpret_cast<const float4*>(r == kRowEmpty ? a.defaults + uint64_t(tb) * a.dim
                                                                       : a.W + uint64_t(r) * a.dim);
      float4* o = reinterpret_cast<float4*>(a.out + b * a.dim);
      for (uint32_t v = gl; v < nvec; v += LPR) {
        // +0.0f + x (and /1.0f for mean) are the identity on every finite x except -0.0.
        float4 x = ldg_stream(p + v);
        x = f4_add(make_float4(0.f, 0.f, 0.f, 0.f), x);
        o[v] = x;
      }
    }
  }
}

// Multi-hot path: a group of LPR lanes owns one bag at a time; the group probes LPR
// keys of the bag in parallel, then accumulates the rows in bag order.
template <int LPR>
__global__ void __launch_bounds__(256) k_lookup_multi(LookupArgs a) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPR, gl = lane % LPR;
  const uint32_t gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const uint32_t nvec = a.dim / 4;
  constexpr int kMaxVpl = 8;  // dim <= 32*4*8 = 1024 on this path
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t n_groups = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  if (a.d_n && gid == 0 && gl == 0) *a.d_n = a.offsets[a.n_bags];
  for (uint64_t bag = gid; bag < a.n_bags; bag += n_groups) {
    const uint32_t lo = a.offsets[bag], hi = a.offsets[bag + 1];
    const uint32_t table = a.slot_table[static_cast<uint32_t>(bag) % a.n_slots];
    const TableDev td = a.tables[table];
    float4 acc[kMaxVpl];
#pragma unroll
    for (int k = 0; k < kMaxVpl; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t c = lo; c < hi; c += LPR) {
      const uint32_t i = c + gl;
      uint32_t row = kRowEmpty;
      if (i < hi) {
        const uint32_t local = probe_find(a.slots, td, a.keys[i]);
        row = local == kRowEmpty ? kRowEmpty : static_cast<uint32_t>(td.row_base + local);
        if (a.occ_row) {
          a.occ_row[i] = local == kRowEmpty ? a.row_absent : row;
          a.occ_bag[i] = static_cast<uint32_t>(bag);
        }
      }
      const uint32_t cnt = min(uint32_t(LPR), hi - c);
      for (uint32_t m = 0; m < cnt; ++m) {
        const uint32_t r = __shfl_sync(gmask, row, grp * LPR + m);
        const float4* p = reinterpret_cast<const float4*>(r == kRowEmpty ? a.defaults + uint64_t(table) * a.dim
                                                                         : a.W + uint64_t(r) * a.dim);
#pragma unroll
        for (int k = 0; k < kMaxVpl; ++k) {
          const uint32_t v = gl + k * LPR;
          if (v < nvec) acc[k] = f4_add(acc[k], ldg_stream(p + v));
        }
      }
    }
    const uint32_t len = hi - lo;
    if (a.bag_len && gl == 0) a.bag_len[bag] = len;
    float4* o = reinterpret_cast<float4*>(a.out + bag * a.dim);
    const float fl = static_cast<float>(len);
#pragma unroll
    for (int k = 0; k < kMaxVpl; ++k) {
      const uint32_t v = gl + k * LPR;
      if (v < nvec) o[v] = (a.mean && len > 0) ? f4_div(acc[k], fl) : acc[k];
    }
  }
}

// ---------------------------------------------------------------------------------
// K4: dedup (segments of the row-sorted occurrence list) + chunk tasks
// ---------------------------------------------------------------------------------
struct SegScanOp {  // heads of equal-row runs -> seg_start[u]
  const uint32_t* rows_sorted;
  uint32_t* seg_start;
  uint64_t* counts;  // [0]=N [1]=U
  __device__ uint64_t size() const { return counts[0]; }
  __device__ uint32_t count(uint64_t i) const {
    return (i == 0 || rows_sorted[i] != rows_sorted[i - 1]) ? 1u : 0u;
  }
  __device__ void emit(uint64_t i, uint64_t excl, uint32_t c) const {
    if (c) seg_start[excl] = static_cast<uint32_t>(i);
  }
  __device__ void total(uint64_t u) const {
    counts[1] = u;
    seg_start[u] = static_cast<uint32_t>(counts[0]);
  }
};

struct TaskScanOp {  // ceil(len/kChunk) reduction tasks per segment
  const uint32_t* seg_start;
  uint32_t* task_off;
  uint32_t* task_seg;
  uint32_t* seg_done;
  uint64_t* counts;  // [1]=U [2]=T
  __device__ uint64_t size() const { return counts[1]; }
  __device__ uint32_t count(uint64_t u) const {
    const uint32_t len = seg_start[u + 1] - seg_start[u];
    return (len + kChunk - 1) / kChunk;
  }
  __device__ void emit(uint64_t u, uint64_t excl, uint32_t c) const {
    task_off[u] = static_cast<uint32_t>(excl);
    seg_done[u] = 0;
    for (uint32_t k = 0; k < c; ++k) task_seg[excl + k] = static_cast<uint32_t>(u);
  }
  __device__ void total(uint64_t t) const {
    counts[2] = t;
    task_off[counts[1]] = static_cast<uint32_t>(t);
  }
};

struct ReduceArgs {
  const uint32_t* rows_sorted;
  const uint32_t* bags_sorted;
  const uint32_t* seg_start;
  const uint32_t* task_off;
  const uint32_t* task_seg;
  uint32_t* seg_done;
  const uint64_t* counts;
  const float* dout;
  const uint32_t* bag_len;  // mean: length of each bag (nullptr: every bag has length 1)
  int mean;
  float* partial;  // [T x dim]
  float* W;
  float* S0;
  float* S1;
  int optimizer;
  hps_opt_params opt;
  uint32_t dim;
  uint32_t row_absent;
};

template <int VPL>
__device__ __forceinline__ void apply_opt(const ReduceArgs& a, uint32_t row, const float4 (&g)[VPL], uint32_t gl,
                                          uint32_t lpr, uint32_t nvec) {
  float4* w = reinterpret_cast<float4*>(a.W + uint64_t(row) * a.dim);
  const float lr = a.opt.lr, eps = a.opt.eps;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t v = gl + k * lpr;
    if (v >= nvec) break;
    float4 wv = w[v];
    float* wf = reinterpret_cast<float*>(&wv);
    const float* gf = reinterpret_cast<const float*>(&g[k]);
    if (a.optimizer == HPS_OPT_SGD) {
#pragma unroll
      for (int c = 0; c < 4; ++c) wf[c] = __fsub_rn(wf[c], __fmul_rn(lr, gf[c]));
    } else if (a.optimizer == HPS_OPT_ADAGRAD) {
      float4* s = reinterpret_cast<float4*>(a.S0 + uint64_t(row) * a.dim);
      float4 sv = s[v];
      float* sf = reinterpret_cast<float*>(&sv);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sf[c] = __fadd_rn(sf[c], __fmul_rn(gf[c], gf[c]));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(lr, gf[c]), __fadd_rn(__fsqrt_rn(sf[c]), eps)));
      }
      s[v] = sv;
    } else {
      float4* m = reinterpret_cast<float4*>(a.S0 + uint64_t(row) * a.dim);
      float4* q = reinterpret_cast<float4*>(a.S1 + uint64_t(row) * a.dim);
      float4 mv = m[v], qv = q[v];
      float* mf = reinterpret_cast<float*>(&mv);
      float* qf = reinterpret_cast<float*>(&qv);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        mf[c] = __fadd_rn(__fmul_rn(a.opt.beta1, mf[c]), __fmul_rn(a.opt.one_minus_beta1, gf[c]));
        qf[c] = __fadd_rn(__fmul_rn(a.opt.beta2, qf[c]), __fmul_rn(a.opt.one_minus_beta2, __fmul_rn(gf[c], gf[c])));
        wf[c] = __fsub_rn(wf[c], __fdiv_rn(__fmul_rn(a.opt.lr_t, mf[c]), __fadd_rn(__fsqrt_rn(qf[c]), eps)));
      }
      m[v] = mv;
      q[v] = qv;
    }
    w[v] = wv;
  }
}

// K4+K5 fused: one LPR-lane group per reduction task (a chunk of <= kChunk occurrences
// of one unique row). Single-chunk segments update their row directly; the last
// finishing chunk of a multi-chunk segment sums the chunk partials in order and updates.
template <int LPR, int VPL>
__global__ void __launch_bounds__(256) k_reduce_update(ReduceArgs a) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPR, gl = lane % LPR;
  const uint32_t gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const uint32_t nvec = a.dim / 4;
  const uint64_t T = a.counts[2];
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t n_groups = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t t = gid; t < T; t += n_groups) {
    const uint32_t u = a.task_seg[t];
    const uint32_t toff = a.task_off[u];
    const uint32_t m = a.task_off[u + 1] - toff;
    const uint32_t s0 = a.seg_start[u], s1 = a.seg_start[u + 1];
    const uint32_t row = a.rows_sorted[s0];
    if (row == a.row_absent) continue;
    const uint32_t lo = s0 + (static_cast<uint32_t>(t) - toff) * kChunk;
    const uint32_t hi = min(s1, lo + kChunk);
    float4 acc[VPL];
    for (uint32_t c = lo; c < hi; c += LPR) {
      const uint32_t i = c + gl;
      const uint32_t my_bag = i < hi ? a.bags_sorted[i] : 0u;
      float my_len = 1.0f;
      if (a.mean && i < hi) my_len = static_cast<float>(a.bag_len ? a.bag_len[my_bag] : 1u);
      const uint32_t cnt = min(uint32_t(LPR), hi - c);
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t b = __shfl_sync(gmask, my_bag, grp * LPR + q);
        const float fl = __shfl_sync(gmask, my_len, grp * LPR + q);
        const float4* d = reinterpret_cast<const float4*>(a.dout + uint64_t(b) * a.dim);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const uint32_t v = gl + k * LPR;
          if (v < nvec) {
            float4 x = __ldg(d + v);
            if (a.mean) x = f4_div(x, fl);
            acc[k] = (c == lo && q == 0) ? x : f4_add(acc[k], x);
          }
        }
      }
    }
    if (m == 1) {
      apply_opt<VPL>(a, row, acc, gl, LPR, nvec);
      continue;
    }
    float4* part = reinterpret_cast<float4*>(a.partial + uint64_t(t) * a.dim);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t v = gl + k * LPR;
      if (v < nvec) __stcg(part + v, acc[k]);
    }
    __threadfence();
    __syncwarp(gmask);
    uint32_t prev = 0;
    if (gl == 0) prev = atomicAdd(&a.seg_done[u], 1u);
    prev = __shfl_sync(gmask, prev, grp * LPR);
    if (prev != m - 1) continue;
    __threadfence();
    for (uint32_t j = 0; j < m; ++j) {
      const float4* pj = reinterpret_cast<const float4*>(a.partial + uint64_t(toff + j) * a.dim);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const uint32_t v = gl + k * LPR;
        if (v < nvec) {
          const float4 x = __ldcg(pj + v);
          acc[k] = j == 0 ? x : f4_add(acc[k], x);
        }
      }
    }
    apply_opt<VPL>(a, row, acc, gl, LPR, nvec);
  }
}

__global__ void k_unique_rows(const uint32_t* rows_sorted, const uint32_t* seg_start, const uint64_t* counts,
                              uint32_t row_absent, uint32_t* out, uint64_t* count_out) {
  const uint64_t U = counts[1];
  const bool has_absent = U > 0 && rows_sorted[seg_start[U - 1]] == row_absent;
  const uint64_t n = has_absent ? U - 1 : U;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_out = n;
  if (!out) return;
  for (uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; u < n; u += uint64_t(gridDim.x) * blockDim.x)
    out[u] = rows_sorted[seg_start[u]];
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

struct hps_gpu_table_s {
  hps_gpu_ctx ctx = nullptr;
  uint32_t n_tables = 0, dim = 0, n_slots = 0;
  int optimizer = 0, n_state = 0;
  uint64_t seed = 0;
  float a0 = 0.f;
  std::vector<uint64_t> row_cap, row_base, slot_cap, slot_base;
  std::vector<TableDev> h_tables;
  uint64_t total_rows = 0, total_slots = 0;
  uint32_t row_absent = 0;
  int sort_bits = 0;
  uint64_t max_keys = 0, max_bags = 0;
  // device state
  TableDev* d_tables = nullptr;
  Slot* d_slots = nullptr;
  float *d_w = nullptr, *d_s0 = nullptr, *d_s1 = nullptr;
  uint64_t* d_row_keys = nullptr;
  uint64_t* d_nrows = nullptr;
  float* d_defaults = nullptr;
  uint32_t* d_slot_table = nullptr;
  // per-batch workspaces (sized at create)
  uint32_t *ws_rows_a = nullptr, *ws_rows_b = nullptr, *ws_bags_a = nullptr, *ws_bags_b = nullptr;
  uint32_t* ws_occ_bag = nullptr;
  uint32_t* ws_bag_len = nullptr;
  uint32_t *ws_seg_start = nullptr, *ws_task_off = nullptr, *ws_task_seg = nullptr, *ws_seg_done = nullptr;
  float* ws_partial = nullptr;
  uint64_t* ws_counts = nullptr;  // [0]=N [1]=U [2]=T [3]=insert new-count
  uint32_t* ws_zero = nullptr;     // sort + scan look-back words, memset per backward
  size_t ws_zero_words = 0;
  uint32_t* ws_abort = nullptr;
  uint64_t* ws_keys_stage = nullptr;
  uint32_t* ws_offsets_stage = nullptr;
  // last training lookup
  bool have_train = false, last_multi = false;
  int last_combiner = 0;
  uint64_t last_n_keys_host = 0;  // exact when known on the host, else max_keys
  bool sorted_in_b = false;
};

namespace {

int check_tbl(hps_gpu_table t) {
  if (!t) {
    set_last_error("null table handle");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  return HPS_GPU_OK;
}

// Words of the zeroed look-back region: sort workspace + 2 scans (status u64 each) + tickets.
size_t zero_words(uint64_t max_keys, int passes) {
  return sort_ws_words(max_keys, passes) + 2 * 2 * scan_tiles(max_keys + 1) + 8;
}

int launch_lookup(hps_gpu_table t, const LookupArgs& a, bool multi) {
  const cudaStream_t st = t->ctx->stream;
  const uint32_t nvec = t->dim / 4;
  const int block = 256;
  if (!multi) {
    const uint64_t warps = (a.n_bags + 31) / 32;
    const int grid = grid_for(warps * 32, block, kNumSMs * 64);
#define HPSG_L1(L) k_lookup_1hot<L><<<grid, block, 0, st>>>(a)
    if (nvec >= 32) HPSG_L1(32);
    else if (nvec >= 16) HPSG_L1(16);
    else if (nvec >= 8) HPSG_L1(8);
    else if (nvec >= 4) HPSG_L1(4);
    else if (nvec >= 2) HPSG_L1(2);
    else HPSG_L1(1);
#undef HPSG_L1
  } else {
    auto groups_grid = [&](int lpr) {
      const uint64_t groups_per_block = (block / 32) * (32 / lpr);
      uint64_t g = (a.n_bags + groups_per_block - 1) / groups_per_block;
      return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, kNumSMs * 64)));
    };
#define HPSG_LM(L) k_lookup_multi<L><<<groups_grid(L), block, 0, st>>>(a)
    if (nvec >= 32) HPSG_LM(32);
    else if (nvec >= 16) HPSG_LM(16);
    else if (nvec >= 8) HPSG_LM(8);
    else if (nvec >= 4) HPSG_LM(4);
    else if (nvec >= 2) HPSG_LM(2);
    else HPSG_LM(1);
#undef HPSG_LM
  }
  HPSG_CHECK_LAUNCH("lookup");
  return HPS_GPU_OK;
}

template <int LPR, int VPL>
void launch_reduce_t(const ReduceArgs& a, cudaStream_t st, uint64_t max_tasks) {
  const uint64_t groups_per_block = 8 * (32 / LPR);
  const uint64_t g = (max_tasks + groups_per_block - 1) / groups_per_block;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, kNumSMs * 16)));
  k_reduce_update<LPR, VPL><<<grid, 256, 0, st>>>(a);
}

int launch_reduce(hps_gpu_table t, const ReduceArgs& a, uint64_t max_tasks) {
  const cudaStream_t st = t->ctx->stream;
  const uint32_t nvec = t->dim / 4;
  if (nvec > 32 * 8) {
    set_last_error("dim > 1024 not supported by the reduce kernel");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (nvec > 128) launch_reduce_t<32, 8>(a, st, max_tasks);
  else if (nvec > 64) launch_reduce_t<32, 4>(a, st, max_tasks);
  else if (nvec > 32) launch_reduce_t<32, 2>(a, st, max_tasks);
  else if (nvec > 16) launch_reduce_t<32, 1>(a, st, max_tasks);
  else if (nvec > 8) launch_reduce_t<16, 1>(a, st, max_tasks);
  else if (nvec > 4) launch_reduce_t<8, 1>(a, st, max_tasks);
  else if (nvec > 2) launch_reduce_t<4, 1>(a, st, max_tasks);
  else if (nvec > 1) launch_reduce_t<2, 1>(a, st, max_tasks);
  else launch_reduce_t<1, 1>(a, st, max_tasks);
  HPSG_CHECK_LAUNCH("reduce");
  return HPS_GPU_OK;
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
  if (cfg->dim == 0 || cfg->dim > 1024 || cfg->dim % 4 != 0) {
    set_last_error("table config: dim must be a multiple of 4 in [4, 1024]");
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
  auto t = new hps_gpu_table_s;
  t->ctx = ctx;
  t->n_tables = cfg->n_tables;
  t->dim = cfg->dim;
  t->n_slots = cfg->n_slots;
  t->optimizer = cfg->optimizer;
  t->n_state = cfg->optimizer == HPS_OPT_SGD ? 0 : cfg->optimizer == HPS_OPT_ADAGRAD ? 1 : 2;
  t->seed = cfg->init_seed;
  t->a0 = cfg->adagrad_initial_accumulator;
  t->max_keys = cfg->max_batch_keys;
  t->max_bags = cfg->max_batch_bags;
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
  t->row_absent = static_cast<uint32_t>(rows);
  t->sort_bits = std::max(1, bits_for(rows));
  const uint64_t D = t->dim, N = t->max_keys, B = t->max_bags;
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dalloc(&t->d_tables, t->n_tables));
  A(dalloc(&t->d_slots, slots));
  A(dalloc(&t->d_w, rows * D));
  if (t->n_state >= 1) A(dalloc(&t->d_s0, rows * D));
  if (t->n_state >= 2) A(dalloc(&t->d_s1, rows * D));
  A(dalloc(&t->d_row_keys, rows));
  A(dalloc(&t->d_nrows, t->n_tables));
  A(dalloc(&t->d_defaults, uint64_t(t->n_tables) * D));
  A(dalloc(&t->d_slot_table, t->n_slots));
  A(dalloc(&t->ws_rows_a, N));
  A(dalloc(&t->ws_rows_b, N));
  A(dalloc(&t->ws_bags_a, N));
  A(dalloc(&t->ws_bags_b, N));
  A(dalloc(&t->ws_occ_bag, N));
  A(dalloc(&t->ws_bag_len, B));
  A(dalloc(&t->ws_seg_start, N + 2));
  A(dalloc(&t->ws_task_off, N + 2));
  A(dalloc(&t->ws_task_seg, N + 1));
  A(dalloc(&t->ws_seg_done, N + 1));
  A(dalloc(&t->ws_partial, N * D));
  A(dalloc(&t->ws_counts, 8));
  t->ws_zero_words = zero_words(N, (t->sort_bits + 7) / 8);
  A(dalloc(&t->ws_zero, t->ws_zero_words));
  A(dalloc(&t->ws_abort, 4));
  A(dalloc(&t->ws_keys_stage, N));
  A(dalloc(&t->ws_offsets_stage, B + 1));
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
  HPSG_CUDA(cudaMemsetAsync(t->ws_counts, 0, 8 * sizeof(uint64_t), s));
  k_fill_slots_empty<<<grid_for(slots, 256, kNumSMs * 32), 256, 0, s>>>(t->d_slots, slots);
  HPSG_CHECK_LAUNCH("k_fill_slots_empty");
  HPSG_CUDA(cudaStreamSynchronize(s));  // the host arrays above are caller-owned
  *out = t;
  return HPS_GPU_OK;
}

int hps_gpu_table_destroy(hps_gpu_table t) {
  if (!t) return HPS_GPU_OK;
  void* ptrs[] = {t->d_tables,   t->d_slots,      t->d_w,         t->d_s0,         t->d_s1,
                  t->d_row_keys, t->d_nrows,      t->d_defaults,  t->d_slot_table, t->ws_rows_a,
                  t->ws_rows_b,  t->ws_bags_a,    t->ws_bags_b,   t->ws_occ_bag,   t->ws_bag_len,
                  t->ws_seg_start, t->ws_task_off, t->ws_task_seg, t->ws_seg_done, t->ws_partial,
                  t->ws_counts,  t->ws_zero,      t->ws_abort,    t->ws_keys_stage, t->ws_offsets_stage};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete t;
  return HPS_GPU_OK;
}

int hps_gpu_table_set_default_vector(hps_gpu_table t, uint32_t table, const float* vec_host) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (!vec_host) return HPS_GPU_E_INVALID_ARGUMENT;
  for (uint32_t j = 0; j < t->dim; ++j) {
    uint32_t b;
    std::memcpy(&b, vec_host + j, 4);
    if ((b & 0x7f800000u) == 0x7f800000u) return HPS_GPU_E_NON_FINITE;
  }
  HPSG_CUDA(cudaMemcpyAsync(t->d_defaults + uint64_t(table) * t->dim, vec_host, t->dim * sizeof(float),
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
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || n >= (1ull << 32) - 1) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const TableDev td = t->h_tables[table];
  uint64_t* ws_slot = nullptr;
  uint32_t* ws_pos = nullptr;
  uint8_t* ws_flag = nullptr;
  uint64_t* scan_status = nullptr;
  const uint64_t tiles = scan_tiles(n);
  // Insert is a bulk/setup call, not a hot call: its scratch is stream-ordered.
  HPSG_CUDA(cudaMallocAsync(&ws_slot, n * sizeof(uint64_t), st));
  HPSG_CUDA(cudaMallocAsync(&ws_pos, n * sizeof(uint32_t), st));
  HPSG_CUDA(cudaMallocAsync(&ws_flag, n, st));
  HPSG_CUDA(cudaMallocAsync(&scan_status, (tiles + 1) * sizeof(uint64_t), st));
  HPSG_CUDA(cudaMemsetAsync(scan_status, 0, (tiles + 1) * sizeof(uint64_t), st));
  HPSG_CUDA(cudaMemsetAsync(t->ws_abort, 0, sizeof(uint32_t), st));
  HPSG_CUDA(cudaMemsetAsync(t->ws_counts + 3, 0, sizeof(uint64_t), st));
  const int grid = grid_for(n, 256, kNumSMs * 32);
  if (rows) k_rows_non_finite<<<grid_for(n * t->dim, 256, kNumSMs * 32), 256, 0, st>>>(rows, n * t->dim, t->ws_abort,
                                                                                      t->ctx->d_status);
  k_insert_claim<<<grid, 256, 0, st>>>(t->d_slots, td, keys, n, ws_slot, t->ws_abort, t->ctx->d_status);
  InsertScanOp op{t->d_slots, td.slot_base, ws_slot, ws_pos, ws_flag, n, t->ws_counts + 3, t->ws_abort};
  k_scan<InsertScanOp><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(
      op, scan_status, reinterpret_cast<uint32_t*>(scan_status + tiles));
  k_insert_commit<<<grid, 256, 0, st>>>(t->d_slots, td, table, keys, n, rows, ws_slot, ws_pos, ws_flag,
                                        t->ws_counts + 3, t->d_nrows, t->d_w, t->d_s0, t->d_s1, t->n_state, t->a0,
                                        t->dim, t->seed, t->d_row_keys, t->ws_abort, t->ctx->d_status);
  k_insert_finish<<<grid, 256, 0, st>>>(t->d_slots, td, table, n, ws_slot, rows_out, t->ws_counts + 3, t->d_nrows,
                                        t->ws_abort);
  HPSG_CHECK_LAUNCH("insert");
  HPSG_CUDA(cudaFreeAsync(ws_slot, st));
  HPSG_CUDA(cudaFreeAsync(ws_pos, st));
  HPSG_CUDA(cudaFreeAsync(ws_flag, st));
  HPSG_CUDA(cudaFreeAsync(scan_status, st));
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
  const uint64_t off = (t->row_base[table] + row_begin) * t->dim, bytes = n * t->dim * sizeof(float);
  cudaStream_t st = t->ctx->stream;
  if (w) HPSG_CUDA(cudaMemcpyAsync(w, t->d_w + off, bytes, cudaMemcpyDeviceToDevice, st));
  if (s0 && t->n_state >= 1) HPSG_CUDA(cudaMemcpyAsync(s0, t->d_s0 + off, bytes, cudaMemcpyDeviceToDevice, st));
  if (s1 && t->n_state >= 2) HPSG_CUDA(cudaMemcpyAsync(s1, t->d_s1 + off, bytes, cudaMemcpyDeviceToDevice, st));
  return HPS_GPU_OK;
}

int hps_gpu_table_row_keys(hps_gpu_table t, uint32_t table, uint64_t row_begin, uint64_t n, uint64_t* keys_out) {
  if (int s = check_tbl(t)) return s;
  if (table >= t->n_tables) return HPS_GPU_E_UNKNOWN_TABLE;
  if (row_begin + n > t->row_cap[table] || !keys_out) return HPS_GPU_E_INVALID_ARGUMENT;
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
  if (n_bags == 0) {
    t->have_train = false;
    return HPS_GPU_OK;
  }
  if (!keys || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const bool multi = offsets != nullptr;
  uint64_t n_keys_host = multi ? t->max_keys : n_bags;
  if (flags & HPS_LOOKUP_KEYS_HOST) {
    // Host buffers: stage H2D on the table's stream (pinned memory -> async copy).
    n_keys_host = multi ? offsets[n_bags] : n_bags;
    if (n_keys_host > t->max_keys) return HPS_GPU_E_INVALID_ARGUMENT;
    HPSG_CUDA(cudaMemcpyAsync(t->ws_keys_stage, keys, n_keys_host * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    if (multi)
      HPSG_CUDA(cudaMemcpyAsync(t->ws_offsets_stage, offsets, (n_bags + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    keys = t->ws_keys_stage;
    if (multi) offsets = t->ws_offsets_stage;
  } else if (!multi && n_bags > t->max_keys) {
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const bool train = (flags & HPS_LOOKUP_TRAIN) != 0;
  LookupArgs a{};
  a.keys = keys;
  a.offsets = offsets;
  a.n_bags = static_cast<uint32_t>(n_bags);
  a.n_slots = t->n_slots;
  a.slot_table = t->d_slot_table;
  a.tables = t->d_tables;
  a.slots = t->d_slots;
  a.W = t->d_w;
  a.defaults = t->d_defaults;
  a.dim = t->dim;
  a.mean = combiner == HPS_COMBINER_MEAN;
  a.out = out;
  a.row_absent = t->row_absent;
  if (train) {
    a.occ_row = t->ws_rows_a;
    a.occ_bag = multi ? t->ws_occ_bag : nullptr;
    a.bag_len = (multi && a.mean) ? t->ws_bag_len : nullptr;
    a.d_n = t->ws_counts;
  }
  if (int s = launch_lookup(t, a, multi)) return s;
  t->have_train = train;
  t->last_multi = multi;
  t->last_combiner = combiner;
  t->last_n_keys_host = n_keys_host;
  return HPS_GPU_OK;
}

int hps_gpu_backward_update(hps_gpu_table t, const float* d_out, const hps_opt_params* opt) {
  if (int s = check_tbl(t)) return s;
  if (!opt) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!t->have_train) {
    set_last_error("backward_update: no preceding lookup_pooled with HPS_LOOKUP_TRAIN");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (!d_out) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = t->ctx->stream;
  const uint64_t nk = t->last_n_keys_host;
  const int passes = (t->sort_bits + 7) / 8;
  uint32_t* z = t->ws_zero;
  const size_t sort_words = sort_ws_words(nk, passes);
  const uint64_t tiles = scan_tiles(nk + 1);
  uint64_t* scan1 = reinterpret_cast<uint64_t*>(z + ((sort_words + 1) & ~size_t(1)));
  uint64_t* scan2 = scan1 + tiles;
  uint32_t* tickets = reinterpret_cast<uint32_t*>(scan2 + tiles);
  const size_t used_words = reinterpret_cast<uint32_t*>(tickets + 4) - z;
  HPSG_CUDA(cudaMemsetAsync(z, 0, used_words * sizeof(uint32_t), st));
  // K4a: stable sort of (global row, bag) by row. Identity payload for one-hot bags.
  cudaError_t err;
  const uint32_t* bag_in = t->last_multi ? t->ws_occ_bag : nullptr;
  // sort workspace lives at the head of the zeroed region (already cleared above)
  {
    const uint64_t stiles = sort_tiles(nk);
    uint32_t* hist = z;
    uint32_t* stick = z + 4 * 256;
    uint32_t* status = stick + 4;
    k_radix_hist<<<grid_for(nk, 256, kNumSMs * 2), 256, 0, st>>>(t->ws_rows_a, t->ws_counts, passes, hist);
    const uint32_t* kin = t->ws_rows_a;
    const uint32_t* vin = bag_in;
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
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_status(err, "radix sort");
  }
  const uint32_t* rows_sorted = t->sorted_in_b ? t->ws_rows_b : t->ws_rows_a;
  const uint32_t* bags_sorted = t->sorted_in_b ? t->ws_bags_b : t->ws_bags_a;
  // K4b: segments (unique rows) and chunk tasks.
  SegScanOp sop{rows_sorted, t->ws_seg_start, t->ws_counts};
  k_scan<SegScanOp><<<static_cast<unsigned>(scan_tiles(nk)), kScanBlock, 0, st>>>(sop, scan1, tickets);
  TaskScanOp top{t->ws_seg_start, t->ws_task_off, t->ws_task_seg, t->ws_seg_done, t->ws_counts};
  k_scan<TaskScanOp><<<static_cast<unsigned>(scan_tiles(nk)), kScanBlock, 0, st>>>(top, scan2, tickets + 1);
  HPSG_CHECK_LAUNCH("dedup scans");
  // K4c + K5: blocked reduction fused with the optimizer.
  ReduceArgs ra{};
  ra.rows_sorted = rows_sorted;
  ra.bags_sorted = bags_sorted;
  ra.seg_start = t->ws_seg_start;
  ra.task_off = t->ws_task_off;
  ra.task_seg = t->ws_task_seg;
  ra.seg_done = t->ws_seg_done;
  ra.counts = t->ws_counts;
  ra.dout = d_out;
  ra.mean = t->last_combiner == HPS_COMBINER_MEAN && t->last_multi;
  ra.bag_len = ra.mean ? t->ws_bag_len : nullptr;
  ra.partial = t->ws_partial;
  ra.W = t->d_w;
  ra.S0 = t->d_s0;
  ra.S1 = t->d_s1;
  ra.optimizer = t->optimizer;
  ra.opt = *opt;
  ra.dim = t->dim;
  ra.row_absent = t->row_absent;
  return launch_reduce(t, ra, nk);
}

int hps_gpu_table_last_unique(hps_gpu_table t, uint64_t* count_out, uint32_t* unique_rows_out) {
  if (int s = check_tbl(t)) return s;
  if (!count_out) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint32_t* rows_sorted = t->sorted_in_b ? t->ws_rows_b : t->ws_rows_a;
  k_unique_rows<<<grid_for(t->last_n_keys_host, 256, kNumSMs * 8), 256, 0, t->ctx->stream>>>(
      rows_sorted, t->ws_seg_start, t->ws_counts, t->row_absent, unique_rows_out, count_out);
  HPSG_CHECK_LAUNCH("k_unique_rows");
  return HPS_GPU_OK;
}

}  // extern "C"
