// sharded.cu — distributed slot placement behind the C-ABI: one training step of a table
// group sharded over the ranks of an NCCL communicator, with no host round trip.
//
// Placement: key k is owned by rank
// partition_of(k, G) (proj/include/hps/hash.hpp:52-54); every rank holds that shard of every
// table (a table group created by the caller). One step, all on the context's stream:
//
//   requester  bucketize the occurrences by owner, stably (exchange.cu xplan)
//              pack them into FIXED-capacity per-peer regions [G x C] (keys, table ids);
//              empty slots carry table id UINT32_MAX
//   NCCL       one grouped all-to-all: keys + table ids (2 x C per peer)
//   owner      gather the rows of all G x C received slots (training record; empty slots
//              read as absent keys: no row, no gradient)
//   NCCL       rows back (C x dim per peer)
//   requester  pool bags straight from the received rows (perm: occurrence -> slot)
//   backward   requester scatters per-occurrence gradients into the same slots; NCCL;
//              the owner's ordinary backward (dedup + blocked reduction + optimizer)
//
// Fixed capacity instead of exact sizes: the per-peer counts never travel to the host, so
// the whole step is one stream of device work — capturable into one CUDA graph with its
// NCCL nodes. C = min(max_keys, ceil(f * max_keys / G) + 1024): hash placement puts
// max_keys/G +- sqrt(max_keys/G) occurrences on each owner, so f = 1.25 leaves > 15 sigma
// at config 2. A batch that overflows a region is refused on the device (latched
// Infeasible; the step's results are then unspecified) instead of overrunning.
// Ordering: slot p*C + r holds requester p's r-th occurrence for this owner in requester
// order, so the owner sees every key's occurrences in global canonical order (ranks in
// order, each rank's own order): the sharded step is bit-identical to one table over the
// concatenated global batch. World of one: the regions alias (no copy, no NCCL call).
#include <nccl.h>

#include <algorithm>
#include <barrier>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"

using namespace hpsg;

struct hps_gpu_dist_s {
  hps_gpu_ctx ctx = nullptr;
  hps_gpu_table shard = nullptr;
  hps_gpu_xplan plan = nullptr;
  uint32_t n_slots = 0, dim = 0, G = 1, rank = 0;
  uint64_t max_keys = 0, max_bags = 0, C = 0;
  uint32_t* d_slot_table = nullptr;
  // requester side
  uint64_t* dense_keys = nullptr;  // bucketize output (stable by owner)
  uint32_t* dense_tables = nullptr;
  uint32_t* dense_perm = nullptr;  // occurrence -> dense send position
  uint32_t* counts = nullptr;      // per owner
  uint32_t* occ_bag = nullptr;
  uint32_t* perm = nullptr;        // occurrence -> slot p*C + r
  uint64_t* send_keys = nullptr;   // [G x C]
  uint32_t* send_tables = nullptr;
  float* rows_back = nullptr;      // [G x C x dim] received rows
  float* grads_send = nullptr;     // [G x C x dim]
  // owner side
  uint64_t* recv_keys = nullptr;
  uint32_t* recv_tables = nullptr;
  float* rows_own = nullptr;       // [G x C x dim]
  float* grads_recv = nullptr;
  // loopback transport (hps_gpu_dist_create_loopback): ranks of one process on one device
  std::shared_ptr<struct LoopGroup> loop;
  cudaEvent_t loop_ev = nullptr;
  // peer-memory transport (hps_gpu_dist_set_transport(HPS_DIST_PEER)): no all-to-all calls —
  // the requester's kernels store keys/tables and gradients straight into the owners'
  // regions and the pooling loads rows straight from the owners' gathered rows
  int transport = HPS_DIST_NCCL;
  struct PeerTab* peer = nullptr;       // host copy of the peer pointer table
  uint64_t* flags = nullptr;            // [3 x G] epochs this rank's peers signal into
  uint64_t* d_epoch = nullptr;          // step counter (device: graph replays advance it)
  std::vector<void*> ipc_opened;        // peer buffers opened through CUDA IPC (NCCL mode)
  // per-destination unique rows (peer transport): the owner maps every received slot to the
  // first slot of the same (table, key) in its requester's region (lead); the requester copies
  // only those leaders' rows over NVLink (into rows_back) and pools locally (perm_u)
  uint32_t* lead = nullptr;             // [G x C] owner side: slot -> leader slot (same region)
  uint32_t* lead_ent = nullptr;         // [G x C] slot -> its hash entry (kNoLead: empty slot)
  uint2* lead_ht = nullptr;             // {claimer slot + 1, min slot}, zero / UINT32_MAX at rest
  uint64_t lead_mask = 0;
  uint32_t* perm_u = nullptr;           // requester: occurrence -> its leader's slot in rows_back
  unsigned long long* d_served = nullptr;  // cumulative unique rows served to requesters (peer)
  // last forward
  const uint32_t* last_offsets = nullptr;
  uint64_t last_bags = 0;
  int last_combiner = 0;
  bool have_fwd = false, train = false;
};

// Every peer's owner-side buffers, as device pointers of this rank (its own: plain pointers;
// a peer's: CUDA-IPC mappings over NVLink, or, for loopback ranks, the same device's memory).
constexpr uint32_t kMaxPeers = 64;
struct PeerTab {
  uint64_t* keys[kMaxPeers];
  uint32_t* tables[kMaxPeers];
  float* rows[kMaxPeers];
  float* grads[kMaxPeers];
  uint64_t* flags[kMaxPeers];
  uint32_t* lead[kMaxPeers];
};

// A group of loopback ranks: the all-to-all is device copies between their buffers, each
// rank's calls on its own host thread (the test harness of the multi-rank path on one GPU).
struct LoopGroup {
  explicit LoopGroup(uint32_t n) : bar(static_cast<std::ptrdiff_t>(n)), members(n, nullptr) {}
  std::barrier<> bar;
  std::vector<hps_gpu_dist_s*> members;
};

namespace {

// Fixed-capacity regions from the dense bucketized order: slot p*C + r <- dense start_p + r
// (r < count_p), empty slots get table id UINT32_MAX; perm[i] = p*C + (dense_perm[i] - start_p).
__global__ void k_fix_regions(const uint64_t* __restrict__ dense_keys, const uint32_t* __restrict__ dense_tables,
                              const uint32_t* __restrict__ dense_perm, const uint32_t* __restrict__ counts, uint32_t G,
                              uint64_t C, uint64_t n, uint64_t* __restrict__ send_keys,
                              uint32_t* __restrict__ send_tables, uint32_t* __restrict__ perm, uint32_t* status) {
  __shared__ uint64_t s_start[257];
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (uint32_t p = 0; p < G; ++p) {
      s_start[p] = run;
      run += counts[p];
    }
    s_start[G] = run;
  }
  __syncthreads();
  const uint64_t total = uint64_t(G) * C;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < total; q += stride) {
    const uint32_t p = static_cast<uint32_t>(q / C);
    const uint64_t r = q - uint64_t(p) * C;
    const uint64_t cnt = s_start[p + 1] - s_start[p];
    if (r < cnt) {
      send_keys[q] = dense_keys[s_start[p] + r];
      send_tables[q] = dense_tables[s_start[p] + r];
    } else {
      send_keys[q] = 0;
      send_tables[q] = 0xffffffffu;
    }
    if (r == 0 && cnt > C) latch_status(status, HPS_GPU_E_INFEASIBLE);  // region overflow
  }
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t d = dense_perm[i];
    uint32_t p = 0;
    while (p + 1 < G && s_start[p + 1] <= d) ++p;
    const uint64_t r = d - s_start[p];
    // an occurrence past its region's capacity (Infeasible is latched: the step's results are
    // unspecified) is pointed at the region's last slot, so nothing reads or writes out of bounds
    perm[i] = static_cast<uint32_t>(uint64_t(p) * C + (r < C ? r : C - 1));
  }
}

// ---- peer-memory transport --------------------------------------------------------------
// Fixed regions stored straight into the owners: this rank's region p goes to rank p's
// receive buffers at [rank * C, +C) (stores over NVLink), perm as in k_fix_regions.
__global__ void k_fix_regions_peer(const uint64_t* __restrict__ dense_keys, const uint32_t* __restrict__ dense_tables,
                                   const uint32_t* __restrict__ dense_perm, const uint32_t* __restrict__ counts,
                                   uint32_t G, uint32_t rank, uint64_t C, uint64_t n, PeerTab pt,
                                   uint32_t* __restrict__ perm, uint32_t* status) {
  __shared__ uint64_t s_start[kMaxPeers + 1];
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (uint32_t p = 0; p < G; ++p) {
      s_start[p] = run;
      run += counts[p];
    }
    s_start[G] = run;
  }
  __syncthreads();
  const uint64_t total = uint64_t(G) * C;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < total; q += stride) {
    const uint32_t p = static_cast<uint32_t>(q / C);
    const uint64_t r = q - uint64_t(p) * C;
    const uint64_t cnt = s_start[p + 1] - s_start[p];
    const uint64_t dst = uint64_t(rank) * C + r;
    if (r < cnt) {
      pt.keys[p][dst] = dense_keys[s_start[p] + r];
      pt.tables[p][dst] = dense_tables[s_start[p] + r];
    } else {
      pt.keys[p][dst] = 0;
      pt.tables[p][dst] = 0xffffffffu;
    }
    if (r == 0 && cnt > C) latch_status(status, HPS_GPU_E_INFEASIBLE);
  }
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t d = dense_perm[i];
    uint32_t p = 0;
    while (p + 1 < G && s_start[p + 1] <= d) ++p;
    const uint64_t r = d - s_start[p];
    perm[i] = static_cast<uint32_t>(uint64_t(p) * C + (r < C ? r : C - 1));
  }
  __threadfence_system();  // the remote stores are performed before the owner is signalled
}

__global__ void k_epoch_bump(uint64_t* e) {
  if (threadIdx.x == 0) *e += 1;
}

// Signal every peer that phase `which` of this step is done on this rank: flags[which][rank].
__global__ void k_signal(PeerTab pt, uint32_t which, uint32_t G, uint32_t rank, const uint64_t* d_epoch) {
  const uint64_t e = *d_epoch;
  __threadfence_system();
  for (uint32_t p = threadIdx.x; p < G; p += blockDim.x) {
    uint64_t* f = pt.flags[p] + uint64_t(which) * G + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
}

// Wait until every peer signalled phase `which` of this step (a single CTA spins), for at most
// kPeerWaitNs: a peer that never arrives (it failed, or was never launched) latches
// HPS_GPU_E_PEER_TIMEOUT instead of hanging the device (the step's results are then unspecified).
constexpr uint64_t kPeerWaitNs = 10ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_wait(const uint64_t* flags, uint32_t which, uint32_t G, const uint64_t* d_epoch, uint32_t* status) {
  const uint64_t e = *d_epoch;
  const uint64_t t0 = global_ns();
  for (uint32_t p = threadIdx.x; p < G; p += blockDim.x) {
    const uint64_t* f = flags + uint64_t(which) * G + p;
    uint64_t v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= e) break;
      if (global_ns() - t0 > kPeerWaitNs) {
        latch_status(status, HPS_GPU_E_PEER_TIMEOUT);
        break;
      }
      __nanosleep(200);
    }
  }
}

// Pooling fused with the rows' all-to-all: occurrence i's row is owner p's gathered row at
// [rank * C + r] (perm[i] = p*C + r), loaded straight from the owner's memory.
template <int LPR>
__global__ void __launch_bounds__(256) k_pool_rows_peer(PeerTab pt, uint32_t rank, uint64_t C,
                                                        const uint32_t* __restrict__ perm,
                                                        const uint32_t* __restrict__ offsets, uint64_t n_bags,
                                                        uint32_t dim, int mean, float* __restrict__ out) {
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
      for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t pr = perm[i], p = static_cast<uint32_t>(pr / C);
        const float* src = pt.rows[p] + (uint64_t(rank) * C + (pr - uint64_t(p) * C)) * dim;
        acc = f4_add(acc, reinterpret_cast<const float4*>(src)[v]);
      }
      if (mean && hi > lo) acc = f4_div(acc, static_cast<float>(hi - lo));
      o[v] = acc;
    }
  }
}

// Gradient scatter fused with the gradients' all-to-all: stored straight into owner p's
// receive region at [rank * C + r].
template <int LPR>
__global__ void __launch_bounds__(256) k_scatter_grads_peer(PeerTab pt, uint32_t rank, uint64_t C,
                                                            const float* __restrict__ dout,
                                                            const uint32_t* __restrict__ perm,
                                                            const uint32_t* __restrict__ offsets, uint64_t n_bags,
                                                            uint32_t dim, int mean) {
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
      for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t pr = perm[i], p = static_cast<uint32_t>(pr / C);
        float* dst = pt.grads[p] + (uint64_t(rank) * C + (pr - uint64_t(p) * C)) * dim;
        reinterpret_cast<float4*>(dst)[v] = x;
      }
    }
  }
  __threadfence_system();
}

// ---- per-destination unique rows (peer transport) -------------------------------------
// Owner side, after the gather: every received slot q of region p = q / C (requester p's
// occurrences) gets lead[q] = the smallest slot of region p holding the same (table, key).
// The hash entry is claimed by the first arriving slot (claimer + 1); later slots compare
// their (region, table, key) with the claimer's and take atomicMin. Empty slots lead
// themselves. Three launches: claim, resolve, reset (the table returns to empty).
constexpr uint32_t kNoLead = 0xffffffffu;
__device__ __forceinline__ uint64_t lead_home(uint64_t key, uint32_t table, uint32_t region, uint64_t mask) {
  return mix64(key ^ mix64((uint64_t(region) << 32) | table)) & mask;
}
__global__ void __launch_bounds__(256) k_lead_claim(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ tables,
                                                    uint64_t GC, uint64_t C, uint2* ht, uint64_t mask,
                                                    uint32_t* __restrict__ ent, uint32_t* __restrict__ lead) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < GC; q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t tb = tables[q];
    if (tb == 0xffffffffu) {  // empty slot of a region
      ent[q] = kNoLead;
      lead[q] = static_cast<uint32_t>(q);
      continue;
    }
    const uint64_t key = keys[q];
    const uint32_t region = static_cast<uint32_t>(q / C);
    uint64_t h = lead_home(key, tb, region, mask);
    while (true) {
      uint32_t cur = __ldcg(&ht[h].x);
      if (cur == 0u) {
        cur = atomicCAS(&ht[h].x, 0u, static_cast<uint32_t>(q) + 1u);
        if (cur == 0u) break;  // claimed
      }
      const uint64_t q2 = cur - 1u;
      if (q2 / C == region && tables[q2] == tb && keys[q2] == key) break;  // same (region, table, key)
      h = (h + 1) & mask;
    }
    atomicMin(&ht[h].y, static_cast<uint32_t>(q));
    ent[q] = static_cast<uint32_t>(h);
  }
}
__global__ void __launch_bounds__(256) k_lead_resolve(const uint2* __restrict__ ht, uint64_t GC,
                                                      const uint32_t* __restrict__ ent, uint32_t* __restrict__ lead) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < GC; q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = ent[q];
    if (e != kNoLead) lead[q] = __ldcg(&ht[e].y);
  }
}
// (+ counts the leaders of non-empty slots: the rows requesters fetch from this owner)
__global__ void __launch_bounds__(256) k_lead_reset(uint2* ht, uint64_t GC, const uint32_t* __restrict__ ent,
                                                    const uint32_t* __restrict__ lead, unsigned long long* served) {
  for (uint64_t base = blockIdx.x * uint64_t(blockDim.x); base < GC; base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t q = base + threadIdx.x;
    const uint32_t e = q < GC ? ent[q] : kNoLead;
    const bool leader = e != kNoLead && lead[q] == q;
    if (leader) ht[e] = make_uint2(0u, 0xffffffffu);  // one writer per entry
    const int c = __syncthreads_count(leader);
    if (threadIdx.x == 0 && c) atomicAdd(served, static_cast<unsigned long long>(c));
  }
}
__global__ void k_lead_init(uint2* ht, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    ht[i] = make_uint2(0u, 0xffffffffu);
}

// Requester side: occurrence i (slot p*C + r of this rank's regions; slot rank*C + r on owner
// p) reads its leader from owner p's lead map; a leader copies its row from owner p's gathered
// rows (over NVLink) into rows_back[p*C + r]; perm_u[i] = its leader's rows_back slot. Only
// U_p rows per owner cross NVLink instead of one per occurrence; the pooling then reads
// rows_back locally (duplicates hit L2).
template <int LPR>
__global__ void __launch_bounds__(256) k_fetch_unique_peer(PeerTab pt, uint32_t rank, uint64_t C,
                                                           const uint32_t* __restrict__ perm, uint64_t n, uint32_t dim,
                                                           float* __restrict__ rows_back, uint32_t* __restrict__ perm_u) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR, nvec = dim / 4;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t i = gid; i < n; i += ng) {
    const uint32_t pr = perm[i], p = static_cast<uint32_t>(pr / C);
    const uint64_t r = pr - uint64_t(p) * C, q = uint64_t(rank) * C + r;
    const uint64_t l = pt.lead[p][q];  // same region: l in [rank*C, rank*C + C)
    if (gl == 0) perm_u[i] = static_cast<uint32_t>(uint64_t(p) * C + (l - uint64_t(rank) * C));
    if (l != q) continue;
    const float4* src = reinterpret_cast<const float4*>(pt.rows[p] + q * dim);
    float4* dst = reinterpret_cast<float4*>(rows_back + uint64_t(pr) * dim);
    if (static_cast<const void*>(src) == static_cast<const void*>(dst)) continue;  // world of one: aliased
    for (uint32_t v = gl; v < nvec; v += LPR) dst[v] = src[v];
  }
}

// The requester's pooling over its local rows_back (after the unique-row fetch): bags in
// occurrence order, sequential float4 sums, then the mean's divide — the same arithmetic as
// exchange.cu's k_pool_rows (bit-identical), in this module so the peer step never loads a
// kernel lazily while a peer's wait kernel spins.
template <int LPR>
__global__ void __launch_bounds__(256) k_pool_local(const float* __restrict__ rows, const uint32_t* __restrict__ perm,
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
      for (uint32_t i = lo; i < hi; ++i) acc = f4_add(acc, reinterpret_cast<const float4*>(rows + uint64_t(perm[i]) * dim)[v]);
      if (mean && hi > lo) acc = f4_div(acc, static_cast<float>(hi - lo));
      o[v] = acc;
    }
  }
}

int lpr_of(uint32_t dim) {
  const uint32_t nvec = dim / 4;
  return nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
}

#define HPSG_LPR_DISPATCH(KERNEL, LPR, GRID, ST, ...)                    \
  do {                                                                  \
    switch (LPR) {                                                      \
      case 32: KERNEL<32><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;    \
      case 16: KERNEL<16><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;    \
      case 8: KERNEL<8><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;      \
      case 4: KERNEL<4><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;      \
      case 2: KERNEL<2><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;      \
      default: KERNEL<1><<<GRID, 256, 0, ST>>>(__VA_ARGS__); break;     \
    }                                                                   \
  } while (0)

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HPS_GPU_OK;
  set_last_error(std::string(what) + ": " + ncclGetErrorString(r));
  return HPS_GPU_E_NCCL;
}
#define HPSG_NCCL(call)                                  \
  do {                                                   \
    ncclResult_t r_ = (call);                            \
    if (r_ != ncclSuccess) return nccl_status(r_, #call); \
  } while (0)

// Which buffer pair an all-to-all moves (the loopback transport reads its peers' copies).
enum Xfer { kXKeys = 0, kXTables = 1, kXRows = 2, kXGrads = 3 };
const void* send_of(const hps_gpu_dist_s* d, int x) {
  return x == kXKeys ? static_cast<const void*>(d->send_keys) : x == kXTables ? static_cast<const void*>(d->send_tables)
         : x == kXRows ? static_cast<const void*>(d->rows_own) : static_cast<const void*>(d->grads_send);
}

int loop_a2a(hps_gpu_dist d, int x, void* recv, size_t bytes) {
  cudaStream_t st = d->ctx->stream;
  HPSG_CUDA(cudaEventRecord(d->loop_ev, st));  // this rank's send buffer is written
  d->loop->bar.arrive_and_wait();
  for (uint32_t p = 0; p < d->G; ++p) {
    const hps_gpu_dist_s* peer = d->loop->members[p];
    HPSG_CUDA(cudaStreamWaitEvent(st, peer->loop_ev, 0));
    HPSG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + p * bytes,
                              static_cast<const char*>(send_of(peer, x)) + size_t(d->rank) * bytes, bytes,
                              cudaMemcpyDeviceToDevice, st));
  }
  HPSG_CUDA(cudaStreamSynchronize(st));  // peers may reuse their send buffers after the barrier
  d->loop->bar.arrive_and_wait();
  return HPS_GPU_OK;
}

// All-to-all of G regions of `elems` elements each (region p of send -> rank p's region
// `rank` of recv). World of one: the caller aliases recv to send.
int a2a(hps_gpu_dist d, int x, const void* send, void* recv, size_t elem_bytes, uint64_t elems) {
  if (d->G == 1) return HPS_GPU_OK;
  if (d->loop) return loop_a2a(d, x, recv, elem_bytes * elems);
  auto comm = static_cast<ncclComm_t>(d->ctx->nccl);
  const size_t bytes = elem_bytes * elems;
  HPSG_NCCL(ncclGroupStart());
  for (uint32_t p = 0; p < d->G; ++p) {
    HPSG_NCCL(ncclSend(static_cast<const char*>(send) + p * bytes, bytes, ncclUint8, static_cast<int>(p), comm,
                       d->ctx->stream));
    HPSG_NCCL(ncclRecv(static_cast<char*>(recv) + p * bytes, bytes, ncclUint8, static_cast<int>(p), comm,
                       d->ctx->stream));
  }
  HPSG_NCCL(ncclGroupEnd());
  return HPS_GPU_OK;
}

template <class T>
int dalloc_n(T** p, uint64_t n) {
  if (cudaMalloc(reinterpret_cast<void**>(p), std::max<uint64_t>(n, 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}

}  // namespace

void hpsg::comm_destroy(hps_gpu_ctx_s* ctx) {
  if (ctx && ctx->nccl) {
    ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
    ctx->nccl = nullptr;
  }
}

namespace {
// The forward with the peer-memory transport (after the bucketize):
//   regions stored into the owners -> signal/wait -> owner gather -> signal/wait -> pooling
//   that loads the owners' rows directly.
int dist_forward_peer(hps_gpu_dist d, const uint32_t* offsets, uint64_t n_bags, uint64_t n, int combiner, float* out,
                      uint32_t flags) {
  cudaStream_t st = d->ctx->stream;
  const uint64_t GC = uint64_t(d->G) * d->C;
  k_epoch_bump<<<1, 32, 0, st>>>(d->d_epoch);
  k_fix_regions_peer<<<grid_for(std::max<uint64_t>(GC, n), 256, kNumSMs * 16), 256, 0, st>>>(
      d->dense_keys, d->dense_tables, d->dense_perm, d->counts, d->G, d->rank, d->C, n, *d->peer, d->perm,
      d->ctx->d_status);
  k_signal<<<1, 64, 0, st>>>(*d->peer, 0, d->G, d->rank, d->d_epoch);
  k_wait<<<1, 64, 0, st>>>(d->flags, 0, d->G, d->d_epoch, d->ctx->d_status);
  HPSG_CHECK_LAUNCH("dist regions (peer)");
  const uint32_t gflags = (flags & HPS_LOOKUP_TRAIN) | (flags & HPS_LOOKUP_INSERT);
  if (int s = hps_gpu_gather_rows(d->shard, d->recv_keys, d->recv_tables, GC, d->rows_own, gflags)) return s;
  if (d->G > 1) {  // the leader map of every requester region (per-destination unique rows;
                   // a world of one moves nothing over NVLink: it pools from its own rows)
    const int g = grid_for(GC, 256, kNumSMs * 8);
    k_lead_claim<<<g, 256, 0, st>>>(d->recv_keys, d->recv_tables, GC, d->C, d->lead_ht, d->lead_mask, d->lead_ent, d->lead);
    k_lead_resolve<<<g, 256, 0, st>>>(d->lead_ht, GC, d->lead_ent, d->lead);
    k_lead_reset<<<g, 256, 0, st>>>(d->lead_ht, GC, d->lead_ent, d->lead, d->d_served);
    HPSG_CHECK_LAUNCH("dist leader map (peer)");
  }
  k_signal<<<1, 64, 0, st>>>(*d->peer, 1, d->G, d->rank, d->d_epoch);
  k_wait<<<1, 64, 0, st>>>(d->flags, 1, d->G, d->d_epoch, d->ctx->d_status);
  const int lpr = lpr_of(d->dim);
  if (d->G > 1) {
    HPSG_LPR_DISPATCH(k_fetch_unique_peer, lpr, grid_for(n * lpr, 256, kNumSMs * 32), st, *d->peer, d->rank, d->C,
                      d->perm, n, d->dim, d->rows_back, d->perm_u);
    HPSG_CHECK_LAUNCH("dist unique-row fetch (peer)");
  }
  HPSG_LPR_DISPATCH(k_pool_local, lpr, grid_for(n_bags * lpr, 256, kNumSMs * 32), st, d->rows_back,
                    d->G > 1 ? d->perm_u : d->perm, offsets, n_bags, d->dim, combiner == HPS_COMBINER_MEAN, out);
  HPSG_CHECK_LAUNCH("dist pool (peer)");
  d->last_offsets = offsets;
  d->last_bags = n_bags;
  d->last_combiner = combiner;
  d->have_fwd = true;
  d->train = (flags & HPS_LOOKUP_TRAIN) != 0;
  return HPS_GPU_OK;
}

void fill_self(hps_gpu_dist d, PeerTab& t, uint32_t p) {
  t.keys[p] = d->recv_keys;
  t.tables[p] = d->recv_tables;
  t.rows[p] = d->rows_own;
  t.grads[p] = d->grads_recv;
  t.flags[p] = d->flags;
  t.lead[p] = d->lead;
}
}  // namespace

extern "C" {

int hps_gpu_dist_set_transport(hps_gpu_dist d, int transport) {
  if (!d || (transport != HPS_DIST_NCCL && transport != HPS_DIST_PEER)) return HPS_GPU_E_INVALID_ARGUMENT;
  if (transport == HPS_DIST_NCCL) {
    d->transport = transport;
    return HPS_GPU_OK;
  }
  if (d->G > kMaxPeers) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaSetDevice(d->ctx->device));
  {  // load every kernel of the peer path now: a lazy module load inside a step could wait for
     // the device while a peer's wait kernel spins on this rank's signal
    cudaFuncAttributes fa;
    for (const void* f : {reinterpret_cast<const void*>(k_fix_regions_peer), reinterpret_cast<const void*>(k_epoch_bump),
                          reinterpret_cast<const void*>(k_signal), reinterpret_cast<const void*>(k_wait),
                          reinterpret_cast<const void*>(k_pool_rows_peer<32>), reinterpret_cast<const void*>(k_pool_rows_peer<16>),
                          reinterpret_cast<const void*>(k_pool_rows_peer<8>), reinterpret_cast<const void*>(k_pool_rows_peer<4>),
                          reinterpret_cast<const void*>(k_pool_rows_peer<2>), reinterpret_cast<const void*>(k_pool_rows_peer<1>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<32>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<16>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<8>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<4>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<2>),
                          reinterpret_cast<const void*>(k_scatter_grads_peer<1>),
                          reinterpret_cast<const void*>(k_lead_claim), reinterpret_cast<const void*>(k_lead_resolve),
                          reinterpret_cast<const void*>(k_lead_reset),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<32>),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<16>),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<8>),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<4>),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<2>),
                          reinterpret_cast<const void*>(k_fetch_unique_peer<1>),
                          reinterpret_cast<const void*>(k_pool_local<32>), reinterpret_cast<const void*>(k_pool_local<16>),
                          reinterpret_cast<const void*>(k_pool_local<8>), reinterpret_cast<const void*>(k_pool_local<4>),
                          reinterpret_cast<const void*>(k_pool_local<2>), reinterpret_cast<const void*>(k_pool_local<1>)})
      HPSG_CUDA(cudaFuncGetAttributes(&fa, f));
  }
  if (!d->peer) d->peer = new PeerTab{};
  PeerTab& t = *d->peer;
  if (d->G == 1) {
    fill_self(d, t, 0);
  } else if (d->loop) {  // loopback ranks: the peers' buffers are this device's memory
    for (uint32_t p = 0; p < d->G; ++p) fill_self(d->loop->members[p], t, p);
  } else {  // NCCL ranks: CUDA-IPC handles of every owner-side buffer, all-gathered over NCCL
    constexpr int kB = 6;
    cudaIpcMemHandle_t mine[kB];
    void* bufs[kB] = {d->recv_keys, d->recv_tables, d->rows_own, d->grads_recv, d->flags, d->lead};
    for (int k = 0; k < kB; ++k) HPSG_CUDA(cudaIpcGetMemHandle(&mine[k], bufs[k]));
    cudaIpcMemHandle_t* d_all = nullptr;
    HPSG_CUDA(cudaMalloc(&d_all, sizeof(mine) * d->G));
    HPSG_CUDA(cudaMemcpy(d_all + kB * d->rank, mine, sizeof(mine), cudaMemcpyHostToDevice));
    HPSG_NCCL(ncclAllGather(d_all + kB * d->rank, d_all, sizeof(mine), ncclUint8, static_cast<ncclComm_t>(d->ctx->nccl),
                            d->ctx->stream));
    HPSG_CUDA(cudaStreamSynchronize(d->ctx->stream));
    std::vector<cudaIpcMemHandle_t> all(kB * d->G);
    HPSG_CUDA(cudaMemcpy(all.data(), d_all, sizeof(mine) * d->G, cudaMemcpyDeviceToHost));
    cudaFree(d_all);
    for (uint32_t p = 0; p < d->G; ++p) {
      if (p == d->rank) {
        fill_self(d, t, p);
        continue;
      }
      void* ptr[kB];
      for (int k = 0; k < kB; ++k) {
        HPSG_CUDA(cudaIpcOpenMemHandle(&ptr[k], all[kB * p + k], cudaIpcMemLazyEnablePeerAccess));
        d->ipc_opened.push_back(ptr[k]);
      }
      t.keys[p] = static_cast<uint64_t*>(ptr[0]);
      t.tables[p] = static_cast<uint32_t*>(ptr[1]);
      t.rows[p] = static_cast<float*>(ptr[2]);
      t.grads[p] = static_cast<float*>(ptr[3]);
      t.flags[p] = static_cast<uint64_t*>(ptr[4]);
      t.lead[p] = static_cast<uint32_t*>(ptr[5]);
    }
  }
  // ... and launch each of them once with no work: the module code is then resident whatever
  // the runtime's lazy-loading policy (loopback ranks share one device, where a load that
  // waits for the device while a peer's k_wait spins would deadlock the step)
  {
    cudaStream_t st = d->ctx->stream;
    uint64_t* scratch = nullptr;
    HPSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(uint64_t), st));
    HPSG_CUDA(cudaMemsetAsync(scratch, 0, sizeof(uint64_t), st));
    k_epoch_bump<<<1, 32, 0, st>>>(scratch);
    k_fix_regions_peer<<<1, 32, 0, st>>>(d->dense_keys, d->dense_tables, d->dense_perm, d->counts, 0, d->rank, d->C, 0,
                                         t, d->perm, d->ctx->d_status);
    k_signal<<<1, 32, 0, st>>>(t, 0, 0, d->rank, scratch);
    k_wait<<<1, 32, 0, st>>>(d->flags, 0, 0, scratch, d->ctx->d_status);
    k_lead_claim<<<1, 32, 0, st>>>(d->recv_keys, d->recv_tables, 0, d->C, d->lead_ht, d->lead_mask, d->lead_ent, d->lead);
    k_lead_resolve<<<1, 32, 0, st>>>(d->lead_ht, 0, d->lead_ent, d->lead);
    k_lead_reset<<<1, 32, 0, st>>>(d->lead_ht, 0, d->lead_ent, d->lead, d->d_served);
#define HPSG_WARM(L)                                                                                           \
  k_pool_rows_peer<L><<<1, 32, 0, st>>>(t, d->rank, d->C, d->perm, nullptr, 0, d->dim, 0, d->rows_back);     \
  k_scatter_grads_peer<L><<<1, 32, 0, st>>>(t, d->rank, d->C, d->grads_send, d->perm, nullptr, 0, d->dim, 0); \
  k_fetch_unique_peer<L><<<1, 32, 0, st>>>(t, d->rank, d->C, d->perm, 0, d->dim, d->rows_back, d->perm_u);     \
  k_pool_local<L><<<1, 32, 0, st>>>(d->rows_back, d->perm, nullptr, 0, d->dim, 0, d->rows_back);
    HPSG_WARM(32) HPSG_WARM(16) HPSG_WARM(8) HPSG_WARM(4) HPSG_WARM(2) HPSG_WARM(1)
#undef HPSG_WARM
    HPSG_CHECK_LAUNCH("peer kernels warm-up");
    HPSG_CUDA(cudaFreeAsync(scratch, st));
    HPSG_CUDA(cudaStreamSynchronize(st));
  }
  d->transport = HPS_DIST_PEER;
  return HPS_GPU_OK;
}

int hps_gpu_nccl_unique_id(void* id_out) {
  if (!id_out) return HPS_GPU_E_INVALID_ARGUMENT;
  ncclUniqueId id;
  HPSG_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == HPS_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return HPS_GPU_OK;
}

int hps_gpu_ctx_comm_init(hps_gpu_ctx ctx, const void* id, int rank, int world) {
  if (!ctx || !id || world < 1 || rank < 0 || rank >= world || world > 256) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaSetDevice(ctx->device));
  comm_destroy(ctx);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  HPSG_NCCL(ncclCommInitRank(&comm, world, uid, rank));
  ctx->nccl = comm;
  ctx->rank = rank;
  ctx->world = world;
  return HPS_GPU_OK;
}

}  // extern "C"

namespace {
int dist_create(hps_gpu_ctx ctx, hps_gpu_table shard, const hps_dist_config* cfg, uint32_t G, uint32_t rank,
                hps_gpu_dist* out) {
  if (!ctx || !shard || !cfg || !out || cfg->n_slots == 0 || !cfg->slot_table_host || cfg->max_keys == 0 ||
      cfg->max_keys >= (1ull << 31) || cfg->max_bags == 0 || cfg->dim == 0 || cfg->dim % 4)
    return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  HPSG_CUDA(cudaSetDevice(ctx->device));
  auto d = new hps_gpu_dist_s;
  d->ctx = ctx;
  d->shard = shard;
  d->n_slots = cfg->n_slots;
  d->dim = cfg->dim;
  d->G = G;
  d->rank = rank;
  d->max_keys = cfg->max_keys;
  d->max_bags = cfg->max_bags;
  const double f = cfg->capacity_factor > 0.f ? cfg->capacity_factor : 1.25;
  d->C = d->G == 1 ? d->max_keys
                   : std::min<uint64_t>(d->max_keys, uint64_t(std::ceil(f * double(d->max_keys) / d->G)) + 1024);
  const uint64_t GC = uint64_t(d->G) * d->C, D = d->dim, N = d->max_keys;
  int st = HPS_GPU_OK;
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  if (int s = hps_gpu_xplan_create(ctx, N, d->G, &d->plan)) A(s);
  A(dalloc_n(&d->d_slot_table, d->n_slots));
  A(dalloc_n(&d->dense_keys, N));
  A(dalloc_n(&d->dense_tables, N));
  A(dalloc_n(&d->dense_perm, N));
  A(dalloc_n(&d->counts, d->G));
  A(dalloc_n(&d->occ_bag, N));
  A(dalloc_n(&d->perm, N));
  A(dalloc_n(&d->send_keys, GC));
  A(dalloc_n(&d->send_tables, GC));
  A(dalloc_n(&d->rows_own, GC * D));
  A(dalloc_n(&d->grads_send, GC * D));
  if (d->G > 1) {
    A(dalloc_n(&d->recv_keys, GC));
    A(dalloc_n(&d->recv_tables, GC));
    A(dalloc_n(&d->rows_back, GC * D));
    A(dalloc_n(&d->grads_recv, GC * D));
  } else {  // a world of one: every region is its own peer's — alias, no copy
    d->recv_keys = d->send_keys;
    d->recv_tables = d->send_tables;
    d->rows_back = d->rows_own;
    d->grads_recv = d->grads_send;
  }
  if (!st && cudaMemcpy(d->d_slot_table, cfg->slot_table_host, d->n_slots * 4, cudaMemcpyHostToDevice) != cudaSuccess)
    st = HPS_GPU_E_CUDA;
  if (!st && cudaEventCreateWithFlags(&d->loop_ev, cudaEventDisableTiming) != cudaSuccess) st = HPS_GPU_E_CUDA;
  A(dalloc_n(&d->lead, GC));
  A(dalloc_n(&d->lead_ent, GC));
  A(dalloc_n(&d->perm_u, N));
  A(dalloc_n(&d->d_served, 1));
  if (!st && cudaMemset(d->d_served, 0, sizeof(unsigned long long)) != cudaSuccess) st = HPS_GPU_E_CUDA;
  {
    uint64_t hs = 1;
    while (hs < 2 * GC) hs <<= 1;
    d->lead_mask = hs - 1;
    A(dalloc_n(&d->lead_ht, hs));
    if (!st) {
      k_lead_init<<<grid_for(hs, 256, kNumSMs * 8), 256, 0, ctx->stream>>>(d->lead_ht, hs);
      if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = HPS_GPU_E_CUDA;
    }
  }
  A(dalloc_n(&d->flags, 3 * uint64_t(d->G)));
  A(dalloc_n(&d->d_epoch, 1));
  if (!st && (cudaMemset(d->flags, 0, 3 * d->G * sizeof(uint64_t)) != cudaSuccess ||
              cudaMemset(d->d_epoch, 0, sizeof(uint64_t)) != cudaSuccess))
    st = HPS_GPU_E_CUDA;
  if (st) {
    hps_gpu_dist_destroy(d);
    return st;
  }
  *out = d;
  return HPS_GPU_OK;
}
}  // namespace

extern "C" {

int hps_gpu_dist_create(hps_gpu_ctx ctx, hps_gpu_table shard, const hps_dist_config* cfg, hps_gpu_dist* out) {
  if (!ctx) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!ctx->nccl && ctx->world != 1) return HPS_GPU_E_INVALID_ARGUMENT;
  return dist_create(ctx, shard, cfg, static_cast<uint32_t>(ctx->nccl ? ctx->world : 1),
                     static_cast<uint32_t>(ctx->nccl ? ctx->rank : 0), out);
}

int hps_gpu_dist_create_loopback(const hps_gpu_ctx* ctxs, const hps_gpu_table* shards, const hps_dist_config* cfg,
                                 uint32_t n, hps_gpu_dist* outs) {
  if (!ctxs || !shards || !outs || n == 0 || n > 256) return HPS_GPU_E_INVALID_ARGUMENT;
  auto group = std::make_shared<LoopGroup>(n);
  for (uint32_t r = 0; r < n; ++r) {
    if (int s = dist_create(ctxs[r], shards[r], cfg, n, r, &outs[r])) {
      for (uint32_t q = 0; q < r; ++q) hps_gpu_dist_destroy(outs[q]);
      return s;
    }
    outs[r]->loop = group;
    group->members[r] = outs[r];
  }
  return HPS_GPU_OK;
}

int hps_gpu_dist_destroy(hps_gpu_dist d) {
  if (!d) return HPS_GPU_OK;
  if (d->loop_ev) cudaEventDestroy(d->loop_ev);
  for (void* p : d->ipc_opened) cudaIpcCloseMemHandle(p);
  delete d->peer;
  if (d->flags) cudaFree(d->flags);
  if (d->d_epoch) cudaFree(d->d_epoch);
  if (d->plan) hps_gpu_xplan_destroy(d->plan);
  void* own[] = {d->d_slot_table, d->dense_keys, d->dense_tables, d->dense_perm, d->counts,   d->occ_bag,
                 d->perm,         d->send_keys,  d->send_tables, d->rows_own,   d->grads_send, d->lead,
                 d->lead_ent,     d->lead_ht,    d->perm_u,      d->d_served};
  for (void* p : own)
    if (p) cudaFree(p);
  if (d->G > 1) {
    void* peer[] = {d->recv_keys, d->recv_tables, d->rows_back, d->grads_recv};
    for (void* p : peer)
      if (p) cudaFree(p);
  }
  delete d;
  return HPS_GPU_OK;
}

int hps_gpu_dist_capacity(hps_gpu_dist d, uint64_t* per_peer_out) {
  if (!d || !per_peer_out) return HPS_GPU_E_INVALID_ARGUMENT;
  *per_peer_out = d->C;
  return HPS_GPU_OK;
}

int hps_gpu_dist_unique_rows(hps_gpu_dist d, uint64_t* served_host) {
  if (!d || !served_host) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaStreamSynchronize(d->ctx->stream));
  unsigned long long v = 0;
  HPSG_CUDA(cudaMemcpy(&v, d->d_served, sizeof(v), cudaMemcpyDeviceToHost));
  *served_host = v;
  return HPS_GPU_OK;
}

int hps_gpu_dist_forward(hps_gpu_dist d, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         uint64_t n_keys, int combiner, float* out, uint32_t flags) {
  if (!d || !out || (combiner != HPS_COMBINER_SUM && combiner != HPS_COMBINER_MEAN)) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint64_t n_bags = uint64_t(n_samples) * d->n_slots;
  const bool multi = offsets != nullptr;
  const uint64_t n = multi ? n_keys : n_bags;
  if (n_bags > d->max_bags || n > d->max_keys || (n && !keys)) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaStream_t st = d->ctx->stream;
  const uint64_t GC = uint64_t(d->G) * d->C;
  if (multi && n_bags)
    if (int s = hps_gpu_occurrence_bags(d->ctx, offsets, n_bags, d->occ_bag)) return s;
  if (int s = hps_gpu_xplan_bucketize(d->plan, keys, n, multi ? d->occ_bag : nullptr, d->n_slots, d->d_slot_table,
                                      d->dense_keys, d->dense_tables, d->dense_perm, d->counts))
    return s;
  if (d->transport == HPS_DIST_PEER) return dist_forward_peer(d, offsets, n_bags, n, combiner, out, flags);
  k_fix_regions<<<grid_for(std::max<uint64_t>(GC, n), 256, kNumSMs * 16), 256, 0, st>>>(
      d->dense_keys, d->dense_tables, d->dense_perm, d->counts, d->G, d->C, n, d->send_keys, d->send_tables, d->perm,
      d->ctx->d_status);
  HPSG_CHECK_LAUNCH("k_fix_regions");
  if (int s = a2a(d, kXKeys, d->send_keys, d->recv_keys, 8, d->C)) return s;
  if (int s = a2a(d, kXTables, d->send_tables, d->recv_tables, 4, d->C)) return s;
  const uint32_t gflags = (flags & HPS_LOOKUP_TRAIN) | (flags & HPS_LOOKUP_INSERT);
  if (int s = hps_gpu_gather_rows(d->shard, d->recv_keys, d->recv_tables, GC, d->rows_own, gflags)) return s;
  if (int s = a2a(d, kXRows, d->rows_own, d->rows_back, 4 * size_t(d->dim), d->C)) return s;
  if (int s = hps_gpu_pool_rows(d->ctx, d->rows_back, d->perm, offsets, n_bags, d->dim, combiner, out)) return s;
  d->last_offsets = offsets;
  d->last_bags = n_bags;
  d->last_combiner = combiner;
  d->have_fwd = true;
  d->train = (flags & HPS_LOOKUP_TRAIN) != 0;
  return HPS_GPU_OK;
}

int hps_gpu_dist_backward(hps_gpu_dist d, const float* d_out, const hps_opt_params* opt) {
  if (!d || !d_out || !opt) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!d->have_fwd || !d->train) {
    set_last_error("dist_backward: no preceding training dist_forward");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (d->transport == HPS_DIST_PEER) {  // gradients stored straight into the owners' regions
    cudaStream_t st = d->ctx->stream;
    const int lpr = lpr_of(d->dim);
    HPSG_LPR_DISPATCH(k_scatter_grads_peer, lpr, grid_for(d->last_bags * lpr, 256, kNumSMs * 32), st, *d->peer,
                      d->rank, d->C, d_out, d->perm, d->last_offsets, d->last_bags, d->dim,
                      d->last_combiner == HPS_COMBINER_MEAN);
    k_signal<<<1, 64, 0, st>>>(*d->peer, 2, d->G, d->rank, d->d_epoch);
    k_wait<<<1, 64, 0, st>>>(d->flags, 2, d->G, d->d_epoch, d->ctx->d_status);
    HPSG_CHECK_LAUNCH("dist backward (peer)");
    if (int s = hps_gpu_backward_update(d->shard, d->grads_recv, opt)) return s;
    d->have_fwd = false;
    return HPS_GPU_OK;
  }
  if (int s = hps_gpu_scatter_grads(d->ctx, d_out, d->perm, d->last_offsets, d->last_bags, d->dim, d->last_combiner,
                                    d->grads_send))
    return s;
  if (int s = a2a(d, kXGrads, d->grads_send, d->grads_recv, 4 * size_t(d->dim), d->C)) return s;
  if (int s = hps_gpu_backward_update(d->shard, d->grads_recv, opt)) return s;
  d->have_fwd = false;
  return HPS_GPU_OK;
}

}  // extern "C"
