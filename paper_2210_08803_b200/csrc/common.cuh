// common.cuh — shared device helpers for the sm_100a sparse-embedding kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <type_traits>

#include <hps/hash.hpp>
#include "hps_gpu.h"

namespace hpsg {

constexpr uint32_t kRowEmpty = 0xffffffffu;    // index slot not in use
constexpr uint32_t kRowPending = 0xfffffffeu;  // slot claimed by an in-flight insert
constexpr uint32_t kAuxNone = 0xffffffffu;     // slot.aux outside of an insert call
constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// One open-addressing index slot: 16 B, one aligned vector access.
struct __align__(16) Slot {
  uint64_t key;
  uint32_t row;  // local row id within its table, or kRowEmpty / kRowPending
  uint32_t aux;  // insert-time scratch: min occurrence index of this key in the call
};

// Per-table placement inside a table group (device-resident array).
struct TableDev {
  uint64_t slot_base;  // first slot of this table's index
  uint64_t slot_mask;  // index capacity - 1 (power of two)
  uint64_t row_base;   // first global row of this table
  uint64_t row_cap;    // max rows
};

// Latched device status word: first error wins.
__device__ __forceinline__ void latch_status(uint32_t* st, uint32_t code) {
  if (st) atomicCAS(st, 0u, code);
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// DESIGN.md §4.1 row initialiser (bit-identical to oracle/oracle.cpp init_value).
__host__ __device__ __forceinline__ float init_value(uint64_t seed, uint64_t key, uint32_t j) {
  uint64_t u = mix64(hps::key_hash(key) + seed * 0xd1b54a32d192ed03ull +
                     (static_cast<uint64_t>(j) + 1) * 0x9e3779b97f4a7c15ull);
  float v = static_cast<float>(u >> 40);
#if defined(__CUDA_ARCH__)
  return __fmul_rn(__fsub_rn(__fmul_rn(v, 5.9604644775390625e-08f), 0.5f), 0.03125f);
#else
  return (v * 5.9604644775390625e-08f - 0.5f) * 0.03125f;
#endif
}

__device__ __forceinline__ bool non_finite_bits(uint32_t b) { return (b & 0x7f800000u) == 0x7f800000u; }

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 128-bit compare-and-swap on a Slot (sm_90+: ATOMG.E.CAS.128). Returns the old slot.
__device__ __forceinline__ Slot slot_cas(Slot* p, const Slot& expect, const Slot& desired) {
  unsigned __int128 e, d;
  e = (static_cast<unsigned __int128>((static_cast<uint64_t>(expect.aux) << 32) | expect.row) << 64) | expect.key;
  d = (static_cast<unsigned __int128>((static_cast<uint64_t>(desired.aux) << 32) | desired.row) << 64) | desired.key;
  unsigned __int128 o = atomicCAS(reinterpret_cast<unsigned __int128*>(p), e, d);
  Slot r;
  r.key = static_cast<uint64_t>(o);
  uint64_t hi = static_cast<uint64_t>(o >> 64);
  r.row = static_cast<uint32_t>(hi);
  r.aux = static_cast<uint32_t>(hi >> 32);
  return r;
}

__device__ __forceinline__ Slot load_slot(const Slot* p) {
  ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
  Slot s;
  s.key = v.x;
  s.row = static_cast<uint32_t>(v.y);
  s.aux = static_cast<uint32_t>(v.y >> 32);
  return s;
}

// Streaming (read-once) 128-bit load: bypass L1 allocation.
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Four binary16 values [4v, 4v+4) of a row, widened to fp32 (exact).
__device__ __forceinline__ float4 ldg_half4(const uint16_t* p, uint32_t v) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p) + v);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
// fp32 -> binary16 bits, round to nearest even (cvt.rn.f16.f32; kernels_scalar.cpp:25-57).
__device__ __forceinline__ uint16_t f32_to_half_bits(float x) { return __half_as_ushort(__float2half_rn(x)); }

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4_div(float4 a, float d) {
  return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d), __fdiv_rn(a.w, d));
}

// ---- Blackwell bulk-copy (TMA 1-D) and mbarrier helpers --------------------------------
// cp.async.bulk moves whole rows global<->shared on the copy engine: no registers are held
// while the bytes are in flight, so a warp can keep tens of KB outstanding.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "HPSG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra HPSG_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Same, with an L2 eviction-priority hint (createpolicy): rows read once per step stream
// through L2 as evict_first so they do not displace the step's small hot working sets.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gdst, const void* smem_src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Generic-proxy smem writes -> visible to the async proxy (before a bulk store reads them).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Programmatic dependent launch. A kernel launched with the PDL attribute may be scheduled
// while its stream predecessor drains; griddepcontrol.wait blocks until the predecessor grid
// has completed and its writes are visible, so every PDL-launched kernel calls pdl_wait()
// before its first global access. Both instructions are no-ops under a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Kernel launch with optional PDL (cudaLaunchKernelEx; captured into graphs as
// programmatic edges).
// coop: cooperative launch (all CTAs co-resident, so a grid-wide barrier is safe even
// with other streams' kernels on the device).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kx(bool pdl, bool coop, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args... args) {
  return launch_kx(pdl, false, kernel, grid, block, smem, st, args...);
}

// Kernels that run side by side (pooling beside the dedup, short beside long reduce) need
// the same L1/shared split: an SM carved out for one cannot take the other's CTAs until
// it drains. Every step kernel asks for the maximum shared carveout (once per kernel).
template <typename... KArgs>
inline cudaError_t prefer_max_smem(void (*kernel)(KArgs...)) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

// One-shot grid barrier over a zeroed counter (cooperative launches only).
__device__ __forceinline__ void grid_barrier_once(uint32_t* counter) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      if (v < gridDim.x) __nanosleep(64);
    } while (v < gridDim.x);
  }
  __syncthreads();
}

// One-time per-DEVICE setup (function attributes are per device): `done` is a bitmask of
// devices already set up (a static per call site); fn() returns a cudaError_t. Thread-safe.
template <class F>
cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& fn) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  static std::mutex m;
  std::lock_guard<std::mutex> g(m);
  if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  const cudaError_t e = fn();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

inline int grid_for(uint64_t n, int block, int max_blocks = kNumSMs * 16) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > static_cast<uint64_t>(max_blocks)) g = max_blocks;
  return static_cast<int>(g);
}

// ---- in-graph kernel timeline (hps_gpu_debug_trace) ----------------
// When a trace buffer is attached, the step kernels stamp %globaltimer: the first CTA's
// start (atomicMin) and every warp's exit (atomicMax), per kernel id. The pointer is a
// per-translation-unit symbol (null = off: one predicated load per CTA).
struct TraceRec {
  unsigned long long start, end;
};
constexpr int kTraceSlots = 32;
enum TraceId : int {
  kTrProbe = 0, kTrPool = 1, kTrAlloc = 2, kTrPlace = 3, kTrHist = 4, kTrPass0 = 5, kTrLongReg = 9,
  kTrReduce = 10, kTrLong = 11, kTrReset = 12, kTrCount = 13, kTrCountLocal = 14, kTrCountGlobal = 15,
  kTrCountCas = 16, kTrCountProbe = 17, kTrScale = 18, kTrInsClaim = 21, kTrInsCommit = 22, kTrInsFinish = 23
};
static __device__ TraceRec* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Records are per (id, SM) so the stamps of thousands of warps never pile onto one L2
// address (that serialisation would distort the kernels being traced); the host reduces.
constexpr int kTraceSMs = 160;
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void trace_begin(int id) {
  if (id >= 0 && threadIdx.x == 0) {
    TraceRec* t = g_trace;
    if (t) atomicMin(&t[id * kTraceSMs + (sm_id() % kTraceSMs)].start, gtimer());
  }
}
__device__ __forceinline__ void trace_end(int id) {
  if (id >= 0 && (threadIdx.x & 31) == 0) {
    TraceRec* t = g_trace;
    if (t) atomicMax(&t[id * kTraceSMs + (sm_id() % kTraceSMs)].end, gtimer());
  }
}
// trace_end once `dep` has landed (the timer is read under a branch on it)
__device__ __forceinline__ void trace_end_after(int id, uint32_t dep) {
  trace_end(dep == 0x9e3779b9u ? -1 : id);
}
inline cudaError_t trace_attach_tu(TraceRec* p) { return cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }
// Op::kTrace when the scan op declares one, else -1 (untraced).
template <class Op, class = void>
struct TraceOf {
  static constexpr int id = -1;
};
template <class Op>
struct TraceOf<Op, std::void_t<decltype(Op::kTrace)>> {
  static constexpr int id = Op::kTrace;
};

// ---- rows of a dim that is not a multiple of 4 ------------------------------------
// Tables and caches store rows at a padded stride (round_up(dim, 4): every kernel moves
// 128-bit vectors); the caller's buffers keep `dim`. These copy [rows x cols] fp32 between
// the two strides (cudaMemcpy2DAsync: capturable, no kernel); widening zero-fills the
// padding so no NaN/Inf check ever sees garbage.
inline uint32_t padded_dim(uint32_t dim) { return (dim + 3u) & ~3u; }
inline cudaError_t rows_narrow(void* dst, uint32_t dim_io, const void* src, uint32_t dim, uint64_t rows,
                               cudaStream_t st, size_t elem = 4) {
  if (rows == 0) return cudaSuccess;
  return cudaMemcpy2DAsync(dst, size_t(dim_io) * elem, src, size_t(dim) * elem, size_t(dim_io) * elem, rows,
                           cudaMemcpyDeviceToDevice, st);
}
inline cudaError_t rows_widen(float* dst, uint32_t dim, const float* src, uint32_t dim_io, uint64_t rows,
                              cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if (cudaError_t e = cudaMemset2DAsync(dst + dim_io, size_t(dim) * 4, 0, size_t(dim - dim_io) * 4, rows, st)) return e;
  return cudaMemcpy2DAsync(dst, size_t(dim) * 4, src, size_t(dim_io) * 4, size_t(dim_io) * 4, rows,
                           cudaMemcpyDeviceToDevice, st);
}

// ---- host-side error plumbing -------------------------------------------------
void set_last_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

}  // namespace hpsg

#define HPSG_CUDA(call)                                               \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) return ::hpsg::cuda_status(e_, #call);     \
  } while (0)

#define HPSG_CHECK_LAUNCH(what) HPSG_CUDA(cudaGetLastError())

// Context layout shared by all translation units.
struct hps_gpu_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t* d_status = nullptr;  // latched device status word
  uint32_t* h_status = nullptr;  // pinned mirror for sync
  bool pdl = true;               // programmatic dependent launch in the step chains (HPS_GPU_NO_PDL=1 disables)
  int num_sms = hpsg::kNumSMs;   // multiProcessorCount of the device (the persistent dedup's grid cap)
  void* nccl = nullptr;          // ncclComm_t of the sharded path (hps_gpu_ctx_comm_init; sharded.cu)
  // The last persistent dedup launched by any table of this context: the next one waits for it.
  // A k_dedup grid needs all its CTAs resident at once (grid barriers); two running together
  // (two tables, e.g. the hybrid hot + cold groups, or two batch slots) could each hold part of
  // the SMs the other needs. (Owned by the table slot that recorded it; cleared on its destroy.)
  cudaEvent_t ev_last_dedup = nullptr;
  unsigned long long last_dedup_capture = 0;
  int rank = 0, world = 1;
};
namespace hpsg {
void comm_destroy(hps_gpu_ctx_s* ctx);  // sharded.cu
}
