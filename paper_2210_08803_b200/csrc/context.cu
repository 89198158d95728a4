// context.cu — context, status plumbing and K1 (hash / partition / finiteness) kernels.
//
// K1 replaces the reference's per-key placement loop (proj/include/hps/hash.hpp:42-54)
// and the ingest finiteness scan (proj/src/kernels/kernels_scalar.cpp:110-116,
// kernels_avx2.cpp:68-78) with grid-stride sm_100a kernels; the hash itself is the
// shared HPS_HD definition in include/hps/hash.hpp, so host and device cannot drift.
#include <cstdio>
#include <cstring>

#include <cstdlib>

#include "common.cuh"

namespace hpsg {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

int cuda_status(cudaError_t e, const char* what) {
  set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return HPS_GPU_E_OUT_OF_MEMORY;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return HPS_GPU_E_NO_DEVICE;
  if (e == cudaErrorStreamCaptureUnsupported || e == cudaErrorStreamCaptureInvalidated)
    return HPS_GPU_E_NOT_CAPTURABLE;
  return HPS_GPU_E_CUDA;
}

namespace {

__global__ void k_key_hash(const uint64_t* __restrict__ keys, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = hps::key_hash(keys[i]);
}

__global__ void k_partition_of(const uint64_t* __restrict__ keys, uint64_t n, hps::FastMod64 fm,
                               uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(fm.mod(hps::key_hash(keys[i])));
}

// Any NaN/Inf? 128-bit loads over the aligned body, scalar head/tail.
__global__ void k_non_finite(const float* __restrict__ v, uint64_t n, uint32_t* __restrict__ flag) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  bool bad = false;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(v) & 15u) / 4u;
  const uint64_t head = mis ? (4 - mis < n ? 4 - mis : n) : 0;
  if (tid < head) bad |= non_finite_bits(__float_as_uint(v[tid]));
  const uint64_t nv = (n - head) / 4;
  const uint4* b = reinterpret_cast<const uint4*>(v + head);
  for (uint64_t i = tid; i < nv; i += stride) {
    uint4 q = __ldg(b + i);
    bad |= non_finite_bits(q.x) | non_finite_bits(q.y) | non_finite_bits(q.z) | non_finite_bits(q.w);
  }
  for (uint64_t i = head + nv * 4 + tid; i < n; i += stride) bad |= non_finite_bits(__float_as_uint(v[i]));
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(flag, 1u);
}

__global__ void k_gen_keys(uint64_t seed, uint64_t first, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = mix64(seed ^ (first + i));
}

int check_ctx(hps_gpu_ctx ctx) {
  if (!ctx) {
    set_last_error("null context");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  return HPS_GPU_OK;
}

}  // namespace
}  // namespace hpsg

using namespace hpsg;

extern "C" {

int hps_gpu_abi_version(void) { return HPS_GPU_ABI_VERSION; }

const char* hps_gpu_last_error_message(void) { return g_last_error.c_str(); }

const char* hps_gpu_status_string(int status) {
  switch (status) {
    case 0: return "OK";
    case 1: return "InvalidArgument";
    case 2: return "BadMagic";
    case 3: return "BadFormatVersion";
    case 4: return "Truncated";
    case 5: return "TrailingBytes";
    case 6: return "DuplicateKey";
    case 7: return "DimMismatch";
    case 8: return "DtypeMismatch";
    case 9: return "F16Range";
    case 10: return "NonFinite";
    case 11: return "UnknownTable";
    case 12: return "TableExists";
    case 13: return "BadShard";
    case 14: return "Io";
    case 15: return "Corruption";
    case 16: return "Infeasible";
    case 17: return "Protocol";
    case HPS_GPU_E_CUDA: return "CudaError";
    case HPS_GPU_E_OUT_OF_MEMORY: return "OutOfMemory";
    case HPS_GPU_E_NO_DEVICE: return "NoDevice";
    case HPS_GPU_E_NOT_CAPTURABLE: return "NotCapturable";
    case HPS_GPU_E_NCCL: return "Nccl";
    case HPS_GPU_E_PEER_TIMEOUT: return "PeerTimeout";
    default: return "Unknown";
  }
}

int hps_gpu_ctx_create(int device, void* stream, hps_gpu_ctx* out) {
  if (!out) return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_last_error("no CUDA device visible: the B200 path has no CPU fallback");
    return HPS_GPU_E_NO_DEVICE;
  }
  if (device < 0 || device >= n) return HPS_GPU_E_INVALID_ARGUMENT;
  cudaDeviceProp prop;
  HPSG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_last_error(std::string("device ") + prop.name + " is not sm_100 (Blackwell B200); kernels are built for sm_100a only");
    return HPS_GPU_E_NO_DEVICE;
  }
  HPSG_CUDA(cudaSetDevice(device));
  auto* c = new hps_gpu_ctx_s;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->stream = static_cast<cudaStream_t>(stream);
  if (const char* e = std::getenv("HPS_GPU_NO_PDL")) c->pdl = e[0] != '1';
  if (cudaMalloc(&c->d_status, sizeof(uint32_t)) != cudaSuccess ||
      cudaMallocHost(&c->h_status, sizeof(uint32_t)) != cudaSuccess) {
    delete c;
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  HPSG_CUDA(cudaMemset(c->d_status, 0, sizeof(uint32_t)));
  *out = c;
  return HPS_GPU_OK;
}

int hps_gpu_ctx_destroy(hps_gpu_ctx ctx) {
  if (!ctx) return HPS_GPU_OK;
  hpsg::comm_destroy(ctx);
  cudaFree(ctx->d_status);
  cudaFreeHost(ctx->h_status);
  delete ctx;
  return HPS_GPU_OK;
}

int hps_gpu_ctx_set_stream(hps_gpu_ctx ctx, void* stream) {
  if (int s = check_ctx(ctx)) return s;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return HPS_GPU_OK;
}

int hps_gpu_ctx_sync(hps_gpu_ctx ctx) {
  if (int s = check_ctx(ctx)) return s;
  HPSG_CUDA(cudaSetDevice(ctx->device));
  HPSG_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  HPSG_CUDA(cudaMemsetAsync(ctx->d_status, 0, sizeof(uint32_t), ctx->stream));
  HPSG_CUDA(cudaStreamSynchronize(ctx->stream));
  int st = static_cast<int>(*ctx->h_status);
  if (st) set_last_error(std::string("device reported ") + hps_gpu_status_string(st));
  return st;
}

int hps_gpu_key_hash(hps_gpu_ctx ctx, const uint64_t* keys, uint64_t n, uint64_t* out) {
  if (int s = check_ctx(ctx)) return s;
  if (n == 0) return HPS_GPU_OK;
  if (!keys || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  k_key_hash<<<grid_for(n, 256), 256, 0, ctx->stream>>>(keys, n, out);
  HPSG_CHECK_LAUNCH("k_key_hash");
  return HPS_GPU_OK;
}

int hps_gpu_partition_of(hps_gpu_ctx ctx, const uint64_t* keys, uint64_t n, uint32_t num_shards, uint32_t* out) {
  if (int s = check_ctx(ctx)) return s;
  if (num_shards == 0) {
    set_last_error("partition_of: num_shards must be >= 1");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  if (n == 0) return HPS_GPU_OK;
  if (!keys || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  k_partition_of<<<grid_for(n, 256), 256, 0, ctx->stream>>>(keys, n, hps::FastMod64(num_shards), out);
  HPSG_CHECK_LAUNCH("k_partition_of");
  return HPS_GPU_OK;
}

int hps_gpu_has_non_finite_f32(hps_gpu_ctx ctx, const float* v, uint64_t n, uint32_t* flag) {
  if (int s = check_ctx(ctx)) return s;
  if (!flag) return HPS_GPU_E_INVALID_ARGUMENT;
  HPSG_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), ctx->stream));
  if (n == 0) return HPS_GPU_OK;
  if (!v) return HPS_GPU_E_INVALID_ARGUMENT;
  k_non_finite<<<grid_for(n / 4 + 1, 256), 256, 0, ctx->stream>>>(v, n, flag);
  HPSG_CHECK_LAUNCH("k_non_finite");
  return HPS_GPU_OK;
}

float hps_gpu_init_value(uint64_t seed, uint64_t key, uint32_t j) { return hpsg::init_value(seed, key, j); }

int hps_gpu_gen_keys(hps_gpu_ctx ctx, uint64_t seed, uint64_t first, uint64_t n, uint64_t* out) {
  if (int s = check_ctx(ctx)) return s;
  if (n == 0) return HPS_GPU_OK;
  if (!out) return HPS_GPU_E_INVALID_ARGUMENT;
  k_gen_keys<<<grid_for(n, 256), 256, 0, ctx->stream>>>(seed, first, n, out);
  HPSG_CHECK_LAUNCH("k_gen_keys");
  return HPS_GPU_OK;
}

}  // extern "C"
