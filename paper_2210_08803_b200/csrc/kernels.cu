// kernels.cu — the reference's value-payload kernel API (proj/include/hps/kernels.hpp:33-43)
// on the B200: f32_to_f16, f16_to_f32, crc32c, has_non_finite_f32/_f16 over device buffers,
// bit-equivalent to the reference's scalar path (kernels_scalar.cpp:25-123, pinned by the
// golden vectors oracle/gen_golden.py records from the reference's own compiled code).
//
// CRC-32C in parallel: the CRC of a concatenation is linear in its parts,
//   crc(A || B) = shift(crc(A), |B|) ^ crc(B),
// where shift(c, L) multiplies c by x^(8L) modulo the Castagnoli polynomial (the combine
// identity of zlib's crc32_combine, with reflected polynomial 0x82f63b78). So every thread
// (or lane) takes the CRC of its own chunk, shifts it past the bytes after the chunk, and the
// shifted CRCs XOR-reduce in any order: one pass over the bytes at full width, no carry chain.
// hps_gpu_crc32c_batch gives one CRC per record (a warp per record: the PDB log-record
// checksum over each record's bytes).
#include "common.cuh"

using namespace hpsg;

namespace {

constexpr uint32_t kCastagnoli = 0x82f63b78u;  // reflected

__device__ __forceinline__ uint32_t crc_byte_table(uint32_t i) {
  uint32_t c = i;
#pragma unroll
  for (int k = 0; k < 8; ++k) c = (c & 1u) ? (kCastagnoli ^ (c >> 1)) : (c >> 1);
  return c;
}

// a(x) * b(x) mod P in the reflected representation (bit 31 = x^0).
__device__ __forceinline__ uint32_t mulmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  while (a) {
    if (a & m) {
      p ^= b;
      a &= ~m;
    }
    m >>= 1;
    b = (b & 1u) ? (b >> 1) ^ kCastagnoli : b >> 1;
  }
  return p;
}

// x^(8 * len) mod P: square-and-multiply over the bits of len (x^8 = one byte of shift).
__device__ __forceinline__ uint32_t xpow8n(uint64_t len) {
  uint32_t result = 1u << 31;  // x^0
  uint32_t sq = 1u << 23;      // x^8
  while (len) {
    if (len & 1u) result = mulmodp(sq, result);
    sq = mulmodp(sq, sq);
    len >>= 1;
  }
  return result;
}

// conditioned CRC-32C of bytes [p, p + n) from crc 0 (kernels_scalar.cpp:100-106 semantics)
__device__ __forceinline__ uint32_t crc_bytes(const uint8_t* __restrict__ p, uint64_t n, const uint32_t* table) {
  uint32_t c = 0xffffffffu;
  for (uint64_t i = 0; i < n; ++i) c = table[(c ^ __ldg(p + i)) & 0xffu] ^ (c >> 8);
  return c ^ 0xffffffffu;
}

constexpr uint32_t kCrcChunk = 512;  // bytes per thread

__global__ void __launch_bounds__(256) k_crc32c(const uint8_t* __restrict__ data, uint64_t n,
                                                uint32_t* __restrict__ acc) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t s_w[8];
  table[threadIdx.x] = crc_byte_table(threadIdx.x);
  __syncthreads();
  uint32_t mine = 0;
  const uint64_t chunks = (n + kCrcChunk - 1) / kCrcChunk;
  for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < chunks; c += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = c * kCrcChunk, e = min(n, b + kCrcChunk);
    mine ^= mulmodp(xpow8n(n - e), crc_bytes(data + b, e - b, table));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine ^= __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t x = 0;
    for (int w = 0; w < 8; ++w) x ^= s_w[w];
    if (x) atomicXor(acc, x);
  }
}

// out = combine(crc_in, crc(data), n): shift the running value past the n new bytes.
__global__ void k_crc32c_finish(uint32_t crc_in, uint64_t n, const uint32_t* acc, uint32_t* out) {
  if (threadIdx.x == 0) *out = mulmodp(xpow8n(n), crc_in) ^ *acc;
}

// One record per warp: lane l takes 64-byte pieces l, l+32, ... of the record.
__global__ void __launch_bounds__(256) k_crc32c_batch(const uint8_t* __restrict__ data,
                                                      const uint64_t* __restrict__ offsets, uint64_t n_rec,
                                                      uint32_t* __restrict__ out) {
  __shared__ uint32_t table[256];
  table[threadIdx.x] = crc_byte_table(threadIdx.x);
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = warp; r < n_rec; r += n_warps) {
    const uint64_t b = offsets[r], e = offsets[r + 1];
    uint32_t mine = 0;
    for (uint64_t p = b + uint64_t(lane) * 64; p < e; p += 32 * 64) {
      const uint64_t q = min(e, p + 64);
      mine ^= mulmodp(xpow8n(e - q), crc_bytes(data + p, q - p, table));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine ^= __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) out[r] = mine;
  }
}

// kernels_scalar.cpp:25-57 semantics: round-to-nearest-even (the hardware cvt.rn.f16.f32 for
// every non-NaN input: overflow to the infinity pattern, subnormals, ties); NaN keeps its top
// payload bits plus the quiet bit (cvt would canonicalise it).
__device__ __forceinline__ uint16_t f32_to_f16_bits(uint32_t bits) {
  const uint32_t abs = bits & 0x7fffffffu;
  if (abs > 0x7f800000u)
    return static_cast<uint16_t>(((bits >> 16) & 0x8000u) | 0x7c00u | ((abs >> 13) & 0x3ffu) | 0x200u);
  return __half_as_ushort(__float2half_rn(__uint_as_float(bits)));
}

// kernels_scalar.cpp:59-77: exact widening; NaN keeps its payload (m << 13).
__device__ __forceinline__ uint32_t f16_to_f32_bits(uint16_t h) {
  if ((h & 0x7c00u) == 0x7c00u) return (static_cast<uint32_t>(h & 0x8000u) << 16) | 0x7f800000u | (uint32_t(h & 0x3ffu) << 13);
  return __float_as_uint(__half2float(__ushort_as_half(h)));
}

__global__ void k_f32_to_f16(const uint32_t* __restrict__ src, uint16_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = f32_to_f16_bits(src[i]);
}

__global__ void k_f16_to_f32(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = f16_to_f32_bits(src[i]);
}

__global__ void k_non_finite_f16(const uint16_t* __restrict__ v, uint64_t n, uint32_t* flag) {
  bool any = false;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    any |= (v[i] & 0x7c00u) == 0x7c00u;
  if (__any_sync(0xffffffffu, any) && lane_id() == 0) atomicOr(flag, 1u);
}

int check_ctx_ptrs(hps_gpu_ctx ctx, bool ok) { return (!ctx || !ok) ? HPS_GPU_E_INVALID_ARGUMENT : HPS_GPU_OK; }

}  // namespace

extern "C" {

int hps_gpu_f32_to_f16(hps_gpu_ctx ctx, const float* src, uint16_t* dst, uint64_t n) {
  if (int s = check_ctx_ptrs(ctx, n == 0 || (src && dst))) return s;
  if (n == 0) return HPS_GPU_OK;
  k_f32_to_f16<<<grid_for(n, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(reinterpret_cast<const uint32_t*>(src), dst, n);
  HPSG_CHECK_LAUNCH("k_f32_to_f16");
  return HPS_GPU_OK;
}

int hps_gpu_f16_to_f32(hps_gpu_ctx ctx, const uint16_t* src, float* dst, uint64_t n) {
  if (int s = check_ctx_ptrs(ctx, n == 0 || (src && dst))) return s;
  if (n == 0) return HPS_GPU_OK;
  k_f16_to_f32<<<grid_for(n, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(src, reinterpret_cast<uint32_t*>(dst), n);
  HPSG_CHECK_LAUNCH("k_f16_to_f32");
  return HPS_GPU_OK;
}

int hps_gpu_has_non_finite_f16(hps_gpu_ctx ctx, const uint16_t* v, uint64_t n, uint32_t* flag_out) {
  if (int s = check_ctx_ptrs(ctx, flag_out && (n == 0 || v))) return s;
  HPSG_CUDA(cudaMemsetAsync(flag_out, 0, sizeof(uint32_t), ctx->stream));
  if (n == 0) return HPS_GPU_OK;
  k_non_finite_f16<<<grid_for(n, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(v, n, flag_out);
  HPSG_CHECK_LAUNCH("k_non_finite_f16");
  return HPS_GPU_OK;
}

int hps_gpu_crc32c(hps_gpu_ctx ctx, uint32_t crc, const void* data, uint64_t n, uint32_t* scratch, uint32_t* crc_out) {
  if (int s = check_ctx_ptrs(ctx, scratch && crc_out && (n == 0 || data))) return s;
  cudaStream_t st = ctx->stream;
  HPSG_CUDA(cudaMemsetAsync(scratch, 0, sizeof(uint32_t), st));
  if (n) {
    const uint64_t chunks = (n + kCrcChunk - 1) / kCrcChunk;
    k_crc32c<<<grid_for(chunks, 256, kNumSMs * 8), 256, 0, st>>>(static_cast<const uint8_t*>(data), n, scratch);
  }
  k_crc32c_finish<<<1, 32, 0, st>>>(crc, n, scratch, crc_out);
  HPSG_CHECK_LAUNCH("k_crc32c");
  return HPS_GPU_OK;
}

int hps_gpu_crc32c_batch(hps_gpu_ctx ctx, const void* data, const uint64_t* offsets, uint64_t n_records,
                         uint32_t* crc_out) {
  if (int s = check_ctx_ptrs(ctx, n_records == 0 || (data && offsets && crc_out))) return s;
  if (n_records == 0) return HPS_GPU_OK;
  k_crc32c_batch<<<grid_for(n_records * 32, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(
      static_cast<const uint8_t*>(data), offsets, n_records, crc_out);
  HPSG_CHECK_LAUNCH("k_crc32c_batch");
  return HPS_GPU_OK;
}

}  // extern "C"
