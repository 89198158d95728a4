// update.cu — UpdateBatch frames into the GPU cache (the online
// update flow "publish -> refresh" of SPEC.md:60-77, 149-157, 419-423).
//
// Frame layout (little-endian; the reference's ByteWriter/ByteReader,
// proj/include/hps/bytes.hpp:33-133, define the primitive encodings):
//   "HPSU" | version u8 = 1 | name_len u16 | name | seq u64 | count u32 | dim u16 |
//   dtype u8 | count x (key u64, dim scalars: 4 B F32 or 2 B F16)
// The host validates the header, the exact length (Truncated / TrailingBytes) and key
// uniqueness (DuplicateKey); the raw entry bytes then go to the device ONCE and a decode
// kernel scatters them into aligned key / fp32 row / version arrays (F16 widened exactly,
// kernels_scalar.cpp's f16_to_f32), which feed the cache refresh (K8) with version = seq.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "hps/types.hpp"

using namespace hpsg;

namespace hpsg {
int cache_info(hps_gpu_cache c, hps_gpu_ctx* ctx, uint32_t* dim);  // cache.cu
}

namespace {

struct Cursor {  // bounds-checked little-endian reads (Truncated past the end)
  const uint8_t* p;
  uint64_t n, pos = 0;
  bool ok = true;
  bool need(uint64_t k) {
    if (n - pos < k) ok = false;
    return ok;
  }
  uint64_t le(int bytes) {
    if (!need(bytes)) return 0;
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= uint64_t(p[pos + i]) << (8 * i);
    pos += bytes;
    return v;
  }
};

void put_le(std::vector<uint8_t>& out, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

__global__ void k_decode_entries(const uint8_t* __restrict__ ent, uint64_t stride, uint32_t count, uint32_t dim,
                                 int dtype, uint64_t seq, uint64_t* __restrict__ keys, float* __restrict__ vecs,
                                 uint64_t* __restrict__ versions) {
  const uint64_t total = uint64_t(count) * dim;
  const uint64_t step = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < count; e += step) {
    const uint8_t* p = ent + e * stride;
    uint64_t k = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) k |= uint64_t(p[i]) << (8 * i);
    keys[e] = k;
    if (versions) versions[e] = seq;
  }
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += step) {
    const uint64_t e = i / dim, j = i % dim;
    const uint8_t* p = ent + e * stride + 8;
    if (dtype == 0) {
      const uint32_t b = uint32_t(p[4 * j]) | uint32_t(p[4 * j + 1]) << 8 | uint32_t(p[4 * j + 2]) << 16 |
                         uint32_t(p[4 * j + 3]) << 24;
      vecs[i] = __uint_as_float(b);
    } else {
      const unsigned short h = static_cast<unsigned short>(p[2 * j] | (p[2 * j + 1] << 8));
      vecs[i] = __half2float(__ushort_as_half(h));  // exact widening (NaN/Inf stay non-finite)
    }
  }
}

}  // namespace

extern "C" {

int hps_update_batch_parse(const uint8_t* frame, uint64_t n, hps_update_header* h) {
  if (!frame || !h) return HPS_GPU_E_INVALID_ARGUMENT;
  std::memset(h, 0, sizeof(*h));
  Cursor c{frame, n};
  if (!c.need(4)) return HPS_GPU_E_TRUNCATED;
  if (std::memcmp(frame, "HPSU", 4) != 0) {
    set_last_error("update batch: bad magic");
    return HPS_GPU_E_BAD_MAGIC;
  }
  c.pos = 4;
  const uint64_t version = c.le(1);
  if (!c.ok) return HPS_GPU_E_TRUNCATED;
  if (version != 1) {
    set_last_error("update batch: unsupported format version");
    return HPS_GPU_E_BAD_FORMAT_VERSION;
  }
  const uint64_t name_len = c.le(2);
  if (!c.need(name_len)) return HPS_GPU_E_TRUNCATED;
  if (name_len > 255) {
    set_last_error("update batch: table name longer than 255 bytes");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  std::memcpy(h->table, frame + c.pos, name_len);
  h->table[name_len] = '\0';
  h->name_len = static_cast<uint32_t>(name_len);
  c.pos += name_len;
  h->seq = c.le(8);
  h->count = static_cast<uint32_t>(c.le(4));
  h->dim = static_cast<uint32_t>(c.le(2));
  const uint64_t dtype = c.le(1);
  if (!c.ok) return HPS_GPU_E_TRUNCATED;
  if (dtype > 1) {
    set_last_error("update batch: unknown dtype byte");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  h->dtype = static_cast<int>(dtype);
  if (h->dim == 0 || h->dim > hps::kMaxDim) {
    set_last_error("update batch: dim outside [1, 4096]");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  h->entries_offset = c.pos;
  h->entry_bytes = 8 + uint64_t(h->dim) * (dtype == 0 ? 4 : 2);
  const uint64_t body = uint64_t(h->count) * h->entry_bytes;
  if (n - c.pos < body) {
    set_last_error("update batch: payload truncated");
    return HPS_GPU_E_TRUNCATED;
  }
  if (n - c.pos > body) {
    set_last_error("update batch: trailing bytes");
    return HPS_GPU_E_TRAILING_BYTES;
  }
  std::vector<uint64_t> keys(h->count);
  for (uint32_t e = 0; e < h->count; ++e) {
    const uint8_t* p = frame + c.pos + e * h->entry_bytes;
    uint64_t k = 0;
    for (int i = 0; i < 8; ++i) k |= uint64_t(p[i]) << (8 * i);
    keys[e] = k;
  }
  std::sort(keys.begin(), keys.end());
  if (std::adjacent_find(keys.begin(), keys.end()) != keys.end()) {
    set_last_error("update batch: duplicate key");
    return HPS_GPU_E_DUPLICATE_KEY;
  }
  return HPS_GPU_OK;
}

int hps_update_batch_encode(const char* table, uint32_t name_len, uint64_t seq, uint32_t count, uint32_t dim,
                            int dtype, const uint64_t* keys, const void* values, uint8_t* out, uint64_t out_cap,
                            uint64_t* out_len) {
  if (!out_len || (name_len && !table) || (count && (!keys || !values))) return HPS_GPU_E_INVALID_ARGUMENT;
  if (name_len > 255 || dim == 0 || dim > 0xffff || (dtype != 0 && dtype != 1)) {
    set_last_error("update batch encode: name length > 255, bad dim or dtype");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  const uint64_t esz = dtype == 0 ? 4 : 2;
  const uint64_t len = 4 + 1 + 2 + name_len + 8 + 4 + 2 + 1 + uint64_t(count) * (8 + dim * esz);
  *out_len = len;
  if (!out) return HPS_GPU_OK;  // size query
  if (out_cap < len) return HPS_GPU_E_INVALID_ARGUMENT;
  std::vector<uint8_t> b;
  b.reserve(len);
  b.insert(b.end(), {'H', 'P', 'S', 'U'});
  put_le(b, 1, 1);
  put_le(b, name_len, 2);
  b.insert(b.end(), table, table + name_len);
  put_le(b, seq, 8);
  put_le(b, count, 4);
  put_le(b, dim, 2);
  put_le(b, static_cast<uint64_t>(dtype), 1);
  const uint8_t* v = static_cast<const uint8_t*>(values);
  for (uint32_t e = 0; e < count; ++e) {
    put_le(b, keys[e], 8);
    const uint8_t* row = v + uint64_t(e) * dim * esz;  // scalars are little-endian in memory (x86/arm)
    b.insert(b.end(), row, row + dim * esz);
  }
  std::memcpy(out, b.data(), len);
  return HPS_GPU_OK;
}

int hps_gpu_update_decode(hps_gpu_ctx ctx, const uint8_t* entries_dev, const hps_update_header* h, uint64_t* keys_out,
                          float* vecs_out, uint64_t* versions_out) {
  if (!ctx || !h || (h->count && (!entries_dev || !keys_out || !vecs_out))) return HPS_GPU_E_INVALID_ARGUMENT;
  if (h->count == 0) return HPS_GPU_OK;
  const uint64_t work = std::max<uint64_t>(h->count, uint64_t(h->count) * h->dim);
  k_decode_entries<<<grid_for(work, 256, kNumSMs * 16), 256, 0, ctx->stream>>>(
      entries_dev, h->entry_bytes, h->count, h->dim, h->dtype, h->seq, keys_out, vecs_out, versions_out);
  HPSG_CHECK_LAUNCH("k_decode_entries");
  return HPS_GPU_OK;
}

int hps_gpu_cache_apply_update(hps_gpu_cache c, const uint8_t* frame_host, uint64_t n, uint64_t* replaced_out) {
  if (!c || !frame_host) return HPS_GPU_E_INVALID_ARGUMENT;
  hps_update_header h;
  if (int s = hps_update_batch_parse(frame_host, n, &h)) return s;
  uint32_t cache_dim = 0;
  hps_gpu_ctx ctx = nullptr;
  if (int s = hpsg::cache_info(c, &ctx, &cache_dim)) return s;
  if (h.dim != cache_dim) {
    set_last_error("update batch: dim differs from the cache's");
    return HPS_GPU_E_DIM_MISMATCH;
  }
  cudaStream_t st = ctx->stream;
  if (h.count == 0) {
    if (replaced_out) HPSG_CUDA(cudaMemsetAsync(replaced_out, 0, sizeof(uint64_t), st));
    return HPS_GPU_OK;
  }
  const uint64_t body = uint64_t(h.count) * h.entry_bytes;
  uint8_t* d_ent = nullptr;
  uint64_t *d_keys = nullptr, *d_ver = nullptr;
  float* d_vecs = nullptr;
  // control-plane call: stream-ordered scratch (the entry bytes cross PCIe once)
  HPSG_CUDA(cudaMallocAsync(&d_ent, body, st));
  HPSG_CUDA(cudaMallocAsync(&d_keys, h.count * sizeof(uint64_t), st));
  HPSG_CUDA(cudaMallocAsync(&d_ver, h.count * sizeof(uint64_t), st));
  HPSG_CUDA(cudaMallocAsync(&d_vecs, uint64_t(h.count) * h.dim * sizeof(float), st));
  HPSG_CUDA(cudaMemcpyAsync(d_ent, frame_host + h.entries_offset, body, cudaMemcpyHostToDevice, st));
  int s = hps_gpu_update_decode(ctx, d_ent, &h, d_keys, d_vecs, d_ver);
  if (!s) s = hps_gpu_cache_refresh(c, d_keys, d_vecs, d_ver, h.count, replaced_out);
  cudaFreeAsync(d_ent, st);
  cudaFreeAsync(d_keys, st);
  cudaFreeAsync(d_ver, st);
  cudaFreeAsync(d_vecs, st);
  if (!s) HPSG_CUDA(cudaStreamSynchronize(st));  // the host frame may be reused once we return
  return s;
}

}  // extern "C"
