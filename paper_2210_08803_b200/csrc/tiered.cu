// tiered.cu — the orchestrator's three-tier lookup:
// L1 = the HPS GPU cache, L2 = the VDB (host shards, tiers.cpp), L3 = the PDB (disk log).
//
//   1  keys D2H; distinct keys in first-occurrence order + the inverse map (one tier probe per
//      distinct key)
//   2  L1: hps_gpu_cache_query over the distinct keys on the device (frequency side effects
//      once per distinct key); hit rows land compacted (input order) in `urows`
//   3  the misses: VDB get_batch, then PDB get_batch for what is still missing, else the PDB
//      table's default vector (source Default); their rows go H2D right after the hits, so
//      urows = [L1 hits | misses] and every input key reads urows[row_of[i]]
//   4  k_tier_expand: out[i] = urows[row_of[i]] (device, LPR lanes per row, 128-bit)
//   5  migrations, started and not waited for (the MigrationTicket of SPEC.md): L2 and L3 hits
//      are inserted into L1 on the context's stream (async copies + hps_gpu_cache_insert at
//      their tier versions); L3-only hits are put into the VDB by a host thread.
//      hps_gpu_tiered_await joins both; the next lookup awaits the previous migrations first.
// The miss path is host/IO work by nature (the tiers live in CPU memory and on disk); the
// L1 part stays on the GPU and the rows never round-trip through the host for hits.
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

using namespace hpsg;

namespace hpsg {
int cache_info(hps_gpu_cache c, hps_gpu_ctx* ctx, uint32_t* dim);
uint64_t cache_max_batch(hps_gpu_cache c);
}  // namespace hpsg

struct hps_gpu_tiered_s {
  hps_gpu_cache l1 = nullptr;
  hps_vdb l2 = nullptr;
  hps_pdb l3 = nullptr;
  std::string table;
  hps_gpu_ctx ctx = nullptr;
  uint32_t dim = 0;
  uint64_t max_batch = 0;
  // device
  uint64_t* d_ukeys = nullptr;
  float* d_urows = nullptr;        // [max_batch x dim]: L1 hit rows, then the miss rows
  uint32_t* d_found_idx = nullptr;
  uint32_t* d_missing_idx = nullptr;
  uint64_t* d_counts = nullptr;
  uint32_t* d_row_of = nullptr;    // input key -> urows row
  uint64_t* d_mig_keys = nullptr;  // migration into L1
  float* d_mig_vecs = nullptr;
  uint64_t* d_mig_ver = nullptr;
  // pinned host
  uint64_t* h_keys = nullptr;
  uint64_t* h_ukeys = nullptr;
  uint32_t* h_row_of = nullptr;
  uint32_t* h_missing_idx = nullptr;
  uint64_t* h_counts = nullptr;
  float* h_rows = nullptr;         // miss rows [max_batch x dim]
  uint64_t* h_mig_keys = nullptr;
  float* h_mig_vecs = nullptr;
  uint64_t* h_mig_ver = nullptr;
  std::vector<float> def;          // the PDB table's default vector
  std::thread mig;                 // the last lookup's L3 -> L2 migration
  int mig_status = HPS_GPU_OK;
  cudaEvent_t ev_mig = nullptr;    // the last lookup's L1 insertion is enqueued before this
};

namespace {
template <int LPR>
__global__ void __launch_bounds__(256) k_tier_expand(const float* __restrict__ urows, const uint32_t* __restrict__ row_of,
                                                     uint64_t n, uint32_t dim, float* __restrict__ out) {
  constexpr int G = 32 / LPR;
  const uint32_t lane = lane_id(), grp = lane / LPR, gl = lane % LPR;
  const uint64_t gid = ((blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5) * G + grp;
  const uint64_t ng = ((uint64_t(gridDim.x) * blockDim.x) >> 5) * G;
  for (uint64_t i = gid; i < n; i += ng) {
    const float* src = urows + uint64_t(row_of[i]) * dim;
    float* dst = out + i * dim;
    if ((dim & 3u) == 0) {
      for (uint32_t v = gl; v < dim / 4; v += LPR)
        reinterpret_cast<float4*>(dst)[v] = __ldg(reinterpret_cast<const float4*>(src) + v);
    } else {
      for (uint32_t v = gl; v < dim; v += LPR) dst[v] = __ldg(src + v);
    }
  }
}

int lpr_of(uint32_t dim) {
  const uint32_t nvec = (dim + 3) / 4;
  return nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
}

template <class T>
int dev_alloc(T** p, uint64_t n) {
  if (cudaMalloc(reinterpret_cast<void**>(p), std::max<uint64_t>(n, 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}
template <class T>
int host_alloc(T** p, uint64_t n) {
  if (cudaHostAlloc(reinterpret_cast<void**>(p), std::max<uint64_t>(n, 1) * sizeof(T), cudaHostAllocDefault) !=
      cudaSuccess) {
    cudaGetLastError();
    return HPS_GPU_E_OUT_OF_MEMORY;
  }
  return HPS_GPU_OK;
}

int await_migrations(hps_gpu_tiered t) {
  if (t->mig.joinable()) t->mig.join();
  HPSG_CUDA(cudaEventSynchronize(t->ev_mig));
  const int s = t->mig_status;
  t->mig_status = HPS_GPU_OK;
  return s;
}
}  // namespace

extern "C" {

int hps_gpu_tiered_create(hps_gpu_cache l1, hps_vdb l2, hps_pdb l3, const char* table, uint64_t max_batch,
                          hps_gpu_tiered* out) {
  if (!l1 || !l2 || !l3 || !table || !out || max_batch == 0 || max_batch >= (1ull << 31))
    return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  hps_gpu_ctx ctx = nullptr;
  uint32_t dim = 0;
  if (int s = cache_info(l1, &ctx, &dim)) return s;
  if (max_batch > cache_max_batch(l1)) {
    set_last_error("tiered: max_batch exceeds the L1 cache's max_batch");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  uint32_t pdim = 0;
  if (int s = hps_pdb_table_info(l3, table, &pdim, nullptr, nullptr)) return s;
  if (pdim != dim) return HPS_GPU_E_DIM_MISMATCH;
  HPSG_CUDA(cudaSetDevice(ctx->device));
  auto t = new hps_gpu_tiered_s;
  t->l1 = l1;
  t->l2 = l2;
  t->l3 = l3;
  t->table = table;
  t->ctx = ctx;
  t->dim = dim;
  t->max_batch = max_batch;
  t->def.resize(dim);
  const uint64_t N = max_batch, D = dim;
  int st = hps_pdb_table_info(l3, table, nullptr, t->def.data(), nullptr);
  auto A = [&](int s) {
    if (s && !st) st = s;
  };
  A(dev_alloc(&t->d_ukeys, N));
  A(dev_alloc(&t->d_urows, N * D));
  A(dev_alloc(&t->d_found_idx, N));
  A(dev_alloc(&t->d_missing_idx, N));
  A(dev_alloc(&t->d_counts, 4));
  A(dev_alloc(&t->d_row_of, N));
  A(dev_alloc(&t->d_mig_keys, N));
  A(dev_alloc(&t->d_mig_vecs, N * D));
  A(dev_alloc(&t->d_mig_ver, N));
  A(host_alloc(&t->h_keys, N));
  A(host_alloc(&t->h_ukeys, N));
  A(host_alloc(&t->h_row_of, N));
  A(host_alloc(&t->h_missing_idx, N));
  A(host_alloc(&t->h_counts, 4));
  A(host_alloc(&t->h_rows, N * D));
  A(host_alloc(&t->h_mig_keys, N));
  A(host_alloc(&t->h_mig_vecs, N * D));
  A(host_alloc(&t->h_mig_ver, N));
  if (!st && cudaEventCreateWithFlags(&t->ev_mig, cudaEventDisableTiming) != cudaSuccess) st = HPS_GPU_E_CUDA;
  if (!st && cudaEventRecord(t->ev_mig, ctx->stream) != cudaSuccess) st = HPS_GPU_E_CUDA;
  if (st) {
    hps_gpu_tiered_destroy(t);
    return st;
  }
  *out = t;
  return HPS_GPU_OK;
}

int hps_gpu_tiered_destroy(hps_gpu_tiered t) {
  if (!t) return HPS_GPU_OK;
  if (t->mig.joinable()) t->mig.join();
  if (t->ev_mig) {
    cudaEventSynchronize(t->ev_mig);
    cudaEventDestroy(t->ev_mig);
  }
  for (void* p : {static_cast<void*>(t->d_ukeys), static_cast<void*>(t->d_urows), static_cast<void*>(t->d_found_idx),
                  static_cast<void*>(t->d_missing_idx), static_cast<void*>(t->d_counts), static_cast<void*>(t->d_row_of),
                  static_cast<void*>(t->d_mig_keys), static_cast<void*>(t->d_mig_vecs),
                  static_cast<void*>(t->d_mig_ver)})
    if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(t->h_keys), static_cast<void*>(t->h_ukeys), static_cast<void*>(t->h_row_of),
                  static_cast<void*>(t->h_missing_idx), static_cast<void*>(t->h_counts), static_cast<void*>(t->h_rows),
                  static_cast<void*>(t->h_mig_keys), static_cast<void*>(t->h_mig_vecs),
                  static_cast<void*>(t->h_mig_ver)})
    if (p) cudaFreeHost(p);
  delete t;
  return HPS_GPU_OK;
}

int hps_gpu_tiered_await(hps_gpu_tiered t) {
  if (!t) return HPS_GPU_E_INVALID_ARGUMENT;
  return await_migrations(t);
}

int hps_gpu_tiered_lookup(hps_gpu_tiered t, const uint64_t* keys, uint64_t n, float* out, uint64_t* source_counts) {
  if (!t || !source_counts || n > t->max_batch || (n && (!keys || !out))) return HPS_GPU_E_INVALID_ARGUMENT;
  for (int k = 0; k < 4; ++k) source_counts[k] = 0;
  if (int s = await_migrations(t)) return s;  // the previous lookup's migrations are visible
  if (n == 0) return HPS_GPU_OK;
  cudaStream_t st = t->ctx->stream;
  const uint64_t D = t->dim;
  // 1. distinct keys, first-occurrence order
  HPSG_CUDA(cudaMemcpyAsync(t->h_keys, keys, n * 8, cudaMemcpyDeviceToHost, st));
  HPSG_CUDA(cudaStreamSynchronize(st));
  std::unordered_map<uint64_t, uint32_t> first;
  first.reserve(n * 2);
  std::vector<uint32_t> inv(n);
  uint64_t u = 0;
  for (uint64_t i = 0; i < n; ++i) {
    auto r = first.emplace(t->h_keys[i], static_cast<uint32_t>(u));
    if (r.second) t->h_ukeys[u++] = t->h_keys[i];
    inv[i] = r.first->second;
  }
  // 2. L1 over the distinct keys (hits compacted into urows)
  HPSG_CUDA(cudaMemcpyAsync(t->d_ukeys, t->h_ukeys, u * 8, cudaMemcpyHostToDevice, st));
  if (int s = hps_gpu_cache_query(t->l1, t->d_ukeys, u, t->d_urows, t->d_found_idx, t->d_missing_idx, t->d_counts))
    return s;
  // the counts and the whole missing list (its valid prefix is counts[1] long) in one round trip
  HPSG_CUDA(cudaMemcpyAsync(t->h_counts, t->d_counts, 2 * 8, cudaMemcpyDeviceToHost, st));
  HPSG_CUDA(cudaMemcpyAsync(t->h_missing_idx, t->d_missing_idx, u * 4, cudaMemcpyDeviceToHost, st));
  HPSG_CUDA(cudaStreamSynchronize(st));
  const uint64_t nf = t->h_counts[0], nm = t->h_counts[1];
  // 3. the misses: L2, then L3, else the default vector
  std::vector<uint8_t> src(u, 0);  // 0 L1, 1 L2, 2 L3, 3 Default
  std::vector<uint32_t> urow(u);
  {
    uint64_t m = 0, h = 0;
    for (uint64_t j = 0; j < u; ++j) {  // hits are the complement of the ascending missing list
      if (m < nm && t->h_missing_idx[m] == j) {
        urow[j] = static_cast<uint32_t>(nf + m);
        ++m;
      } else {
        urow[j] = static_cast<uint32_t>(h++);
      }
    }
  }
  std::vector<uint64_t> mkeys(nm), mver(nm);
  std::vector<uint8_t> f2(nm), f3;
  uint64_t n_mig = 0;
  std::vector<uint64_t> l3_keys, l3_ver;
  std::vector<float> l3_vecs;
  if (nm) {
    for (uint64_t m = 0; m < nm; ++m) mkeys[m] = t->h_ukeys[t->h_missing_idx[m]];
    if (int s = hps_vdb_get_batch(t->l2, mkeys.data(), nm, t->h_rows, mver.data(), f2.data(), nullptr)) return s;
    std::vector<uint64_t> rest;
    std::vector<uint32_t> rest_m;
    for (uint64_t m = 0; m < nm; ++m) {
      if (f2[m]) {
        src[t->h_missing_idx[m]] = 1;
        t->h_mig_keys[n_mig] = mkeys[m];
        t->h_mig_ver[n_mig] = mver[m];
        std::memcpy(t->h_mig_vecs + n_mig * D, t->h_rows + m * D, D * 4);
        ++n_mig;
      } else {
        rest.push_back(mkeys[m]);
        rest_m.push_back(static_cast<uint32_t>(m));
      }
    }
    if (!rest.empty()) {
      std::vector<float> v3(rest.size() * D);
      std::vector<uint64_t> ver3(rest.size());
      f3.assign(rest.size(), 0);
      if (int s = hps_pdb_get_batch(t->l3, t->table.c_str(), rest.data(), rest.size(), v3.data(), ver3.data(), f3.data(),
                                    nullptr))
        return s;
      for (size_t q = 0; q < rest.size(); ++q) {
        const uint32_t m = rest_m[q];
        float* row = t->h_rows + uint64_t(m) * D;
        if (f3[q]) {
          src[t->h_missing_idx[m]] = 2;
          std::memcpy(row, &v3[q * D], D * 4);
          t->h_mig_keys[n_mig] = rest[q];
          t->h_mig_ver[n_mig] = ver3[q];
          std::memcpy(t->h_mig_vecs + n_mig * D, row, D * 4);
          ++n_mig;
          l3_keys.push_back(rest[q]);
          l3_ver.push_back(ver3[q]);
          l3_vecs.insert(l3_vecs.end(), row, row + D);
        } else {
          src[t->h_missing_idx[m]] = 3;
          std::memcpy(row, t->def.data(), D * 4);  // absent everywhere: default, migrated nowhere
        }
      }
    }
    HPSG_CUDA(cudaMemcpyAsync(t->d_urows + nf * D, t->h_rows, nm * D * 4, cudaMemcpyHostToDevice, st));
  }
  // 4. rows in input order
  for (uint64_t i = 0; i < n; ++i) {
    t->h_row_of[i] = urow[inv[i]];
    ++source_counts[src[inv[i]]];
  }
  HPSG_CUDA(cudaMemcpyAsync(t->d_row_of, t->h_row_of, n * 4, cudaMemcpyHostToDevice, st));
  {
    const int lpr = lpr_of(t->dim);
    const int grid = grid_for(n * lpr, 256, kNumSMs * 16);
    switch (lpr) {
      case 32: k_tier_expand<32><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
      case 16: k_tier_expand<16><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
      case 8: k_tier_expand<8><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
      case 4: k_tier_expand<4><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
      case 2: k_tier_expand<2><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
      default: k_tier_expand<1><<<grid, 256, 0, st>>>(t->d_urows, t->d_row_of, n, t->dim, out); break;
    }
    HPSG_CHECK_LAUNCH("k_tier_expand");
  }
  // 5. migrations (not waited for): L2/L3 hits -> L1 on the stream; L3-only hits -> L2 on a thread
  if (n_mig) {
    HPSG_CUDA(cudaMemcpyAsync(t->d_mig_keys, t->h_mig_keys, n_mig * 8, cudaMemcpyHostToDevice, st));
    HPSG_CUDA(cudaMemcpyAsync(t->d_mig_vecs, t->h_mig_vecs, n_mig * D * 4, cudaMemcpyHostToDevice, st));
    HPSG_CUDA(cudaMemcpyAsync(t->d_mig_ver, t->h_mig_ver, n_mig * 8, cudaMemcpyHostToDevice, st));
    if (int s = hps_gpu_cache_insert(t->l1, t->d_mig_keys, t->d_mig_vecs, t->d_mig_ver, n_mig, nullptr)) return s;
  }
  HPSG_CUDA(cudaEventRecord(t->ev_mig, st));
  if (!l3_keys.empty()) {
    t->mig = std::thread([t, k = std::move(l3_keys), v = std::move(l3_vecs), ver = std::move(l3_ver)]() {
      t->mig_status = hps_vdb_put_batch(t->l2, k.data(), v.data(), ver.data(), k.size(), nullptr);
    });
  }
  return HPS_GPU_OK;
}

}  // extern "C"
