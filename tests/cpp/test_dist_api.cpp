// C++ driver of the sharded C-ABI (include/hps_gpu.h hps_gpu_dist_*, csrc/sharded.cu), as a
// reference-side C++ caller would use it. Exit 0 = pass.
//  1. NCCL world of one: hps_gpu_nccl_unique_id + hps_gpu_ctx_comm_init, then dist steps
//     against the unsharded path (lookup_pooled + backward_update) on a twin table: pooled
//     outputs and the final rows bitwise equal.
//  2. Loopback world of two (one thread per rank, hps_gpu_dist_create_loopback), with the
//     copy transport and with the peer-memory transport (HPS_DIST_PEER): each rank owns
//     partition_of(key, 2) == rank (proj/include/hps/hash.hpp:52-54); outputs and every owned
//     row bitwise equal to ONE table driven with the concatenated batch (rank-major).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include <hps/hash.hpp>
#include "hps_gpu.h"

#define REQUIRE(c)                                                        \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                           \
    }                                                                     \
  } while (0)
#define OK(call) REQUIRE((call) == 0)

namespace {
constexpr uint32_t kDim = 16, kB = 64, kS = 3;
const uint64_t kCaps[2] = {500, 7};
const uint32_t kSlots[kS] = {0, 1, 0};

template <class T>
T* dev(const std::vector<T>& h) {
  T* p = nullptr;
  cudaMalloc(&p, h.size() * sizeof(T));
  cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return p;
}
template <class T>
std::vector<T> host(const T* d, size_t n) {
  std::vector<T> h(n);
  cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost);
  return h;
}

// (the slot map only matters to the unsharded tables' lookup_pooled: a shard is addressed
// through the table ids the requesters send)
hps_gpu_table make_table(hps_gpu_ctx ctx, uint64_t max_keys) {
  hps_table_config c{};
  c.n_tables = 2;
  c.dim = kDim;
  c.row_capacity_host = kCaps;
  c.n_slots = kS;
  c.slot_table_host = kSlots;
  c.optimizer = HPS_OPT_ADAGRAD;
  c.max_batch_keys = max_keys;
  c.max_batch_bags = max_keys;
  c.init_seed = 11;
  c.adagrad_initial_accumulator = 0.1f;
  hps_gpu_table t = nullptr;
  return hps_gpu_table_create(ctx, &c, &t) == 0 ? t : nullptr;
}

hps_opt_params adagrad() {
  hps_opt_params p{};
  p.lr = 0.05f;
  p.eps = 1e-7f;
  return p;
}

// row values of `keys` in table t (weights then AdaGrad state), via find + export
std::vector<float> rows_of(hps_gpu_ctx ctx, hps_gpu_table tb, uint32_t t, const std::vector<uint64_t>& keys) {
  uint64_t* dk = dev(keys);
  uint64_t* dr = nullptr;
  cudaMalloc(&dr, keys.size() * 8);
  hps_gpu_table_find(tb, t, dk, keys.size(), dr);
  hps_gpu_ctx_sync(ctx);
  auto r = host(dr, keys.size());
  float *w = nullptr, *s0 = nullptr;
  cudaMalloc(&w, kCaps[t] * kDim * 4);
  cudaMalloc(&s0, kCaps[t] * kDim * 4);
  hps_gpu_table_export(tb, t, 0, kCaps[t], w, s0, nullptr);
  hps_gpu_ctx_sync(ctx);
  auto hw = host(w, kCaps[t] * kDim), hs = host(s0, kCaps[t] * kDim);
  std::vector<float> out;
  for (uint64_t row : r)
    for (uint32_t j = 0; j < kDim; ++j) {
      out.push_back(row == ~0ull ? -1.f : hw[row * kDim + j]);
      out.push_back(row == ~0ull ? -1.f : hs[row * kDim + j]);
    }
  cudaFree(dk);
  cudaFree(dr);
  cudaFree(w);
  cudaFree(s0);
  return out;
}

std::vector<uint64_t> batch(std::mt19937_64& rng, const std::vector<std::vector<uint64_t>>& pools, uint32_t samples) {
  std::vector<uint64_t> k;
  for (uint32_t b = 0; b < samples * kS; ++b) {
    const auto& p = pools[kSlots[b % kS]];
    k.push_back(p[rng() % (rng() % 3 == 0 ? 3 : p.size())]);  // hot keys too (long segments)
  }
  return k;
}
}  // namespace

int main() {
  // the loopback ranks of the peer transport spin-wait on each other inside one process: every
  // module is loaded up front (a lazy load could wait for the device while a peer spins)
  setenv("CUDA_MODULE_LOADING", "EAGER", 1);
  std::mt19937_64 rng(42);
  std::vector<std::vector<uint64_t>> pools(2);
  for (int t = 0; t < 2; ++t)
    for (uint64_t i = 0; i < kCaps[t]; ++i) pools[t].push_back(rng());
  std::vector<float> dout(2 * kB * kS * kDim);
  std::normal_distribution<float> nd;
  const hps_opt_params p = adagrad();

  // ---- 1. NCCL world of one ----
  {
    hps_gpu_ctx ctx = nullptr;
    OK(hps_gpu_ctx_create(0, nullptr, &ctx));
    uint8_t id[HPS_NCCL_ID_BYTES];
    OK(hps_gpu_nccl_unique_id(id));
    OK(hps_gpu_ctx_comm_init(ctx, id, 0, 1));
    hps_gpu_table plain = make_table(ctx, kB * kS), shard = make_table(ctx, kB * kS);
    REQUIRE(plain && shard);
    for (uint32_t t = 0; t < 2; ++t) {
      uint64_t* dk = dev(pools[t]);
      OK(hps_gpu_table_insert(plain, t, dk, pools[t].size(), nullptr, nullptr));
      OK(hps_gpu_table_insert(shard, t, dk, pools[t].size(), nullptr, nullptr));
      OK(hps_gpu_ctx_sync(ctx));
      cudaFree(dk);
    }
    hps_dist_config dc{kS, kSlots, kDim, kB * kS, kB * kS, 0.f};
    hps_gpu_dist d = nullptr;
    OK(hps_gpu_dist_create(ctx, shard, &dc, &d));
    uint64_t cap = 0;
    OK(hps_gpu_dist_capacity(d, &cap));
    REQUIRE(cap == kB * kS);
    float *o1 = nullptr, *o2 = nullptr, *dd = nullptr;
    cudaMalloc(&o1, kB * kS * kDim * 4);
    cudaMalloc(&o2, kB * kS * kDim * 4);
    for (int step = 0; step < 3; ++step) {
      auto keys = batch(rng, pools, kB);
      uint64_t* dk = dev(keys);
      for (auto& x : dout) x = nd(rng);
      dd = dev(std::vector<float>(dout.begin(), dout.begin() + kB * kS * kDim));
      OK(hps_gpu_lookup_pooled(plain, dk, nullptr, kB, HPS_COMBINER_SUM, o1, HPS_LOOKUP_TRAIN));
      OK(hps_gpu_dist_forward(d, dk, nullptr, kB, keys.size(), HPS_COMBINER_SUM, o2, HPS_LOOKUP_TRAIN));
      OK(hps_gpu_ctx_sync(ctx));
      REQUIRE(host(o1, kB * kS * kDim) == host(o2, kB * kS * kDim));
      OK(hps_gpu_backward_update(plain, dd, &p));
      OK(hps_gpu_dist_backward(d, dd, &p));
      OK(hps_gpu_ctx_sync(ctx));
      cudaFree(dk);
      cudaFree(dd);
    }
    for (uint32_t t = 0; t < 2; ++t) REQUIRE(rows_of(ctx, plain, t, pools[t]) == rows_of(ctx, shard, t, pools[t]));
    cudaFree(o1);
    cudaFree(o2);
    OK(hps_gpu_dist_destroy(d));
    OK(hps_gpu_table_destroy(plain));
    OK(hps_gpu_table_destroy(shard));
    OK(hps_gpu_ctx_destroy(ctx));
  }

  // ---- 2. loopback world of two, one thread per rank (all-to-alls as copies, then the
  //         peer-memory transport: the kernels load/store each other's regions) ----
  for (int transport : {HPS_DIST_NCCL, HPS_DIST_PEER}) {
    constexpr uint32_t G = 2;
    hps_gpu_ctx single_ctx = nullptr, ctxs[G] = {};
    OK(hps_gpu_ctx_create(0, nullptr, &single_ctx));
    cudaStream_t streams[G];
    for (uint32_t r = 0; r < G; ++r) {
      cudaStreamCreateWithFlags(&streams[r], cudaStreamNonBlocking);
      OK(hps_gpu_ctx_create(0, streams[r], &ctxs[r]));
    }
    const uint64_t mk = kB * kS, cap = std::min<uint64_t>(mk, uint64_t((1.25 * mk + G - 1) / G) + 1024);
    hps_gpu_table single = make_table(single_ctx, G * mk), shards[G];
    for (uint32_t r = 0; r < G; ++r) REQUIRE((shards[r] = make_table(ctxs[r], G * cap)) != nullptr);
    for (uint32_t t = 0; t < 2; ++t) {
      uint64_t* dk = dev(pools[t]);
      OK(hps_gpu_table_insert(single, t, dk, pools[t].size(), nullptr, nullptr));
      OK(hps_gpu_ctx_sync(single_ctx));
      cudaFree(dk);
      for (uint32_t r = 0; r < G; ++r) {
        std::vector<uint64_t> mine;
        for (uint64_t k : pools[t])
          if (hps::partition_of(k, G) == r) mine.push_back(k);
        uint64_t* dm = dev(mine);
        OK(hps_gpu_table_insert(shards[r], t, dm, mine.size(), nullptr, nullptr));
        OK(hps_gpu_ctx_sync(ctxs[r]));
        cudaFree(dm);
      }
    }
    hps_dist_config dc{kS, kSlots, kDim, mk, kB * kS, 0.f};
    hps_gpu_dist ds[G];
    OK(hps_gpu_dist_create_loopback(ctxs, shards, &dc, G, ds));
    for (uint32_t r = 0; r < G; ++r) OK(hps_gpu_dist_set_transport(ds[r], transport));
    float* os = nullptr;
    cudaMalloc(&os, G * kB * kS * kDim * 4);
    float* ol[G];
    for (uint32_t r = 0; r < G; ++r) cudaMalloc(&ol[r], kB * kS * kDim * 4);
    for (int step = 0; step < 3; ++step) {
      auto keys = batch(rng, pools, G * kB);
      for (auto& x : dout) x = nd(rng);
      uint64_t* dk = dev(keys);
      float* dd = dev(dout);
      OK(hps_gpu_lookup_pooled(single, dk, nullptr, G * kB, HPS_COMBINER_SUM, os, HPS_LOOKUP_TRAIN));
      OK(hps_gpu_backward_update(single, dd, &p));
      OK(hps_gpu_ctx_sync(single_ctx));
      int rc[G] = {};
      auto run = [&](uint32_t r, bool fwd) {
        rc[r] = fwd ? hps_gpu_dist_forward(ds[r], dk + r * kB * kS, nullptr, kB, kB * kS, HPS_COMBINER_SUM, ol[r],
                                           HPS_LOOKUP_TRAIN)
                    : hps_gpu_dist_backward(ds[r], dd + r * kB * kS * kDim, &p);
        if (!rc[r]) rc[r] = hps_gpu_ctx_sync(ctxs[r]);
      };
      for (bool fwd : {true, false}) {
        std::thread t0(run, 0, fwd), t1(run, 1, fwd);
        t0.join();
        t1.join();
        REQUIRE(rc[0] == 0 && rc[1] == 0);
        if (fwd) {
          auto ref = host(os, G * kB * kS * kDim);
          for (uint32_t r = 0; r < G; ++r) {
            auto got = host(ol[r], kB * kS * kDim);
            REQUIRE(std::memcmp(got.data(), ref.data() + r * kB * kS * kDim, got.size() * 4) == 0);
          }
        }
      }
      cudaFree(dk);
      cudaFree(dd);
    }
    for (uint32_t t = 0; t < 2; ++t)
      for (uint32_t r = 0; r < G; ++r) {
        std::vector<uint64_t> mine;
        for (uint64_t k : pools[t])
          if (hps::partition_of(k, G) == r) mine.push_back(k);
        REQUIRE(rows_of(single_ctx, single, t, mine) == rows_of(ctxs[r], shards[r], t, mine));
      }
    for (uint32_t r = 0; r < G; ++r) {
      OK(hps_gpu_dist_destroy(ds[r]));
      OK(hps_gpu_table_destroy(shards[r]));
      OK(hps_gpu_ctx_destroy(ctxs[r]));
      cudaFree(ol[r]);
    }
    cudaFree(os);
    OK(hps_gpu_table_destroy(single));
    OK(hps_gpu_ctx_destroy(single_ctx));
  }
  std::printf("hps_gpu_dist C-ABI test passed\n");
  return 0;
}
