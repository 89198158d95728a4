// placement.cpp — host-side placement planners, C++ behind the C-ABI.
//
// These decide which GPU owns what before any kernel runs:
//   plan_localized   LPT: slots in descending byte size (ties: lower slot id first), each
//                    to the device with the most remaining budget (ties: lower device id);
//                    Infeasible if a slot fits nowhere
//   plan_distributed device = key_hash(key) mod G (hash.hpp:52-54);
//                    Infeasible unless total/G <= min budget * 1.05
//   plan_hybrid      hot set = top keys by (count desc, key asc) filling the per-device hot
//                    budget, replicated; cold keys sharded as distributed
//   estimate_comm    all-to-all volume model
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include <hps/hash.hpp>
#include "hps_gpu.h"

extern "C" {

int hps_plan_localized(const hps_slot_spec* slots, uint32_t n_slots, const uint64_t* budget, uint32_t n_devices,
                       uint32_t* slot_device_out) {
  if ((!slots && n_slots) || !budget || n_devices == 0 || (!slot_device_out && n_slots)) return HPS_GPU_E_INVALID_ARGUMENT;
  std::vector<uint32_t> order(n_slots);
  std::iota(order.begin(), order.end(), 0u);
  auto bytes = [&](uint32_t s) { return slots[s].vocab_size * uint64_t(slots[s].dim) * 4ull; };
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return bytes(a) > bytes(b); });
  std::vector<uint64_t> remaining(budget, budget + n_devices);
  for (uint32_t s : order) {
    uint32_t best = 0;
    for (uint32_t d = 1; d < n_devices; ++d)
      if (remaining[d] > remaining[best]) best = d;
    if (bytes(s) > remaining[best]) return HPS_GPU_E_INFEASIBLE;
    remaining[best] -= bytes(s);
    slot_device_out[s] = best;
  }
  return HPS_GPU_OK;
}

int hps_plan_distributed(const hps_slot_spec* slots, uint32_t n_slots, const uint64_t* budget, uint32_t n_devices) {
  if ((!slots && n_slots) || !budget || n_devices == 0) return HPS_GPU_E_INVALID_ARGUMENT;
  long double total = 0;
  for (uint32_t s = 0; s < n_slots; ++s) total += static_cast<long double>(slots[s].vocab_size) * slots[s].dim * 4.0L;
  const uint64_t min_budget = *std::min_element(budget, budget + n_devices);
  return total / n_devices <= static_cast<long double>(min_budget) * 1.05L ? HPS_GPU_OK : HPS_GPU_E_INFEASIBLE;
}

// Host mirrors of the shared hash.hpp definitions (for ABI-level tests of the header).
uint64_t hps_key_hash_host(uint64_t key) { return hps::key_hash(key); }
uint64_t hps_fastmod_u64_host(uint64_t a, uint64_t d) { return hps::FastMod64(d).mod(a); }

void hps_shard_of(const uint64_t* keys, uint64_t n, uint32_t n_devices, uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = hps::partition_of(keys[i], n_devices);
}

int hps_plan_hybrid(const uint64_t* keys, const uint64_t* counts, uint64_t n_keys, uint32_t dim,
                    uint64_t hot_budget_bytes, uint64_t* hot_keys_out, uint64_t* n_hot_out) {
  if ((!keys || !counts) && n_keys) return HPS_GPU_E_INVALID_ARGUMENT;
  if (!n_hot_out || dim == 0) return HPS_GPU_E_INVALID_ARGUMENT;
  const uint64_t row_bytes = uint64_t(dim) * 4;
  const uint64_t k = std::min<uint64_t>(n_keys, hot_budget_bytes / row_bytes);
  std::vector<uint64_t> idx(n_keys);
  std::iota(idx.begin(), idx.end(), 0ull);
  auto better = [&](uint64_t a, uint64_t b) {
    return counts[a] != counts[b] ? counts[a] > counts[b] : keys[a] < keys[b];
  };
  if (k < n_keys) std::nth_element(idx.begin(), idx.begin() + k, idx.end(), better);
  std::sort(idx.begin(), idx.begin() + k, better);
  if (hot_keys_out)
    for (uint64_t i = 0; i < k; ++i) hot_keys_out[i] = keys[idx[i]];
  *n_hot_out = k;
  return HPS_GPU_OK;
}

int hps_estimate_comm(int strategy, uint64_t batch, const hps_slot_spec* slots, uint32_t n_slots, uint32_t n_devices,
                      const double* p_cold, double* fwd_bytes, double* bwd_bytes) {
  if ((!slots && n_slots) || n_devices == 0 || !fwd_bytes || !bwd_bytes) return HPS_GPU_E_INVALID_ARGUMENT;
  const long double share = static_cast<long double>(n_devices - 1) / n_devices;
  long double v = 0;
  if (strategy == HPS_PLAN_LOCALIZED || strategy == HPS_PLAN_DISTRIBUTED) {
    for (uint32_t s = 0; s < n_slots; ++s) v += static_cast<long double>(slots[s].dim) * 4.0L;
    v *= static_cast<long double>(batch) * share;
  } else if (strategy == HPS_PLAN_HYBRID) {
    if (!p_cold) return HPS_GPU_E_INVALID_ARGUMENT;
    for (uint32_t s = 0; s < n_slots; ++s)
      v += static_cast<long double>(slots[s].hotness) * p_cold[s] * slots[s].dim * 4.0L;
    v *= static_cast<long double>(batch) * share;
  } else {
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  *fwd_bytes = static_cast<double>(v);
  *bwd_bytes = static_cast<double>(v);  // symmetric model
  return HPS_GPU_OK;
}

}  // extern "C"
