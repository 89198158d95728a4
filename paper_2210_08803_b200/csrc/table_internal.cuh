// table_internal.cuh — table-group state shared by table.cu (index + forward) and
// backward.cu (dedup + reduction + optimizers).
#pragma once

#include <vector>

#include "common.cuh"
#include "primitives.cuh"

namespace hpsg {

constexpr uint32_t kChunk = 32;  // blocked reduction width

// Zeroed-per-backward region: [radix sort words][pad][segment-scan status (u64) x tiles]
// [scan ticket][long packed counter][piece counter][item ticket][spare x2] — one memset.
inline size_t bwd_sort_words(uint64_t max_keys, int passes) { return (sort_ws_words(max_keys, passes) + 1) & ~size_t(1); }
inline size_t bwd_zero_words(uint64_t max_keys, int passes) {
  return bwd_sort_words(max_keys, passes) + 2 * (scan_tiles(max_keys) + 6);
}
// Level-1 chunks of segments longer than kChunk: sum ceil(len/32) <= N/32 + N/33.
inline uint64_t bwd_max_chunks(uint64_t max_keys) { return max_keys / kChunk + max_keys / (kChunk + 1) + 4; }
inline uint64_t bwd_max_long(uint64_t max_keys) { return max_keys / (kChunk + 1) + 2; }
// Tree nodes above level 1 over all long segments: sum_j (ceil(m_j/32) + ceil(m_j/1024) + ...)
// <= total_chunks/31 + (levels <= 5) per segment.
inline uint64_t bwd_max_nodes(uint64_t max_keys) { return bwd_max_chunks(max_keys) / 31 + 5 * bwd_max_long(max_keys) + 8; }

}  // namespace hpsg

struct hps_gpu_table_s {
  hps_gpu_ctx ctx = nullptr;
  uint32_t n_tables = 0, dim = 0, n_slots = 0;
  int optimizer = 0, n_state = 0;
  uint64_t seed = 0;
  float a0 = 0.f;
  std::vector<uint64_t> row_cap, row_base, slot_cap, slot_base;
  std::vector<hpsg::TableDev> h_tables;
  uint64_t total_rows = 0, total_slots = 0;
  uint32_t row_absent = 0;  // sort key of an absent-key occurrence (= total_rows, sorts last)
  int sort_bits = 0;        // bits of a global row id (incl. row_absent)
  uint64_t max_keys = 0, max_bags = 0;
  // device state
  hpsg::TableDev* d_tables = nullptr;
  hpsg::Slot* d_slots = nullptr;
  float *d_w = nullptr, *d_s0 = nullptr, *d_s1 = nullptr;
  uint64_t* d_row_keys = nullptr;
  uint64_t* d_nrows = nullptr;
  float* d_defaults = nullptr;
  uint32_t* d_slot_table = nullptr;
  // per-batch workspaces (sized at create, never reallocated)
  uint32_t *ws_rows_a = nullptr, *ws_rows_b = nullptr;  // occurrence rows / sort ping-pong
  uint32_t *ws_bags_a = nullptr, *ws_bags_b = nullptr;  // sort payload: bag of the occurrence
  uint32_t* ws_occ_bag = nullptr;   // occurrence -> bag (multi-hot)
  uint32_t* ws_bag_len = nullptr;   // bag lengths (multi-hot mean)
  uint32_t *ws_seg_start = nullptr, *ws_seg_end = nullptr;  // unique-row segments of the sorted list
  uint32_t *ws_long_seg = nullptr, *ws_long_base = nullptr;  // long segments: id -> segment, first chunk
  uint32_t* ws_task_long = nullptr; // level-1 chunk -> long segment id
  float* ws_partial = nullptr;      // level-1 chunk partials of long segments
  float* ws_partial2 = nullptr;     // tree nodes above level 1 [max_nodes x dim]
  uint32_t* ws_long_hbase = nullptr;  // long segment -> its first node in ws_partial2
  uint32_t* ws_node_cnt = nullptr;    // arrivals per node; zero at rest (reset by the completing warp)
  uint64_t max_chunks = 0, max_long = 0;
  uint64_t* ws_counts = nullptr;    // [0]=N occurrences [1]=U segments
  uint32_t* ws_zero = nullptr;      // look-back words + tickets + long counters, zeroed per backward
  size_t zero_words = 0;
  uint32_t* ws_abort = nullptr;
  uint64_t* ws_keys_stage = nullptr;
  // insert scratch for batches up to max_keys (insert-on-miss runs inside the step)
  uint64_t* ws_ins_slot = nullptr;
  uint32_t* ws_ins_pos = nullptr;
  uint8_t* ws_ins_flag = nullptr;
  uint64_t* ws_ins_scan = nullptr;
  uint32_t* ws_offsets_stage = nullptr;
  // last training lookup
  bool have_train = false, last_multi = false, sorted_in_b = false;
  bool no_tma = false;  // HPS_GPU_NO_TMA=1: use the register-staged gather (A/B measurement)
  int last_combiner = 0;
  uint64_t last_n_keys_host = 0;  // exact when known on the host, else max_keys
};
