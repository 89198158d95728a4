// table_internal.cuh — table-group state shared by table.cu (index + forward) and
// backward.cu (dedup + reduction + optimizers).
#pragma once

#include <vector>

#include "common.cuh"

namespace hpsg {

constexpr uint32_t kChunk = 32;            // blocked reduction width
constexpr uint32_t kNoScr = 0xffffffffu;   // occurrence of an absent key: no gradient
constexpr uint64_t kScrEmpty = 0x00000000ffffffffull;  // dedup slot {row = ~0, count = 0}
constexpr uint32_t kSortSmemMax = 4096;    // long segments up to this length sort in smem

// Per-batch dedup table: open addressing on the global row id, {row:u32 | count:u32}.
// Filled by the training forward (arrival rank = atomic count), drained and reset by
// the backward's compaction scan, so it is empty again at the end of every step.
__device__ __forceinline__ uint32_t scr_home(uint32_t row, int bits) {
  return static_cast<uint32_t>((uint64_t(row) * 0x9e3779b97f4a7c15ull) >> (64 - bits));
}

__device__ __forceinline__ void scr_insert(uint64_t* scr, int bits, uint32_t row, uint32_t* slot, uint32_t* rank) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t s = scr_home(row, bits);
  while (true) {
    const unsigned long long old =
        atomicCAS(reinterpret_cast<unsigned long long*>(scr + s), kScrEmpty, (1ull << 32) | row);
    if (old == kScrEmpty) {
      *slot = s;
      *rank = 0;
      return;
    }
    if (static_cast<uint32_t>(old) == row) {
      const unsigned long long prev = atomicAdd(reinterpret_cast<unsigned long long*>(scr + s), 1ull << 32);
      *slot = s;
      *rank = static_cast<uint32_t>(prev >> 32);
      return;
    }
    s = (s + 1) & mask;
  }
}

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
  uint64_t* ws_scr = nullptr;  // dedup table [2^scr_bits]
  int scr_bits = 0;
  uint32_t* ws_slot_u = nullptr;    // dedup slot -> unique id
  uint32_t* ws_occ_scr = nullptr;   // occurrence -> dedup slot (kNoScr: absent key)
  uint32_t* ws_occ_rank = nullptr;  // occurrence -> arrival rank among its key's occurrences
  uint32_t* ws_occ_bag = nullptr;   // occurrence -> bag (multi-hot)
  uint32_t* ws_bag_len = nullptr;   // bag lengths (multi-hot mean)
  uint32_t* ws_occ_list = nullptr;  // occurrences grouped by unique key
  uint32_t *ws_seg_row = nullptr, *ws_seg_len = nullptr, *ws_seg_off = nullptr;
  uint32_t *ws_long_seg = nullptr, *ws_long_base = nullptr, *ws_task_long = nullptr;
  float* ws_partial = nullptr;      // chunk partials of long segments
  uint64_t max_chunks = 0;
  uint32_t* ws_bitmap = nullptr;    // per-CTA occurrence bitmaps for very long segments
  uint64_t bitmap_words = 0;
  int long_ctas = 0;
  uint64_t* ws_counts = nullptr;    // [0]=N occurrences [1]=U [2]=valid occurrences [3]=packed (n_long<<32 | chunks) [4]=long ticket
  uint64_t* ws_scan = nullptr;      // look-back words of the dedup scan (+ ticket)
  size_t scan_words = 0;
  uint32_t* ws_abort = nullptr;
  uint64_t* ws_keys_stage = nullptr;
  uint32_t* ws_offsets_stage = nullptr;
  uint32_t* ws_sort_a = nullptr;   // last_unique() scratch (not on the hot path)
  uint32_t* ws_sort_b = nullptr;
  // last training lookup
  bool have_train = false, last_multi = false, scr_dirty = false;
  int last_combiner = 0;
  uint64_t last_n_keys_host = 0;  // exact when known on the host, else max_keys
};
