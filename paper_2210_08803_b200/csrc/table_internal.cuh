// table_internal.cuh — table-group state shared by table.cu (index + forward) and
// backward.cu (dedup + reduction + optimizers).
#pragma once

#include <vector>

#include "common.cuh"
#include "primitives.cuh"

namespace hpsg {

constexpr uint32_t kChunk = 32;  // blocked reduction width

// Zeroed-per-training-lookup region (u32 words), DESIGN.md §3 K4:
//   [0,2)  u64 short-segment allocator: (segments << 32) | occurrences
//   [2]    long segments   [3] tree nodes allocated above level 1
//   [4,6)  u64 long occurrences (place-scan total)   [6,8) u64 level-1 chunks of long segments
//   [8,10) u64 long-segment allocator: (segments << 32) | occurrences (word 9 = the count)
//   then   place-scan look-back (u64 x tiles + ticket) and the radix-sort words of the
//          long-occurrence sort.
constexpr uint32_t kLongFlag = 0x80000000u;  // batch-table value after allocation: long segment id
constexpr uint32_t kBtEmpty = 0xffffffffu;   // batch-table key of a free entry
inline uint64_t bwd_max_long(uint64_t max_keys) { return max_keys / (kChunk + 1) + 2; }
inline int bwd_long_passes(uint64_t max_keys) {
  const uint64_t m = bwd_max_long(max_keys);
  int b = 0;
  while (b < 32 && (m >> b)) ++b;
  return b <= 8 ? 1 : (b + 7) / 8;
}
struct BwdZero {
  size_t place, sort, coop, total;
};
inline BwdZero bwd_zero_layout(uint64_t nk) {
  BwdZero z;
  z.place = 10;
  z.sort = z.place + 2 * (scan_tiles(nk) + 1);
  z.coop = z.sort + ((sort_ws_words(nk, bwd_long_passes(nk)) + 1) & ~size_t(1));  // 3 barriers + per-CTA counts
  z.total = z.coop + 4 + 160;
  return z;
}
// Level-1 chunks of segments longer than kChunk: sum ceil(len/32) <= N/32 + N/33.
inline uint64_t bwd_max_chunks(uint64_t max_keys) { return max_keys / kChunk + max_keys / (kChunk + 1) + 4; }
// Tree nodes above level 1 over all long segments: sum_j (ceil(m_j/32) + ceil(m_j/1024) + ...)
// <= total_chunks/31 + (levels <= 5) per segment.
inline uint64_t bwd_max_nodes(uint64_t max_keys) { return bwd_max_chunks(max_keys) / 31 + 5 * bwd_max_long(max_keys) + 8; }

}  // namespace hpsg

struct hps_gpu_table_s;
namespace hpsg {
int launch_dedup(hps_gpu_table_s* t, cudaStream_t st);  // backward.cu: K4a-K4d (on t->side)
int choose_dedup(bool* flat_out);  // backward.cu: persistent k_dedup if one CTA fits every SM, else flat
// table.cu: hps_gpu_table_read_through + the source tier of every key (src_out[i]: 0 cache,
// 1 table, 3 default vector; may be NULL)
int table_read_through(hps_gpu_table_s* t, uint32_t table, const uint64_t* keys, const float* found_vecs,
                       const uint32_t* found_idx, const uint32_t* missing_idx, const uint64_t* counts, uint64_t n,
                       float* out, uint64_t* miss_keys, float* miss_vecs, uint8_t* miss_absent, uint8_t* src_out, bool hits_in_place = false);
cudaError_t trace_attach_table(TraceRec* p);  // table.cu's copy of the trace pointer
}

// Per-batch state of a table group: the training record, the dedup's products and the
// backward's scratch, plus the side stream their kernels run on. A table holds one slot by
// default; hps_gpu_table_set_pipeline(depth) adds slots so the record + dedup of batch i+1
// (hps_gpu_table_prefetch) can run while batch i's pooling and backward use another slot.
// The table's own fields of this type are the CURRENT slot (the one lookups and backwards
// use); the others are parked in hps_gpu_table_s::parked and swapped in by use_slot().
struct BatchSlot {
  uint32_t* ws_rows_a = nullptr;  // occurrence -> global row (row_absent: key absent)
  uint32_t* ws_rank = nullptr;    // occurrence -> arrival rank within its row
  // Batch table: open addressing {row, value} over next_pow2(8 N) entries (L2-resident),
  // value = UINT32_MAX + occurrences of the row in the batch, then its segment locator;
  // every entry the backward touches is reset to {kBtEmpty, UINT32_MAX}.
  uint2* ws_bt = nullptr;
  uint32_t* ws_occ_ent = nullptr;   // occurrence -> batch-table entry of its row
  uint32_t* ws_lead = nullptr;      // k_dedup: leaders (rank-0 occurrences), per-CTA lists
  uint32_t* ws_long_ent = nullptr;  // long segment -> batch-table entry
  uint32_t* ws_occ_bag = nullptr;   // occurrence -> bag (multi-hot)
  uint32_t* ws_bag_len = nullptr;   // bag lengths (multi-hot mean)
  uint4* ws_short_rec = nullptr;    // short segments {row, first, len, 0}, CSR over ws_short_bag
  uint32_t* ws_short_bag = nullptr; // bags of the short segments' occurrences
  uint32_t *ws_long_row = nullptr, *ws_long_len = nullptr, *ws_long_start = nullptr;
  uint32_t *ws_lkey_a = nullptr, *ws_lval_a = nullptr, *ws_lkey_b = nullptr, *ws_lval_b = nullptr;
  uint32_t* ws_long_base = nullptr;  // long segment -> first level-1 chunk
  uint32_t* ws_task_long = nullptr; // level-1 chunk -> long segment id
  float* ws_partial = nullptr;      // level-1 chunk partials of long segments
  float* ws_partial2 = nullptr;     // tree nodes above level 1 [max_nodes x dim]
  uint32_t* ws_long_hbase = nullptr;  // long segment -> its first node in ws_partial2
  uint32_t* ws_node_cnt = nullptr;    // arrivals per node; zero at rest (reset by the completing warp)
  uint64_t* ws_counts = nullptr;    // [0]=N occurrences [1]=U segments [5] unconsumed record [6] its size
  uint32_t* ws_zero = nullptr;      // bwd_zero_layout(): allocators + look-back words, zeroed per training lookup
  uint64_t* ws_keys_stage = nullptr;
  uint32_t* ws_offsets_stage = nullptr;
  // insert scratch for batches up to max_keys (insert-on-miss runs inside the step)
  uint64_t* ws_ins_slot = nullptr;
  uint32_t* ws_ins_pos = nullptr;
  uint8_t* ws_ins_flag = nullptr;
  uint64_t* ws_ins_scan = nullptr;  // insert: [abort flag, new-key count, scan status, ticket] (one memset)
  // last training lookup recorded in this slot
  bool have_train = false, last_multi = false;
  bool have_unique = false;   // the segment lists describe the last backward (last_unique)
  // The backward's dedup runs on a side stream, forked after the training probe and joined
  // by backward_update (table.cu record_and_fork).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_bwd = nullptr, ev_join2 = nullptr;  // backward: long reduce on the side stream
  cudaEvent_t ev_done = nullptr;  // the whole dedup (long-segment part included) is done
  cudaEvent_t ev_pre = nullptr;   // prefetch: the table stream's position it is ordered after
  cudaEvent_t ev_probe = nullptr; // prefetch: the record (probe) is complete
  bool dedup_pending = false;
  bool dedup_deferred = false;  // no_fork: the dedup runs at backward_update
  bool prefetched = false;      // the record + dedup came from hps_gpu_table_prefetch
  bool pre_keys_host = false;   // ... with HPS_LOOKUP_KEYS_HOST (offsets staged in ws_offsets_stage)
  unsigned long long pre_capture = 0;  // stream-capture id the prefetch was enqueued under (0: none)
  int last_combiner = 0;
  uint32_t pre_n_bags = 0;
  uint64_t last_n_keys_host = 0;  // exact when known on the host, else max_keys
};

struct hps_gpu_table_s : BatchSlot {
  hps_gpu_ctx ctx = nullptr;
  uint32_t n_tables = 0, dim = 0, n_slots = 0;
  uint32_t dim_io = 0;      // the caller's dim; `dim` = padded_dim(dim_io) is the storage stride
  float* ws_io = nullptr;   // dim_io != dim: [max_bags x dim] staging of pooled outputs / gradients
  float* ws_dscale = nullptr;  // mean combiner: [max_bags x dim] gradient rows / bag length (backward_impl)
  int optimizer = 0, n_state = 0;
  uint64_t seed = 0;
  float a0 = 0.f;
  std::vector<uint64_t> row_cap, row_base, slot_cap, slot_base;
  std::vector<hpsg::TableDev> h_tables;
  uint64_t total_rows = 0, total_slots = 0;
  uint32_t row_absent = 0;  // occurrence row of an absent key (= total_rows): no gradient
  int sort_bits = 0;        // bits of a global row id (incl. row_absent)
  uint64_t max_keys = 0, max_bags = 0;
  // device state
  hpsg::TableDev* d_tables = nullptr;
  hpsg::Slot* d_slots = nullptr;
  float *d_w = nullptr, *d_s0 = nullptr, *d_s1 = nullptr;  // (d_w unused by F16 tables)
  bool f16 = false;              // HPS_DTYPE_F16: rows in d_wh as binary16 (inference table)
  uint16_t* d_wh = nullptr;
  uint64_t* d_row_keys = nullptr;
  uint64_t* d_nrows = nullptr;
  float* d_defaults = nullptr;
  uint32_t* d_slot_table = nullptr;
  uint64_t bt_mask = 0;
  uint64_t max_chunks = 0, max_long = 0;
  size_t zero_words = 0;
  // batch slots: `cur` is the one held in the BatchSlot base; parked[k] holds slot k otherwise
  std::vector<BatchSlot> parked;  // size = pipeline depth (entry `cur` is stale while current)
  uint32_t cur = 0;

  bool flat_dedup = false;  // the three-kernel dedup (choose_dedup at create)
  bool no_fork = false;         // HPS_GPU_NO_FORK=1: everything on the main stream (A/B measurement)
  bool no_tma = false;  // HPS_GPU_NO_TMA=1: use the register-staged gather (A/B measurement)
};

namespace hpsg {
// Make batch slot k the table's current slot (parks the current one).
inline void use_slot(hps_gpu_table_s* t, uint32_t k) {
  if (k == t->cur) return;
  t->parked[t->cur] = static_cast<BatchSlot&>(*t);
  static_cast<BatchSlot&>(*t) = t->parked[k];
  t->cur = k;
}
// Capture id of a stream's active capture (0: not capturing).
inline unsigned long long capture_id(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &cs, &id) != cudaSuccess || cs != cudaStreamCaptureStatusActive) return 0;
  return id;
}
// Stream `s` waits for `ev`, recorded under capture `rec_capture` (0: eagerly). Same context:
// a plain wait. An eager record seen from a capture: an external-event wait node. A record
// made inside another graph: no wait — that graph ends joined, and graphs of one stream run
// in order.
inline cudaError_t wait_recorded(cudaStream_t s, cudaEvent_t ev, unsigned long long rec_capture) {
  const unsigned long long cid = capture_id(s);
  if (cid == rec_capture) return cudaStreamWaitEvent(s, ev, 0);
  if (cid != 0 && rec_capture == 0) return cudaStreamWaitEvent(s, ev, cudaEventWaitExternal);
  return cudaSuccess;
}
}  // namespace hpsg
