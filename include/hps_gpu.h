/* hps_gpu.h — C-ABI of the B200 sparse-embedding hot path (sm_100a only).
 *
 * This is the drop-in boundary. It replaces, for the embedding
 * path, the reference's operator API pattern (proj/include/hps/kernels.hpp:33-66:
 * free functions over raw pointers + counts, caller-owned buffers, no exceptions
 * inside kernels, one backend chosen once) with ONE implementation: hand-written
 * CUDA kernels for sm_100a. There is no vtable, no "scalar" backend and no CPU
 * fallback: if no usable B200 is present every entry point returns
 * HPS_GPU_E_NO_DEVICE.
 *
 * Conventions
 *   - Every function returns int: 0 = OK, 1..17 = hps::ErrorCode values
 *     (proj/include/hps/error.hpp:24-42), >= 256 = device failures.
 *   - Pointer arguments are DEVICE pointers (stream-ordered on the handle's
 *     stream) unless the parameter name ends in `_host`.
 *   - Calls are asynchronous on the context's stream unless documented as
 *     "syncs". Data errors found on the device (NaN/Inf on insert -> NonFinite,
 *     row capacity exhausted -> Infeasible) are latched in a device status word
 *     and reported by the next syncing call (hps_gpu_ctx_sync).
 *   - Handles are externally synchronised: one thread/stream mutates a handle at a
 *     time; different handles are independent.
 *   - Hot calls (lookup_pooled, backward_update, cache_query, ...) never allocate,
 *     never synchronise and are capturable into a CUDA graph.
 *   - Keys are hps::EmbeddingKey (uint64, any value legal). Placement always uses
 *     hps::key_hash / hps::partition_of (proj/include/hps/hash.hpp:42-54).
 */
#ifndef HPS_GPU_H_
#define HPS_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_GPU_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------- */
enum {
  HPS_GPU_OK = 0,
  /* 1..17 mirror hps::ErrorCode (proj/include/hps/error.hpp:24-42) */
  HPS_GPU_E_INVALID_ARGUMENT = 1,
  HPS_GPU_E_BAD_MAGIC = 2,
  HPS_GPU_E_BAD_FORMAT_VERSION = 3,
  HPS_GPU_E_TRUNCATED = 4,
  HPS_GPU_E_TRAILING_BYTES = 5,
  HPS_GPU_E_DUPLICATE_KEY = 6,
  HPS_GPU_E_DIM_MISMATCH = 7,
  HPS_GPU_E_DTYPE_MISMATCH = 8,
  HPS_GPU_E_F16_RANGE = 9,
  HPS_GPU_E_NON_FINITE = 10,
  HPS_GPU_E_UNKNOWN_TABLE = 11,
  HPS_GPU_E_BAD_SHARD = 13,
  HPS_GPU_E_IO = 14,
  HPS_GPU_E_CORRUPTION = 15,
  HPS_GPU_E_INFEASIBLE = 16,
  /* device failures */
  HPS_GPU_E_CUDA = 256,
  HPS_GPU_E_OUT_OF_MEMORY = 257,
  HPS_GPU_E_NO_DEVICE = 258,
  HPS_GPU_E_NOT_CAPTURABLE = 259,
  HPS_GPU_E_NCCL = 260,            /* an NCCL call of the sharded path failed */
  HPS_GPU_E_PEER_TIMEOUT = 261     /* peer transport: a peer never signalled its phase (10 s) */
};

/* Human readable name of a status ("OK", "InvalidArgument", ..., "CudaError"). */
const char* hps_gpu_status_string(int status);
/* ABI version of the loaded library (HPS_GPU_ABI_VERSION it was built with). */
int hps_gpu_abi_version(void);
/* Last error message recorded on this thread (empty string if none). */
const char* hps_gpu_last_error_message(void);

/* ---- context: device + stream + device status word ------------------------- */
typedef struct hps_gpu_ctx_s* hps_gpu_ctx;

/* stream: a cudaStream_t (NULL = the legacy default stream). */
int hps_gpu_ctx_create(int device, void* stream, hps_gpu_ctx* out_host);
int hps_gpu_ctx_destroy(hps_gpu_ctx ctx);
int hps_gpu_ctx_set_stream(hps_gpu_ctx ctx, void* stream);
/* syncs: waits for the stream, returns and clears the latched device status. */
int hps_gpu_ctx_sync(hps_gpu_ctx ctx);

/* ---- K1: hashing / placement (proj/include/hps/hash.hpp:42-54) -------------- */
int hps_gpu_key_hash(hps_gpu_ctx ctx, const uint64_t* keys, uint64_t n, uint64_t* hashes_out);
/* out[i] = partition_of(keys[i], num_shards); num_shards == 0 -> InvalidArgument. */
int hps_gpu_partition_of(hps_gpu_ctx ctx, const uint64_t* keys, uint64_t n,
                         uint32_t num_shards, uint32_t* shard_out);
/* flag_out[0] = 1 if any of v[0..n) is NaN/Inf else 0 (kernels.hpp:41-43 semantics). */
int hps_gpu_has_non_finite_f32(hps_gpu_ctx ctx, const float* v, uint64_t n, uint32_t* flag_out);
/* The rest of the reference's kernel API (proj/include/hps/kernels.hpp:33-43) over device
 * buffers, bit-equivalent to its scalar path (kernels_scalar.cpp:25-123; golden vectors
 * from the reference's compiled code): binary16 narrowing (round to nearest even, overflow
 * -> the infinity pattern, NaN payload kept + quiet bit), exact widening, the binary16
 * NaN/Inf scan (*flag_out = 1 if any), and CRC-32C (Castagnoli) — of one buffer continuing
 * from the running value `crc` (start from 0; scratch: one device u32), or one CRC (from 0)
 * per record [offsets[r], offsets[r+1]) of `data` (the PDB log-record checksum). */
int hps_gpu_f32_to_f16(hps_gpu_ctx ctx, const float* src, uint16_t* dst, uint64_t n);
int hps_gpu_f16_to_f32(hps_gpu_ctx ctx, const uint16_t* src, float* dst, uint64_t n);
int hps_gpu_has_non_finite_f16(hps_gpu_ctx ctx, const uint16_t* v, uint64_t n, uint32_t* flag_out);
int hps_gpu_crc32c(hps_gpu_ctx ctx, uint32_t crc, const void* data, uint64_t n, uint32_t* scratch,
                   uint32_t* crc_out);
int hps_gpu_crc32c_batch(hps_gpu_ctx ctx, const void* data, const uint64_t* offsets, uint64_t n_records,
                         uint32_t* crc_out);

/* ---- embedding table group (K2..K5) ------------------------------------------
 * A table group holds n_tables independent tables (key namespaces)
 * of one dim, fp32 rows, plus one open-addressing key->row index per table and
 * the optimizer state rows. A model has n_slots slots; slot s reads table
 * slot_table[s]. A batch is n_samples x n_slots bags in sample-major order
 * (bag = sample * n_slots + slot); bag b holds keys[offsets[b] .. offsets[b+1])
 * (offsets == NULL: exactly one key per bag, keys[b]).                          */
typedef struct hps_gpu_table_s* hps_gpu_table;

enum { HPS_OPT_SGD = 0, HPS_OPT_ADAGRAD = 1, HPS_OPT_ADAM = 2 };
enum { HPS_COMBINER_SUM = 0, HPS_COMBINER_MEAN = 1 };
/* Storage dtype of table / cached rows (hps::Dtype, proj/include/hps/types.hpp:36-40). */
enum { HPS_DTYPE_F32 = 0, HPS_DTYPE_F16 = 1 };

typedef struct {
  uint32_t n_tables;
  uint32_t dim;                     /* 1..1024 (hps::kMaxDim is 4096: wider rows -> InvalidArgument). Rows
                                       are stored at round_up(dim, 4) floats; a dim that is not a
                                       multiple of 4 is served through a staging copy on the core
                                       entry points (insert/find/export/lookup/prefetch/backward), while
                                       the exchange, hybrid and read-through paths refuse it */
  const uint64_t* row_capacity_host;/* [n_tables] max rows per table */
  uint32_t n_slots;
  const uint32_t* slot_table_host;  /* [n_slots] table id of each slot */
  int optimizer;                    /* HPS_OPT_* : sizes the state rows */
  uint64_t max_batch_keys;          /* workspace sizing: keys per lookup call */
  uint64_t max_batch_bags;          /* workspace sizing: bags per lookup call */
  uint64_t init_seed;               /* row initialiser seed (see hps_gpu_init_value) */
  float adagrad_initial_accumulator;/* AdaGrad a0 (state rows start at this) */
  uint32_t dtype;                   /* HPS_DTYPE_F32 (0, default) or HPS_DTYPE_F16: binary16 rows, an
                                       inference table (insert/find/export/lookup/read-through;
                                       training calls on it -> DtypeMismatch). Insert rounds to
                                       nearest even; a row beyond binary16 range -> F16Range
                                       (latched, the call refused) — SPEC.md:78-86 */
} hps_table_config;

typedef struct {
  float lr;
  float eps;
  float beta1, beta2;               /* Adam */
  float one_minus_beta1, one_minus_beta2;
  float lr_t;                       /* Adam: lr*sqrt(1-b2^t)/(1-b1^t), computed by the caller in fp32 */
  const float* lr_t_device;         /* optional (NULL: use lr_t): device fp32 read by the kernels at
                                       run time, so one captured CUDA graph serves every Adam step */
} hps_opt_params;

int hps_gpu_table_create(hps_gpu_ctx ctx, const hps_table_config* cfg_host, hps_gpu_table* out_host);
int hps_gpu_table_destroy(hps_gpu_table tbl);
/* Default vector of a table (host array of dim floats; all-zero when never set). */
int hps_gpu_table_set_default_vector(hps_gpu_table tbl, uint32_t table, const float* vec_host);
/* syncs: rows currently held by `table`. */
int hps_gpu_table_size(hps_gpu_table tbl, uint32_t table, uint64_t* n_rows_host);

/* Insert keys into `table`. New keys get row ids in order of first occurrence in
 * keys[] (continuing from the table's row count); existing keys keep theirs.
 * rows == NULL: new rows are initialised with hps_gpu_init_value(seed,key,j);
 * otherwise rows[i*dim..] is the value of keys[i]: the FIRST occurrence of a key in
 * keys[] wins, both for a new key and for an existing row it overwrites. rows_out (may be
 * NULL) receives the row id of every key. NaN/Inf in rows -> NonFinite (latched);
 * more distinct keys than capacity -> Infeasible (latched). */
int hps_gpu_table_insert(hps_gpu_table tbl, uint32_t table, const uint64_t* keys, uint64_t n,
                         const float* rows, uint64_t* rows_out);
/* rows_out[i] = row id of keys[i] in `table`, or UINT64_MAX when absent. */
int hps_gpu_table_find(hps_gpu_table tbl, uint32_t table, const uint64_t* keys, uint64_t n,
                       uint64_t* rows_out);
/* The same lookup with another probe scheme (A/B evidence): group 1 = the
 * per-thread linear probe of hps_gpu_table_find; 2, 4, 8 = warp-cooperative probing, that
 * many lanes reading consecutive slots of an aligned window per step. Identical results. */
int hps_gpu_debug_find_variant(hps_gpu_table tbl, uint32_t table, const uint64_t* keys, uint64_t n,
                               uint64_t* rows_out, uint32_t group);
/* Copy rows [row_begin, row_begin+n) of `table` (weights, and when state != NULL the
 * optimizer state rows: state[k] for k < n_state_rows) out as fp32 [n x dim]. */
int hps_gpu_table_export(hps_gpu_table tbl, uint32_t table, uint64_t row_begin, uint64_t n,
                         float* weights_out, float* state0_out, float* state1_out);
/* Key stored at each row (inverse of the index) for rows [row_begin, row_begin+n). */
int hps_gpu_table_row_keys(hps_gpu_table tbl, uint32_t table, uint64_t row_begin, uint64_t n,
                           uint64_t* keys_out);

enum {
  HPS_LOOKUP_KEYS_HOST = 1u << 0,  /* keys/offsets are pinned HOST memory: staged H2D inside the call */
  HPS_LOOKUP_TRAIN = 1u << 1,      /* remember per-key rows/bags for the following backward_update */
  HPS_LOOKUP_INSERT = 1u << 2,     /* dynamic table: insert absent keys first (single-table groups,
                                      host-known key count); rows materialise on first touch */
  HPS_LOOKUP_PREFETCHED = 1u << 3  /* training lookup of the batch hps_gpu_table_prefetch recorded in
                                      slot HPS_LOOKUP_SLOT_OF(flags): pooling only (implies TRAIN;
                                      keys are not read; offsets must be the prefetch's, or are
                                      taken from its host staging) */
};
#define HPS_LOOKUP_SLOT(k) ((uint32_t)(k) << 16)            /* batch slot of a PREFETCHED lookup */
#define HPS_LOOKUP_SLOT_OF(flags) (((uint32_t)(flags) >> 16) & 0xffu)

/* K1+K2+K3 fused: out[bag*dim + j] = combiner over the bag's rows, fp32, keys in bag
 * order, from +0.0f; mean divides by the bag length (IEEE); an empty bag gives
 * zeros; a key absent from its table contributes the table's default vector. */
int hps_gpu_lookup_pooled(hps_gpu_table tbl, const uint64_t* keys, const uint32_t* offsets,
                          uint32_t n_samples, int combiner, float* out, uint32_t flags);

/* K4+K5: gradients of the last HPS_LOOKUP_TRAIN lookup. d_out is [n_bags x dim]; each
 * key occurrence receives d_out[bag] (sum) or d_out[bag]/len (mean); occurrences of
 * the same key are dedup'ed and reduced in canonical (occurrence) order with the
 * blocked rule of DESIGN.md §4.3; the optimizer then updates each unique row in place.
 * Absent keys (default-vector occurrences) receive no update. */
int hps_gpu_backward_update(hps_gpu_table tbl, const float* d_out, const hps_opt_params* opt_host);

/* Batch pipelining (DESIGN.md §3 "Prefetch"). A table keeps `depth` batch slots (default 1):
 * a slot holds one training record (probe), its dedup (segments) and the backward's scratch.
 * hps_gpu_table_set_pipeline allocates the slots (setup call, not hot; depth 1..4).
 * hps_gpu_table_prefetch records batch i+1 into `slot` — [insert-on-miss] + probe + dedup —
 * on the slot's own stream: ordered after everything enqueued on the table's stream before
 * the call, and concurrent with what is enqueued after it (the pooling and backward of batch
 * i in another slot). The dedup reads no weights, so only the pooling and the update remain
 * on the step's critical path. hps_gpu_lookup_pooled(... HPS_LOOKUP_PREFETCHED |
 * HPS_LOOKUP_SLOT(slot) ...) then pools from that record and backward_update consumes it.
 * Results are bit-identical to the unpipelined lookup/backward sequence (HPS_LOOKUP_INSERT:
 * rows are created in prefetch order, which must then be the batch order). Refused
 * (InvalidArgument): a slot >= depth, or the slot of a training lookup still awaiting its
 * backward. hps_gpu_table_join_prefetch makes the table's stream wait for every outstanding
 * prefetch; a stream capture that contains a prefetch must call it before the capture ends. */
int hps_gpu_table_set_pipeline(hps_gpu_table tbl, uint32_t depth);
int hps_gpu_table_prefetch(hps_gpu_table tbl, uint32_t slot, const uint64_t* keys, const uint32_t* offsets,
                           uint32_t n_samples, int combiner, uint32_t flags);
int hps_gpu_table_join_prefetch(hps_gpu_table tbl);

/* After backward_update: number of unique rows updated (device u64 at *count_out),
 * and optionally their row ids in ascending row order (unique_rows_out: exactly
 * *count_out entries are written, so a buffer of the unique count suffices). Used by
 * the dedup parity tests. */
int hps_gpu_table_last_unique(hps_gpu_table tbl, uint64_t* count_out, uint32_t* unique_rows_out);

/* Tracing (no reference counterpart): in-graph timeline of the training
 * step's kernels, %globaltimer ns. mode 1 attaches a zeroed trace buffer, 2 copies
 * 32 x {first CTA start, last warp end} (u64 pairs; start = UINT64_MAX: not run) into
 * trace_host and re-arms, 0 detaches. Ids: 0 probe, 1 pool, 2 segment alloc, 3 place,
 * 4 long-sort histogram, 5..8 long-sort passes, 9 long registration, 10 short reduce,
 * 11 long reduce, 12 counter reset, 13 counts (14, 15: end of its local / global phase). Synchronises the device; not for hot paths. */
int hps_gpu_debug_trace(int mode, uint64_t* trace_host);
/* Debug: a one-warp kernel on `stream` that stamps %globaltimer into trace slot `id` (start and
   end), marking a point in the stream's order on the hps_gpu_debug_trace timeline. */
int hps_gpu_debug_stamp(void* stream, int id);

/* Invariant check for tests: entries of the table's per-batch dedup table still in use
 * (0 whenever no training record is pending). Synchronises. */
int hps_gpu_debug_batch_table_used(hps_gpu_table tbl, uint64_t* used_host);

/* Owner side of the distributed exchange: rows of keys[i] in table tables[i] (one key per
 * "bag"; absent keys give the table's default vector). With HPS_LOOKUP_TRAIN the following
 * backward_update takes d_out = [n x dim] per-key gradients (already combiner-scaled). */
int hps_gpu_gather_rows(hps_gpu_table tbl, const uint64_t* keys, const uint32_t* tables, uint64_t n,
                        float* rows_out, uint32_t flags);

/* ---- model-parallel exchange helpers (exchange.cu) ------------------ */
typedef struct hps_gpu_xplan_s* hps_gpu_xplan;

int hps_gpu_xplan_create(hps_gpu_ctx ctx, uint64_t max_keys, uint32_t n_shards, hps_gpu_xplan* out_host);
int hps_gpu_xplan_destroy(hps_gpu_xplan plan);
/* occ_bag_out[i] = bag of occurrence i of a CSR batch. */
int hps_gpu_occurrence_bags(hps_gpu_ctx ctx, const uint32_t* offsets, uint64_t n_bags, uint32_t* occ_bag_out);
/* Stable bucketing of n occurrences by owner = partition_of(key, n_shards): send_keys /
 * send_tables grouped by owner (each group in occurrence order), perm[i] = send position
 * of occurrence i, counts[g] = occurrences for owner g (u32, device). occ_bag == NULL: one
 * key per bag. Table of occurrence i = slot_table[bag % n_slots] (slot_table on device). */
int hps_gpu_xplan_bucketize(hps_gpu_xplan plan, const uint64_t* keys, uint64_t n, const uint32_t* occ_bag,
                            uint32_t n_slots, const uint32_t* slot_table, uint64_t* send_keys,
                            uint32_t* send_tables, uint32_t* perm, uint32_t* counts);
/* out[bag] = combiner over rows[perm[i]] for the bag's occurrences (offsets == NULL: one each). */
int hps_gpu_pool_rows(hps_gpu_ctx ctx, const float* rows, const uint32_t* perm, const uint32_t* offsets,
                      uint64_t n_bags, uint32_t dim, int combiner, float* out);
/* grads_out[perm[i]] = d_out[bag(i)] (/ bag length for mean). */
int hps_gpu_scatter_grads(hps_gpu_ctx ctx, const float* d_out, const uint32_t* perm, const uint32_t* offsets,
                          uint64_t n_bags, uint32_t dim, int combiner, float* grads_out);
/* Localized slot: the bags of slots sel[0..n_sel) for every sample, as CSR (sample-major).
 * lens_ws: n_samples*n_sel u32; scan_ws: scan_tiles+1 u64 (see exchange.py). */
int hps_gpu_regroup_bags(hps_gpu_ctx ctx, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         uint32_t n_slots, const uint32_t* sel, uint32_t n_sel, uint32_t* lens_ws,
                         uint64_t* out_keys, uint32_t* out_offsets, uint64_t* scan_ws);
/* offsets_out[0..n] = exclusive scan of lens[0..n) (the owner's CSR over received bag
 * lengths). scan_ws: scan_tiles(n)+1 u64. */
int hps_gpu_lengths_to_offsets(hps_gpu_ctx ctx, const uint32_t* lens, uint64_t n, uint32_t* offsets_out,
                               uint64_t* scan_ws);
/* direction 0: dst[b*n_slots + sel[j]] = src[b*n_sel + j]; direction 1: the reverse gather. */
int hps_gpu_place_pooled(hps_gpu_ctx ctx, const float* src, const uint32_t* sel, uint32_t n_sel,
                         uint32_t n_samples, uint32_t n_slots, uint32_t dim, int direction, float* dst);

/* ---- hybrid sparse embedding ------------------------
 * Hot keys (plan_hybrid) are replicated on every rank in a "hot" table group (DP); all
 * other keys are sharded by partition_of (MP, the distributed exchange above). Per step:
 *   hps_gpu_hybrid_probe   hot-index probe of every occurrence; records the hot group's
 *                          training state (like a training lookup, no pooling) and
 *                          compacts the cold occurrences (keys, bags, cold_pos[i] = index
 *                          of occurrence i among the cold ones; count on the device)
 *   cold occurrences -> hps_gpu_xplan_bucketize (occ_bag = cold bags) -> all-to-all ->
 *                          owner hps_gpu_gather_rows -> all-to-all back
 *   hps_gpu_hybrid_pool    bag sums in occurrence order from the hot replica or the
 *                          returned cold rows (cold_rows[perm[cold_pos[i]]])
 *   hps_gpu_cold_grads     cold gradient rows in send order -> all-to-all -> owner backward
 *   hps_gpu_backward_reduce  (hot group) per-row gradient sums of this rank's batch
 *   hps_gpu_sum_partials   rank-ordered sum of every rank's partials (deterministic
 *                          all-reduce: all-to-all of row slices, sum, all-gather)
 *   hps_gpu_apply_grads    (hot group) identical optimizer step on every replica        */
int hps_gpu_hybrid_probe(hps_gpu_table hot, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         int combiner, uint64_t n_keys_host, uint32_t* cold_pos_out, uint64_t* cold_keys_out,
                         uint32_t* cold_bags_out, uint64_t* cold_count_out);
int hps_gpu_hybrid_pool(hps_gpu_table hot, const uint32_t* cold_pos, const uint32_t* perm, const float* cold_rows,
                        const uint32_t* offsets, uint64_t n_bags, int combiner, float* out);
/* grads_out[perm[c]] = d_out[bags[c]] (/ bag length from offsets for mean). */
int hps_gpu_cold_grads(hps_gpu_ctx ctx, const float* d_out, const uint32_t* bags, const uint32_t* perm,
                       const uint32_t* offsets, uint64_t n, uint32_t dim, int combiner, float* grads_out);
/* out[r] = sum over p in order of the parts with touched[p][r] (the first starts the sum). */
int hps_gpu_sum_partials(hps_gpu_ctx ctx, const float* parts, const uint32_t* touched, uint32_t n_parts, uint64_t rows,
                         uint32_t dim, float* out, uint32_t* touched_out);
/* Gradient-only backward of the last training lookup/probe: per-row sums (the canonical
 * blocked tree) into grads_out[global row x dim], touched_out[row] = 1; rows not in the
 * batch are left as they were. No optimizer step. */
int hps_gpu_backward_reduce(hps_gpu_table tbl, const float* d_out, float* grads_out, uint32_t* touched_out);
/* Optimizer step for every global row r with touched[r], gradient grads[r x dim]. */
int hps_gpu_apply_grads(hps_gpu_table tbl, const float* grads, const uint32_t* touched, const hps_opt_params* opt);

/* ---- sharded step over NCCL (sharded.cu): distributed slot placement ---------------
 * SPEC.md:470, 487-491 (partition_of placement), PAPER.md:173-177, 188 (model-parallel
 * embedding, all-to-all over NVLink). The context joins an NCCL communicator (rank 0 makes
 * the id with hps_gpu_nccl_unique_id and ships it out of band — MPI, torch.distributed, a
 * file); a hps_gpu_dist is this rank's half of every step: the requester's bucketize +
 * pack into fixed-capacity per-peer regions, one grouped all-to-all of keys + table ids,
 * the owner's gather of its shard (`shard`, a table group holding the keys with
 * partition_of(key, world) == rank of every table), rows back, pooling; the backward sends
 * per-occurrence gradients to the owners, whose ordinary backward_update applies them. No
 * host synchronisation: a whole step is capturable into one CUDA graph. Results are
 * bit-identical to one table over the concatenated global batch (rank-major order).
 * Region capacity C = min(max_keys, ceil(f * max_keys / world) + 1024) occurrences per peer
 * (hps_gpu_dist_capacity); the shard must be created with max_batch_keys and
 * max_batch_bags >= world * C. A step whose occurrences for one owner exceed C latches
 * Infeasible (its results are then unspecified). */
#define HPS_NCCL_ID_BYTES 128
int hps_gpu_nccl_unique_id(void* id_out /* HPS_NCCL_ID_BYTES */);
int hps_gpu_ctx_comm_init(hps_gpu_ctx ctx, const void* id /* HPS_NCCL_ID_BYTES */, int rank, int world);

typedef struct hps_gpu_dist_s* hps_gpu_dist;
typedef struct {
  uint32_t n_slots;
  const uint32_t* slot_table_host;  /* [n_slots] table id of each slot (table ids of the shard group) */
  uint32_t dim;
  uint64_t max_keys;                /* key occurrences per rank per step (requester side) */
  uint64_t max_bags;                /* bags per rank per step */
  float capacity_factor;            /* f above; 0 -> 1.25 */
} hps_dist_config;
int hps_gpu_dist_create(hps_gpu_ctx ctx, hps_gpu_table shard, const hps_dist_config* cfg_host, hps_gpu_dist* out_host);
int hps_gpu_dist_destroy(hps_gpu_dist dist);
int hps_gpu_dist_capacity(hps_gpu_dist dist, uint64_t* per_peer_host);
/* Forward of this rank's batch: keys in bag order, offsets == NULL for one key per bag
 * (else device CSR offsets and n_keys = offsets[n_bags], known to the caller); flags:
 * HPS_LOOKUP_TRAIN, HPS_LOOKUP_INSERT (dynamic single-table shards). out: [n_bags x dim]. */
int hps_gpu_dist_forward(hps_gpu_dist dist, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                         uint64_t n_keys, int combiner, float* out, uint32_t flags);
/* Backward of the last training forward: d_out [n_bags x dim]; every owner updates its rows. */
int hps_gpu_dist_backward(hps_gpu_dist dist, const float* d_out, const hps_opt_params* opt_host);
/* Transport of the exchanges. HPS_DIST_NCCL (default): grouped ncclSend/ncclRecv of the
 * regions. HPS_DIST_PEER: no collective calls — the requester's region kernel stores keys and
 * table ids straight into the owners' receive buffers; each owner maps every received slot to
 * the first slot of the same (table, key) in that requester's region, and the requester copies
 * only those per-destination UNIQUE rows from the owner's gathered rows (U_p rows per owner
 * cross NVLink instead of one per occurrence) and pools them locally; the gradient scatter
 * stores per-occurrence gradients into the owners' gradient regions (the owner's backward
 * needs them in canonical order: bit-identical results). NVLink peer loads/stores go through
 * CUDA-IPC mappings, exchanged once over NCCL; the
 * loopback ranks of one device use each other's memory directly). Phases are ordered by
 * per-step epochs the ranks write into each other's flag words (release/acquire at system
 * scope), so a peer-transport step is graph-capturable too. Collective: every rank sets it. */
enum { HPS_DIST_NCCL = 0, HPS_DIST_PEER = 1 };
int hps_gpu_dist_set_transport(hps_gpu_dist dist, int transport);
/* Cumulative count of unique rows this owner has served to requesters over the peer transport
 * (one per distinct (table, key) per requester region per step): the rows that crossed NVLink.
 * Synchronises the context's stream. */
int hps_gpu_dist_unique_rows(hps_gpu_dist dist, uint64_t* served_host);
/* Loopback transport (tests, single-GPU bring-up): n ranks of ONE process on one device,
 * the all-to-alls done as device copies between their buffers. Rank r's calls must run on
 * their own host thread (every all-to-all is a rendezvous of the n ranks); ctxs[r] should
 * have distinct streams. Same kernels, regions and ordering as the NCCL path. With the peer
 * transport the ranks' wait kernels spin on each other on the SAME device: a rank's host
 * thread must not call a device-synchronising API (cudaMalloc/cudaFree, a synchronous
 * memcpy, cudaDeviceSynchronize) between its forward/backward calls of one step, or it can
 * block before enqueuing the signal a peer spins on (the bounded wait then reports
 * HPS_GPU_E_PEER_TIMEOUT). Separate GPUs (one rank per device) are not affected. */
int hps_gpu_dist_create_loopback(const hps_gpu_ctx* ctxs, const hps_gpu_table* shards, const hps_dist_config* cfg_host,
                                 uint32_t n, hps_gpu_dist* outs_host);

/* ---- HPS inference cache (K6..K8), SPEC.md:112-190 ---------------------------- */
typedef struct hps_gpu_cache_s* hps_gpu_cache;

typedef struct {
  uint64_t capacity;        /* resident entries; capacity % ways == 0 */
  uint32_t ways;            /* 1..32, default 8 */
  uint64_t aging_interval;  /* accesses per set-aging epoch numerator; 0 -> 10*capacity */
  uint32_t dim;             /* 1..4096 (hps::kMaxDim); stored at round_up(dim, 4) */
  uint64_t max_batch;       /* workspace sizing: keys per call */
  uint32_t dtype;           /* HPS_DTYPE_F32 (0, default) or HPS_DTYPE_F16: rows held as IEEE binary16
                               (round-to-nearest-even on insert/refresh, exact widening on query;
                               an entry with a value beyond binary16 range is rejected: F16Range,
                               latched like NonFinite, the entry skipped) — SPEC.md:78-86 */
} hps_cache_config;

typedef struct {
  uint64_t queries, hits, misses, insertions, admissions_rejected, refresh_replacements, evictions;
} hps_cache_stats;

int hps_gpu_cache_create(hps_gpu_ctx ctx, const hps_cache_config* cfg_host, hps_gpu_cache* out_host);
int hps_gpu_cache_destroy(hps_gpu_cache cache);
/* found_vecs: [n x dim] rows of the hits, compacted in input order; found_idx /
 * missing_idx: input positions (uint32, ascending); counts[0] = n_found,
 * counts[1] = n_missing (device u64). */
int hps_gpu_cache_query(hps_gpu_cache cache, const uint64_t* keys, uint64_t n, float* found_vecs,
                        uint32_t* found_idx, uint32_t* missing_idx, uint64_t* counts);
/* SPEC.md:140-148. admitted_out: device u64 (may be NULL). NaN/Inf -> NonFinite (latched,
 * the entry is skipped). */
int hps_gpu_cache_insert(hps_gpu_cache cache, const uint64_t* keys, const float* vecs,
                         const uint64_t* versions, uint64_t n, uint64_t* admitted_out);
/* SPEC.md:149-157. replaced_out: device u64 (may be NULL). */
int hps_gpu_cache_refresh(hps_gpu_cache cache, const uint64_t* keys, const float* vecs,
                          const uint64_t* versions, uint64_t n, uint64_t* replaced_out);
/* insert with the entry count produced on the device (*count <= n_max); versions may be
 * NULL (= kBulkLoadVersion); skip[i] != 0 (may be NULL) drops entry i without an access. */
int hps_gpu_cache_insert_count(hps_gpu_cache cache, const uint64_t* keys, const float* vecs,
                               const uint64_t* versions, uint64_t n_max, const uint64_t* count,
                               const uint8_t* skip, uint64_t* admitted_out);
/* Orchestrator read-through after a cache query: out[i] (input order) =
 * the hit row, else the row of keys[i] in `table` (or its default vector). The misses are
 * listed (miss_keys, miss_vecs, miss_absent) for hps_gpu_cache_insert_count. counts =
 * the query's device counts [n_found, n_missing]. */
int hps_gpu_table_read_through(hps_gpu_table tbl, uint32_t table, const uint64_t* keys, const float* found_vecs,
                               const uint32_t* found_idx, const uint32_t* missing_idx, const uint64_t* counts,
                               uint64_t n, float* out, uint64_t* miss_keys, float* miss_vecs, uint8_t* miss_absent);
/* ---- orchestrator batch lookup (orchestrator.cu) --------------
 * The orchestrator's red data flow on one GPU: the cache (L1) in front of table `table`
 * of a table group (the lower tier; the VDB/PDB tiers are not on the GPU path).
 * lookup: out[i] (input order, [n x dim] fp32) = the row of keys[i] from the first tier
 * holding it — the cache, else the table, else the table's default vector. Duplicate keys
 * are served from ONE probe per distinct key: the distinct keys, in order of first
 * occurrence, are what the cache sees (one access each: stats count distinct keys). The
 * distinct misses present in the table are migrated into the cache once each (version
 * kBulkLoadVersion); keys absent everywhere are never cached. source_counts_out (device
 * u64[4], may be NULL) = per INPUT key {L1 cache, L2 table, L3 = 0, Default}
 * (LookupResult.source_counts); n_unique_out (device u64, may be NULL).
 * Asynchronous, no allocation, capturable. The cache, the table and the read-through
 * share one context; max_batch <= the cache's max_batch. */
typedef struct hps_gpu_readthrough_s* hps_gpu_readthrough;
int hps_gpu_readthrough_create(hps_gpu_cache cache, hps_gpu_table tbl, uint32_t table, uint64_t max_batch,
                               hps_gpu_readthrough* out_host);
int hps_gpu_readthrough_destroy(hps_gpu_readthrough rt);
int hps_gpu_readthrough_lookup(hps_gpu_readthrough rt, const uint64_t* keys, uint64_t n, float* out,
                               uint64_t* source_counts_out, uint64_t* n_unique_out);

/* syncs. */
int hps_gpu_cache_stats(hps_gpu_cache cache, hps_cache_stats* stats_host);
int hps_gpu_cache_reset_stats(hps_gpu_cache cache);
/* syncs: number of resident entries. */
int hps_gpu_cache_size(hps_gpu_cache cache, uint64_t* n_host);
/* White-box parity (tests): the whole set-major state, way e = set * ways + w — keys,
 * versions, freq (0 = empty way), last_touch [capacity], the per-set aging counters
 * [capacity / ways], and the raw rows (fp32, or binary16 bits for an F16 cache)
 * [capacity x dim]. Device pointers, any may be NULL; asynchronous on the stream. */
int hps_gpu_cache_debug_export(hps_gpu_cache cache, uint64_t* keys, uint64_t* versions, uint8_t* freq,
                               uint64_t* last_touch, uint64_t* set_access, void* vecs);

/* ---- UpdateBatch frames -> cache refresh (update.cu) ----
 * Frame (little-endian): "HPSU" | version u8 = 1 | name_len u16 | name |
 * seq u64 | count u32 | dim u16 | dtype u8 (0 F32, 1 F16) | count x (key u64, dim scalars).
 * There is no encode/decode in the reference sources; these follow SPEC.md with the
 * primitive encodings of proj/include/hps/bytes.hpp:33-133 (ByteWriter / ByteReader). */
typedef struct {
  char table[256];          /* NUL-terminated table name */
  uint32_t name_len;
  uint64_t seq;
  uint32_t count;
  uint32_t dim;
  int dtype;                /* 0 = F32, 1 = F16 */
  uint64_t entries_offset;  /* byte offset of entry 0 within the frame */
  uint64_t entry_bytes;     /* 8 + dim * scalar size */
} hps_update_header;

/* Host: validate a frame (BadMagic, BadFormatVersion, Truncated, TrailingBytes,
 * DuplicateKey, InvalidArgument for dim/dtype/name) and fill *header_host. */
int hps_update_batch_parse(const uint8_t* frame_host, uint64_t n, hps_update_header* header_host);
/* Host: encode a frame (values: count x dim scalars, float or uint16 F16 bits). With
 * out_host == NULL only *out_len_host (the frame size) is produced. */
int hps_update_batch_encode(const char* table_host, uint32_t name_len, uint64_t seq, uint32_t count, uint32_t dim,
                            int dtype, const uint64_t* keys_host, const void* values_host, uint8_t* out_host,
                            uint64_t out_cap, uint64_t* out_len_host);
/* Device: decode the entries (frame bytes from entries_offset, already on the device)
 * into keys, fp32 rows (F16 widened exactly) and versions (= seq; may be NULL). */
int hps_gpu_update_decode(hps_gpu_ctx ctx, const uint8_t* entries, const hps_update_header* header_host,
                          uint64_t* keys_out, float* vecs_out, uint64_t* versions_out);
/* syncs: parse on the host, move the entry bytes to the device once, decode, then
 * hps_gpu_cache_refresh with version = seq (replace only resident keys with an older
 * version). replaced_out (device, may be NULL) receives the replacement count. */
int hps_gpu_cache_apply_update(hps_gpu_cache cache, const uint8_t* frame_host, uint64_t n, uint64_t* replaced_out);

/* ---- placement planners (host-side) ---------------------------- */
enum { HPS_PLAN_LOCALIZED = 0, HPS_PLAN_DISTRIBUTED = 1, HPS_PLAN_HYBRID = 2 };

typedef struct {
  uint64_t vocab_size;  /* keys in the slot's table */
  uint32_t dim;
  uint32_t hotness;     /* max keys per sample */
} hps_slot_spec;

/* LPT over bytes (vocab*dim*4): slot_device_out[s] = owner. Infeasible if a slot fits nowhere. */
int hps_plan_localized(const hps_slot_spec* slots_host, uint32_t n_slots, const uint64_t* budget_host,
                       uint32_t n_devices, uint32_t* slot_device_out_host);
/* Feasibility of key_hash-mod-G sharding (total/G <= min budget * 1.05). */
int hps_plan_distributed(const hps_slot_spec* slots_host, uint32_t n_slots, const uint64_t* budget_host,
                         uint32_t n_devices);
/* Host evaluations of include/hps/hash.hpp (the same inline definitions the kernels use). */
uint64_t hps_key_hash_host(uint64_t key);
uint64_t hps_fastmod_u64_host(uint64_t a, uint64_t d);
/* Host mirror of the distributed shard rule: out[i] = partition_of(keys[i], n_devices). */
void hps_shard_of(const uint64_t* keys_host, uint64_t n, uint32_t n_devices, uint32_t* out_host);
/* Hot set for hybrid placement: top floor(budget/(dim*4)) keys by (count desc, key asc). */
int hps_plan_hybrid(const uint64_t* keys_host, const uint64_t* counts_host, uint64_t n_keys, uint32_t dim,
                    uint64_t hot_budget_bytes, uint64_t* hot_keys_out_host, uint64_t* n_hot_out_host);
/* All-to-all bytes per iteration (forward; backward is symmetric). p_cold: per-slot cold
 * mass, required for HPS_PLAN_HYBRID. */
int hps_estimate_comm(int strategy, uint64_t batch, const hps_slot_spec* slots_host, uint32_t n_slots,
                      uint32_t n_devices, const double* p_cold_host, double* fwd_bytes_host, double* bwd_bytes_host);

/* ---- lower tiers of the miss path: VDB (L2) and PDB (L3), host-resident (tiers.cpp) ----
 * SPEC.md:192-250 (volatile-store) and :252-318 (persistent-store); SURVEY.md §8(f) rank 4.
 * The VDB holds one table: shard = partition_of(key, num_shards) (hps/hash.hpp), at most
 * per_shard_capacity entries per shard; a put stores an entry iff its version is newer than
 * the resident one (or the key is absent); a put into a full shard drops the entry
 * (HPS_VDB_REJECT_NEW) or first removes the shard's entry with the smallest version
 * (HPS_VDB_EVICT_OLDEST_VERSION). get has no side effects. Shards lock single-writer /
 * multi-reader and are worked in parallel. All pointers are HOST pointers. */
enum { HPS_VDB_REJECT_NEW = 0, HPS_VDB_EVICT_OLDEST_VERSION = 1 };
typedef struct hps_vdb_s* hps_vdb;
int hps_vdb_create(uint32_t num_shards, uint64_t per_shard_capacity, int overflow_policy, uint32_t dim,
                   hps_vdb* out_host);
int hps_vdb_destroy(hps_vdb vdb);
int hps_vdb_put_batch(hps_vdb vdb, const uint64_t* keys, const float* vecs, const uint64_t* versions, uint64_t n,
                      uint64_t* stored_out);
int hps_vdb_get_batch(hps_vdb vdb, const uint64_t* keys, uint64_t n, float* vecs_out, uint64_t* versions_out,
                      uint8_t* found_out, uint64_t* n_found_out);
/* Point-in-time listing of one shard, ascending key; *n_out = its size (only the count when
 * cap < size). Bad index -> HPS_GPU_E_BAD_SHARD. */
int hps_vdb_shard_snapshot(hps_vdb vdb, uint32_t shard, uint64_t* keys, float* vecs, uint64_t* versions, uint64_t cap,
                           uint64_t* n_out);
int hps_vdb_size(hps_vdb vdb, uint64_t* n_out);

/* PDB: <root>/<table>/MANIFEST + append-only segments seg_NNNNNNNN.log of LogRecords
 *   key u64 | version u64 | dim u16 | dtype u8 (0 = f32) | payload dim x f32 | crc32c u32
 * (little-endian; CRC-32C of the preceding record bytes). open rebuilds the index (highest
 * version per key); a torn tail of a table's newest segment is dropped and truncated
 * (*dropped_tail_out counts them), a bad record anywhere else fails with
 * HPS_GPU_E_CORRUPTION. put appends iff newer; segments rotate at 64 MiB
 * (HPS_PDB_SEGMENT_BYTES overrides) with a file flush, and close flushes. */
typedef struct hps_pdb_s* hps_pdb;
int hps_pdb_open(const char* root, hps_pdb* out_host, uint64_t* dropped_tail_out);
int hps_pdb_close(hps_pdb pdb);
int hps_pdb_table_count(hps_pdb pdb, uint64_t* n_out);
int hps_pdb_create_table(hps_pdb pdb, const char* name, uint32_t dim, const float* default_vec /* NULL: zeros */);
int hps_pdb_table_info(hps_pdb pdb, const char* table, uint32_t* dim_out, float* default_vec_out, uint64_t* keys_out);
int hps_pdb_put_batch(hps_pdb pdb, const char* table, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                      uint64_t n, uint64_t* stored_out);
int hps_pdb_get_batch(hps_pdb pdb, const char* table, const uint64_t* keys, uint64_t n, float* vecs_out,
                      uint64_t* versions_out, uint8_t* found_out, uint64_t* n_found_out);
int hps_pdb_scan(hps_pdb pdb, const char* table, uint64_t* keys, float* vecs, uint64_t* versions, uint64_t cap,
                 uint64_t* n_out);
int hps_pdb_compact(hps_pdb pdb, const char* table, uint64_t* reclaimed_bytes_out);
/* CRC-32C of host bytes continuing `crc` (0 to start): the PDB record checksum (SSE4.2). */
uint32_t hps_crc32c_host(uint32_t crc, const void* data, size_t len);

/* ---- the tiered orchestrator: L1 GPU cache -> L2 VDB -> L3 PDB (tiered.cu) -----------
 * SPEC.md:322-345. lookup(keys) on the cache's context: distinct keys in first-occurrence
 * order (one tier probe per distinct key), L1 = hps_gpu_cache_query, the misses from the
 * VDB, then the PDB, else the PDB table's default vector (source Default); out[n x dim]
 * (device) in input order; source_counts_host[4] = per input key {L1, L2, L3, Default}.
 * Migrations are started and NOT waited for: keys found in L2 are inserted into L1 (at their
 * VDB version), keys found only in L3 into L2 and L1 (at their PDB version); absent keys are
 * inserted nowhere. hps_gpu_tiered_await(t) = the last lookup's migrations are visible.
 * One lookup at a time per hps_gpu_tiered (its staging buffers are reused); the VDB and PDB
 * themselves may be shared by several (their shards/tables lock). */
typedef struct hps_gpu_tiered_s* hps_gpu_tiered;
int hps_gpu_tiered_create(hps_gpu_cache l1, hps_vdb l2, hps_pdb l3, const char* table, uint64_t max_batch,
                          hps_gpu_tiered* out_host);
int hps_gpu_tiered_destroy(hps_gpu_tiered t);
int hps_gpu_tiered_lookup(hps_gpu_tiered t, const uint64_t* keys, uint64_t n, float* out,
                          uint64_t* source_counts_host);
int hps_gpu_tiered_await(hps_gpu_tiered t);

/* ---- synthetic workload helpers (device-side generators) ------- */
/* The deterministic row initialiser of DESIGN.md §4.1 (host-callable, for checks). */
float hps_gpu_init_value(uint64_t seed, uint64_t key, uint32_t j);
/* out[i] = mix64(seed ^ (first + i)) : distinct keys (mix64 is a bijection). */
int hps_gpu_gen_keys(hps_gpu_ctx ctx, uint64_t seed, uint64_t first, uint64_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* HPS_GPU_H_ */
