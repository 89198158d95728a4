// oracle/oracle.cpp — CPU restatement of the sparse-embedding hot path.
//
// TEST INFRASTRUCTURE ONLY. This library is the parity checker for the B200 CUDA
// path (paper_2210_08803_b200/csrc). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it. The product path
// never links, imports or falls back to it.
//
// Parity status
//   * key_hash / partition_of / f16 / finiteness: PINNED against the reference's own
//     compiled code (oracle/_ref/libhps_ref.so, built from /root/reference/proj by
//     oracle/Makefile) through tests/golden/ref_vectors.json (gen: oracle/gen_golden.py).
//   * hot cache: restates SPEC.md:112-190 with the resolutions of DESIGN.md §5;
//     pinned to the SPEC examples only (the reference ships no cache code).
//   * row init, pooling, backward dedup/reduction and optimizers: the reference has
//     no code for these -> "parity unpinned"; this file DEFINES
//     them and the GPU must match it.
//
// Floating point: compiled with -ffp-contract=off, every expression is written in
// the exact operation order the CUDA kernels use (no FMA on either side).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;  // hash.hpp:27
constexpr uint64_t kFnvPrime = 0x100000001b3ull;       // hash.hpp:28

// proj/include/hps/hash.hpp:42-49 — FNV-1a 64 over the 8 little-endian key bytes.
inline uint64_t key_hash(uint64_t key) {
  uint64_t h = kFnvBasis;
  for (int i = 0; i < 8; ++i) {
    h ^= (key >> (8 * i)) & 0xffu;
    h *= kFnvPrime;
  }
  return h;
}

// splitmix64 finaliser: a bijection on u64.
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// deterministic initial row value, exact in fp32 on every platform.
inline float init_value(uint64_t seed, uint64_t key, uint32_t j) {
  uint64_t u = mix64(key_hash(key) + seed * 0xd1b54a32d192ed03ull +
                     (static_cast<uint64_t>(j) + 1) * 0x9e3779b97f4a7c15ull);
  float v = static_cast<float>(u >> 40);           // 24-bit integer, exact
  return (v * 5.9604644775390625e-08f - 0.5f) * 0.03125f;  // (v*2^-24 - 0.5) * 2^-5
}

inline bool non_finite(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  return (b & 0x7f800000u) == 0x7f800000u;  // kernels_scalar.cpp:110-116
}

struct OptParams {
  float lr, eps, beta1, beta2, one_minus_beta1, one_minus_beta2, lr_t;
};

constexpr uint32_t kChunk = 32;  // DESIGN.md §4.3 blocked reduction width

// ---------------------------------------------------------------------------
// Table group model
// ---------------------------------------------------------------------------
struct Table {
  uint32_t n_tables = 0, dim = 0, n_slots = 0;
  int optimizer = 0;
  uint64_t seed = 0;
  float a0 = 0.f;
  std::vector<uint64_t> cap, row_base, n_rows;
  std::vector<uint32_t> slot_table;
  std::vector<std::unordered_map<uint64_t, uint64_t>> index;  // per table key -> local row
  std::vector<uint64_t> row_key;                              // global row -> key
  std::vector<float> w, s0, s1;                               // [R x dim]
  std::vector<std::vector<float>> defaults;
  // state of the last training lookup
  std::vector<uint64_t> occ_row;  // global row or UINT64_MAX (absent)
  std::vector<uint32_t> occ_bag;
  std::vector<uint32_t> bag_len;
  int last_combiner = 0;
  uint64_t last_n_bags = 0;
  std::vector<uint32_t> last_unique;
  bool f16 = false;  // binary16 rows (inference table): stored as their exact fp32 widening

  int n_state() const { return optimizer == 0 ? 0 : optimizer == 1 ? 1 : 2; }
};
float f16_round_trip(float x);
bool f16_overflows(float x);

// DESIGN.md §4.1 insert: new keys get rows in order of first occurrence, continuing
// from the table's row count; with `rows`, every distinct key of the call (new or
// existing) takes the row of its FIRST occurrence; without, new rows get init_value.
int table_insert(Table* t, uint32_t table, const uint64_t* keys, uint64_t n, const float* rows,
                 uint64_t* rows_out) {
  if (table >= t->n_tables) return 11;
  auto& idx = t->index[table];
  const uint32_t D = t->dim;
  // NaN/Inf rejected on ingest (types.cpp:67-70 semantics): the whole call is refused.
  if (rows) {
    for (uint64_t i = 0; i < n * D; ++i)
      if (non_finite(rows[i])) return 10;
    if (t->f16)  // binary16 table: a value whose rounding overflows refuses the call (F16Range)
      for (uint64_t i = 0; i < n * D; ++i)
        if (f16_overflows(rows[i])) return 9;
  }
  uint64_t new_cnt = 0;
  {
    std::unordered_map<uint64_t, char> seen;
    for (uint64_t i = 0; i < n; ++i)
      if (!idx.count(keys[i]) && seen.emplace(keys[i], 1).second) ++new_cnt;
  }
  if (t->n_rows[table] + new_cnt > t->cap[table]) return 16;  // Infeasible: nothing inserted
  std::unordered_map<uint64_t, char> written;
  for (uint64_t i = 0; i < n; ++i) {
    auto it = idx.find(keys[i]);
    uint64_t local;
    const bool fresh = it == idx.end();
    if (fresh) {
      local = t->n_rows[table]++;
      idx.emplace(keys[i], local);
    } else {
      local = it->second;
    }
    const uint64_t g = t->row_base[table] + local;
    if (fresh) {
      t->row_key[g] = keys[i];
      if (t->optimizer == 1)
        for (uint32_t j = 0; j < D; ++j) t->s0[g * D + j] = t->a0;
      if (t->optimizer == 2)
        for (uint32_t j = 0; j < D; ++j) t->s0[g * D + j] = 0.f, t->s1[g * D + j] = 0.f;
      if (!rows)
        for (uint32_t j = 0; j < D; ++j) t->w[g * D + j] = init_value(t->seed, keys[i], j);
    }
    if (rows && written.emplace(keys[i], 1).second)
      std::memcpy(&t->w[g * D], &rows[i * D], D * sizeof(float));
    if (t->f16 && (fresh || rows))  // rows are held rounded to binary16
      for (uint32_t j = 0; j < D; ++j) t->w[g * D + j] = f16_round_trip(t->w[g * D + j]);
    if (rows_out) rows_out[i] = local;
  }
  return 0;
}

// DESIGN.md §4.2 pooling. keys sample-major; offsets==nullptr => one key per bag.
int lookup_pooled(Table* t, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                  int combiner, float* out, int train, int n_threads) {
  const uint32_t D = t->dim, S = t->n_slots;
  const uint64_t n_bags = static_cast<uint64_t>(n_samples) * S;
  const uint64_t n_keys = offsets ? offsets[n_bags] : n_bags;
  if (train) {
    t->occ_row.assign(n_keys, UINT64_MAX);
    t->occ_bag.assign(n_keys, 0);
    t->bag_len.assign(n_bags, 0);
    t->last_combiner = combiner;
    t->last_n_bags = n_bags;
  }
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(n_threads)
#endif
  for (int64_t b = 0; b < static_cast<int64_t>(n_bags); ++b) {
    const uint32_t slot = static_cast<uint32_t>(b % S);
    const uint32_t table = t->slot_table[slot];
    const uint64_t lo = offsets ? offsets[b] : b, hi = offsets ? offsets[b + 1] : b + 1;
    float* o = out + b * D;
    for (uint32_t j = 0; j < D; ++j) o[j] = 0.0f;
    for (uint64_t i = lo; i < hi; ++i) {
      auto it = t->index[table].find(keys[i]);
      const float* src;
      if (it == t->index[table].end()) {
        src = t->defaults[table].data();
      } else {
        uint64_t g = t->row_base[table] + it->second;
        src = &t->w[g * D];
        if (train) t->occ_row[i] = g;
      }
      if (train) t->occ_bag[i] = static_cast<uint32_t>(b);
      for (uint32_t j = 0; j < D; ++j) o[j] = o[j] + src[j];
    }
    const uint32_t len = static_cast<uint32_t>(hi - lo);
    if (train) t->bag_len[b] = len;
    if (combiner == 1 && len > 0) {
      const float fl = static_cast<float>(len);
      for (uint32_t j = 0; j < D; ++j) o[j] = o[j] / fl;
    }
  }
  return 0;
}

// DESIGN.md §4.4 optimizers, in the exact operation order of the CUDA kernels.
inline void apply_optimizer(int optimizer, float* w, float* s0, float* s1, uint32_t D, const float* g,
                            const OptParams& p) {
  if (optimizer == 3) {  // gradient only (hybrid hot rows): w <- g, s0[0] <- 1 (touched)
    for (uint32_t j = 0; j < D; ++j) w[j] = g[j];
    if (s0) s0[0] = 1.0f;
  } else if (optimizer == 0) {  // SGD: w -= lr*g
    for (uint32_t j = 0; j < D; ++j) w[j] = w[j] - p.lr * g[j];
  } else if (optimizer == 1) {  // AdaGrad: a += g^2; w -= lr*g/(sqrt(a)+eps)
    for (uint32_t j = 0; j < D; ++j) {
      s0[j] = s0[j] + g[j] * g[j];
      w[j] = w[j] - (p.lr * g[j]) / (std::sqrt(s0[j]) + p.eps);
    }
  } else {  // Adam (lazy): m,v moments; lr_t carries the bias correction
    for (uint32_t j = 0; j < D; ++j) {
      s0[j] = p.beta1 * s0[j] + p.one_minus_beta1 * g[j];
      s1[j] = p.beta2 * s1[j] + p.one_minus_beta2 * (g[j] * g[j]);
      w[j] = w[j] - (p.lr_t * s0[j]) / (std::sqrt(s1[j]) + p.eps);
    }
  }
}

// per-occurrence gradient, dedup by row (stable in occurrence order),
// kChunk-ary blocked tree reduction (chunks of kChunk summed sequentially; the list of
// chunk partials reduced the same way until one remains — plain sequential order for
// <= kChunk occurrences), then the optimizer on each unique row. `row_ptr(row, k)` gives
// the weight (k=0) and state (k=1,2) row of a global row id.
template <class RowPtr>
void reduce_and_update(const std::vector<uint64_t>& occ_row, const std::vector<uint32_t>& occ_bag,
                       const std::vector<uint32_t>& bag_len, bool mean, const float* dout, uint32_t D, int optimizer,
                       const OptParams& p, int n_threads, std::vector<uint32_t>* unique_out, RowPtr row_ptr) {
  const uint64_t N = occ_row.size();
  std::vector<uint64_t> order;
  order.reserve(N);
  for (uint64_t i = 0; i < N; ++i)
    if (occ_row[i] != UINT64_MAX) order.push_back(i);
  std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return occ_row[a] < occ_row[b]; });
  std::vector<uint64_t> seg;  // segment starts into `order`
  for (uint64_t i = 0; i < order.size(); ++i)
    if (i == 0 || occ_row[order[i]] != occ_row[order[i - 1]]) seg.push_back(i);
  seg.push_back(order.size());
  const uint64_t U = seg.size() - 1;
  if (unique_out) {
    unique_out->resize(U);
    for (uint64_t u = 0; u < U; ++u) (*unique_out)[u] = static_cast<uint32_t>(occ_row[order[seg[u]]]);
  }
#ifdef _OPENMP
#pragma omp parallel num_threads(n_threads)
#endif
  {
    std::vector<float> acc(D), part(D), gi(D);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
    for (int64_t u = 0; u < static_cast<int64_t>(U); ++u) {
      const uint64_t lo = seg[u], hi = seg[u + 1];
      auto grad_of = [&](uint64_t occ, float* dst) {
        const uint32_t b = occ_bag[occ];
        const float* d = dout + static_cast<uint64_t>(b) * D;
        if (mean) {
          const float fl = static_cast<float>(bag_len[b]);
          for (uint32_t j = 0; j < D; ++j) dst[j] = d[j] / fl;
        } else {
          for (uint32_t j = 0; j < D; ++j) dst[j] = d[j];
        }
      };
      // Level 1: chunks of kChunk occurrences, each summed sequentially from its first element.
      std::vector<float> level;  // partials, D floats each
      for (uint64_t c = lo; c < hi; c += kChunk) {
        const uint64_t ce = std::min<uint64_t>(hi, c + kChunk);
        grad_of(order[c], part.data());
        for (uint64_t i = c + 1; i < ce; ++i) {
          grad_of(order[i], gi.data());
          for (uint32_t j = 0; j < D; ++j) part[j] = part[j] + gi[j];
        }
        level.insert(level.end(), part.begin(), part.end());
      }
      // Levels 2..: the partial list is reduced the same way (chunks of kChunk, sequential)
      // until one vector remains — a kChunk-ary blocked tree in canonical order.
      while (level.size() > D) {
        const uint64_t m = level.size() / D;
        std::vector<float> next;
        for (uint64_t c = 0; c < m; c += kChunk) {
          const uint64_t ce = std::min<uint64_t>(m, c + kChunk);
          std::copy(level.begin() + c * D, level.begin() + (c + 1) * D, part.begin());
          for (uint64_t i = c + 1; i < ce; ++i)
            for (uint32_t j = 0; j < D; ++j) part[j] = part[j] + level[i * D + j];
          next.insert(next.end(), part.begin(), part.end());
        }
        level.swap(next);
      }
      std::copy(level.begin(), level.end(), acc.begin());
      const uint64_t r = occ_row[order[lo]];
      apply_optimizer(optimizer, row_ptr(r, 0), row_ptr(r, 1), row_ptr(r, 2), D, acc.data(), p);
    }
  }
}

int backward_update(Table* t, const float* dout, const OptParams& p, int n_threads) {
  const uint32_t D = t->dim;
  reduce_and_update(t->occ_row, t->occ_bag, t->bag_len, t->last_combiner == 1, dout, D, t->optimizer, p, n_threads,
                    &t->last_unique, [&](uint64_t r, int k) -> float* {
                      if (k == 0) return &t->w[r * D];
                      if (k == 1) return t->s0.empty() ? nullptr : &t->s0[r * D];
                      return t->s1.empty() ? nullptr : &t->s1[r * D];
                    });
  return 0;
}

// ---------------------------------------------------------------------------
// Sparse (lazily materialised) model of a fully pre-loaded table group, for the CPU
// baseline at BASELINE scale: every key of every table logically exists with its
// init_value row (exactly the GPU bench's bulk-loaded state); rows are materialised on
// first touch instead of allocating 96 GB of host memory.
// ---------------------------------------------------------------------------
struct Sparse {
  uint32_t n_tables = 0, dim = 0, n_slots = 0;
  int optimizer = 0;
  uint64_t seed = 0;
  float a0 = 0.f;
  std::vector<uint32_t> slot_table;
  std::vector<std::unordered_map<uint64_t, uint64_t>> index;
  std::vector<float> w, s0, s1;
  uint64_t rows = 0;
  std::vector<uint64_t> occ_row;
  std::vector<uint32_t> occ_bag, bag_len;

  uint64_t touch(uint32_t table, uint64_t key) {
    auto it = index[table].find(key);
    if (it != index[table].end()) return it->second;
    const uint64_t r = rows++;
    index[table].emplace(key, r);
    if (w.size() < rows * dim) {
      const uint64_t cap = std::max<uint64_t>(rows * dim * 2, 1 << 20);
      w.resize(cap);
      if (optimizer >= 1) s0.resize(cap);
      if (optimizer >= 2) s1.resize(cap);
    }
    for (uint32_t j = 0; j < dim; ++j) w[r * dim + j] = init_value(seed, key, j);
    if (optimizer == 1)
      for (uint32_t j = 0; j < dim; ++j) s0[r * dim + j] = a0;
    if (optimizer == 2)
      for (uint32_t j = 0; j < dim; ++j) s0[r * dim + j] = 0.f, s1[r * dim + j] = 0.f;
    return r;
  }
};

// ---------------------------------------------------------------------------
// binary16 storage (restates kernels_scalar.cpp:25-57 f32_bits_to_f16_bits
// and its inverse — pinned against the compiled reference in tests/test_golden_cpu.py):
// IEEE round-to-nearest-even, overflow to infinity, NaN kept quiet with its top payload.
// ---------------------------------------------------------------------------
uint16_t f32_to_f16_bits(uint32_t b) {
  const uint32_t sign = (b >> 16) & 0x8000u, a = b & 0x7fffffffu;
  if (a > 0x7f800000u) return static_cast<uint16_t>(sign | 0x7e00u | ((a >> 13) & 0x3ffu));
  if (a == 0x7f800000u) return static_cast<uint16_t>(sign | 0x7c00u);
  const int exp = static_cast<int>(a >> 23) - 112;  // binary16 exponent field (bias 15 vs 127)
  if (exp >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
  if (exp <= 0) {  // binary16 subnormal (or zero): quantum 2^-24
    if (exp < -10) return static_cast<uint16_t>(sign);
    const uint32_t m = (a & 0x7fffffu) | 0x800000u, shift = static_cast<uint32_t>(14 - exp);
    uint32_t q = m >> shift;
    const uint32_t r = m & ((1u << shift) - 1u), half = 1u << (shift - 1u);
    if (r > half || (r == half && (q & 1u))) ++q;
    return static_cast<uint16_t>(sign | q);
  }
  uint32_t q = (static_cast<uint32_t>(exp) << 10) | ((a >> 13) & 0x3ffu);
  const uint32_t r = a & 0x1fffu;
  if (r > 0x1000u || (r == 0x1000u && (q & 1u))) ++q;  // a carry may reach 0x7c00 (infinity)
  return static_cast<uint16_t>(sign | q);
}
uint32_t f16_to_f32_bits(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  if (e == 31) return sign | 0x7f800000u | (m << 13);
  if (e) return sign | ((e + 112u) << 23) | (m << 13);
  if (!m) return sign;
  int k = 0;  // subnormal: normalise
  uint32_t mm = m;
  while (!(mm & 0x400u)) {
    mm <<= 1;
    ++k;
  }
  return sign | (static_cast<uint32_t>(113 - k) << 23) | ((mm & 0x3ffu) << 13);
}
float f16_round_trip(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  const uint32_t w = f16_to_f32_bits(f32_to_f16_bits(b));
  float y;
  std::memcpy(&y, &w, 4);
  return y;
}
bool f16_overflows(float x) {  // finite x whose binary16 rounding is infinite
  uint32_t b;
  std::memcpy(&b, &x, 4);
  return ((f32_to_f16_bits(b) & 0x7fffu) == 0x7c00u) && (b & 0x7fffffffu) < 0x7f800000u;
}

// ---------------------------------------------------------------------------
// Hot cache model: SPEC.md:112-190 with DESIGN.md §5 resolutions
// ---------------------------------------------------------------------------
struct Cache {
  uint64_t capacity = 0, num_sets = 0, aging_period = 0;
  uint32_t ways = 0, dim = 0;
  uint64_t clock = 0;
  std::vector<uint64_t> key, version, last_touch, set_acc;
  std::vector<uint8_t> freq;  // 0 == empty way
  std::vector<float> vec;  // binary16 storage: values held as their exact fp32 widening
  bool f16 = false;
  uint64_t st[7] = {0, 0, 0, 0, 0, 0, 0};  // queries hits misses insertions rejected refresh evictions
  // Validate an entry (NaN/Inf -> NonFinite 10; binary16 out of range -> F16Range 9).
  int check(const float* v) const {
    bool bad = false, range = false;
    for (uint32_t j = 0; j < dim; ++j) {
      bad |= non_finite(v[j]);
      if (f16) range |= f16_overflows(v[j]);
    }
    return bad ? 10 : range ? 9 : 0;
  }
  void store(uint64_t e, const float* v) {
    for (uint32_t j = 0; j < dim; ++j) vec[e * dim + j] = f16 ? f16_round_trip(v[j]) : v[j];
  }

  uint64_t set_of(uint64_t k) const { return key_hash(k) % num_sets; }
  // One access to set s (counted before the access is applied; the
  // access that completes an aging period first halves the set's counters).
  void access(uint64_t s) {
    if (++set_acc[s] >= aging_period) {
      set_acc[s] = 0;
      for (uint32_t w = 0; w < ways; ++w) {
        uint8_t& f = freq[s * ways + w];
        if (f) f = std::max<uint8_t>(1, f >> 1);
      }
    }
  }
  int find(uint64_t s, uint64_t k) const {
    for (uint32_t w = 0; w < ways; ++w)
      if (freq[s * ways + w] && key[s * ways + w] == k) return static_cast<int>(w);
    return -1;
  }
};

}  // namespace

extern "C" {

uint64_t orc_key_hash(uint64_t key) { return key_hash(key); }
void orc_key_hash_n(const uint64_t* keys, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = key_hash(keys[i]);
}
// hash.hpp:52-54
void orc_partition_of_n(const uint64_t* keys, uint64_t n, uint32_t shards, uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(key_hash(keys[i]) % shards);
}
uint64_t orc_fnv1a64(const uint8_t* data, uint64_t n) {  // hash.hpp:30-37
  uint64_t h = kFnvBasis;
  for (uint64_t i = 0; i < n; ++i) h = (h ^ data[i]) * kFnvPrime;
  return h;
}
uint64_t orc_mix64(uint64_t x) { return mix64(x); }
float orc_init_value(uint64_t seed, uint64_t key, uint32_t j) { return init_value(seed, key, j); }
int orc_has_non_finite_f32(const float* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (non_finite(v[i])) return 1;
  return 0;
}
int orc_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// ---- table ----
void* orc_table_create(uint32_t n_tables, uint32_t dim, const uint64_t* caps, uint32_t n_slots,
                       const uint32_t* slot_table, int optimizer, uint64_t seed, float a0) {
  auto* t = new Table;
  t->n_tables = n_tables;
  t->dim = dim;
  t->n_slots = n_slots;
  t->optimizer = optimizer;
  t->seed = seed;
  t->a0 = a0;
  t->cap.assign(caps, caps + n_tables);
  t->row_base.resize(n_tables);
  uint64_t r = 0;
  for (uint32_t i = 0; i < n_tables; ++i) t->row_base[i] = r, r += caps[i];
  t->n_rows.assign(n_tables, 0);
  t->slot_table.assign(slot_table, slot_table + n_slots);
  t->index.resize(n_tables);
  t->row_key.assign(r, 0);
  t->w.assign(r * dim, 0.f);
  if (t->n_state() >= 1) t->s0.assign(r * dim, 0.f);
  if (t->n_state() >= 2) t->s1.assign(r * dim, 0.f);
  t->defaults.assign(n_tables, std::vector<float>(dim, 0.f));
  return t;
}
void orc_table_destroy(void* h) { delete static_cast<Table*>(h); }
void orc_table_set_dtype(void* h, int dtype) { static_cast<Table*>(h)->f16 = dtype == 1; }
void orc_table_set_default(void* h, uint32_t table, const float* v) {
  auto* t = static_cast<Table*>(h);
  std::memcpy(t->defaults[table].data(), v, t->dim * sizeof(float));
}
uint64_t orc_table_size(void* h, uint32_t table) { return static_cast<Table*>(h)->n_rows[table]; }
int orc_table_insert(void* h, uint32_t table, const uint64_t* keys, uint64_t n, const float* rows,
                     uint64_t* rows_out) {
  return table_insert(static_cast<Table*>(h), table, keys, n, rows, rows_out);
}
void orc_table_find(void* h, uint32_t table, const uint64_t* keys, uint64_t n, uint64_t* rows_out) {
  auto* t = static_cast<Table*>(h);
  for (uint64_t i = 0; i < n; ++i) {
    auto it = t->index[table].find(keys[i]);
    rows_out[i] = it == t->index[table].end() ? UINT64_MAX : it->second;
  }
}
void orc_table_export(void* h, uint32_t table, uint64_t row_begin, uint64_t n, float* w, float* s0,
                      float* s1) {
  auto* t = static_cast<Table*>(h);
  const uint64_t g = t->row_base[table] + row_begin, D = t->dim;
  if (w) std::memcpy(w, &t->w[g * D], n * D * sizeof(float));
  if (s0 && t->n_state() >= 1) std::memcpy(s0, &t->s0[g * D], n * D * sizeof(float));
  if (s1 && t->n_state() >= 2) std::memcpy(s1, &t->s1[g * D], n * D * sizeof(float));
}
void orc_table_row_keys(void* h, uint32_t table, uint64_t row_begin, uint64_t n, uint64_t* out) {
  auto* t = static_cast<Table*>(h);
  std::memcpy(out, &t->row_key[t->row_base[table] + row_begin], n * sizeof(uint64_t));
}
int orc_lookup_pooled(void* h, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples,
                      int combiner, float* out, int train, int n_threads) {
  return lookup_pooled(static_cast<Table*>(h), keys, offsets, n_samples, combiner, out, train,
                       n_threads < 1 ? 1 : n_threads);
}
// Owner side of the distributed exchange: rows of keys[i] in tables[i]; with `train` the
// next backward takes one gradient row per key (bag == occurrence, length 1, sum).
int orc_gather_rows(void* h, const uint64_t* keys, const uint32_t* tables, uint64_t n, float* out, int train) {
  auto* t = static_cast<Table*>(h);
  const uint32_t D = t->dim;
  if (train) {
    t->occ_row.assign(n, UINT64_MAX);
    t->occ_bag.resize(n);
    t->bag_len.assign(n, 1);
    t->last_combiner = 0;
    t->last_n_bags = n;
  }
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t table = tables[i];
    auto it = t->index[table].find(keys[i]);
    const float* src;
    if (it == t->index[table].end()) {
      src = t->defaults[table].data();
    } else {
      const uint64_t g = t->row_base[table] + it->second;
      src = &t->w[g * D];
      if (train) t->occ_row[i] = g;
    }
    if (train) t->occ_bag[i] = static_cast<uint32_t>(i);
    for (uint32_t j = 0; j < D; ++j) out[i * D + j] = 0.0f + src[j];
  }
  return 0;
}
// Hybrid embedding (backward.cu kOptGrad / hps_gpu_backward_reduce): the canonical
// per-row gradient sums of the last training lookup into grads_out [R x dim], and
// touched_out[r] = 1 for every row with an occurrence. No optimizer step.
int orc_reduce_only(void* h, const float* dout, float* grads_out, float* touched_out) {
  Table* t = static_cast<Table*>(h);
  const uint32_t D = t->dim;
  reduce_and_update(t->occ_row, t->occ_bag, t->bag_len, t->last_combiner == 1, dout, D, 3, OptParams{}, 1, nullptr,
                    [&](uint64_t r, int k) -> float* {
                      if (k == 0) return grads_out + r * D;
                      if (k == 1) return touched_out + r;
                      return nullptr;
                    });
  return 0;
}
// The optimizer on every global row r with touched[r] != 0 and gradient grads[r x dim].
int orc_apply_grads(void* h, const float* grads, const uint32_t* touched, const float* opt7) {
  Table* t = static_cast<Table*>(h);
  const uint32_t D = t->dim;
  OptParams p{opt7[0], opt7[1], opt7[2], opt7[3], opt7[4], opt7[5], opt7[6]};
  const uint64_t R = t->row_key.size();
  for (uint64_t r = 0; r < R; ++r) {
    if (!touched[r]) continue;
    apply_optimizer(t->optimizer, &t->w[r * D], t->s0.empty() ? nullptr : &t->s0[r * D],
                    t->s1.empty() ? nullptr : &t->s1[r * D], D, grads + r * D, p);
  }
  return 0;
}

int orc_backward_update(void* h, const float* dout, const float* opt7, int n_threads) {
  OptParams p{opt7[0], opt7[1], opt7[2], opt7[3], opt7[4], opt7[5], opt7[6]};
  return backward_update(static_cast<Table*>(h), dout, p, n_threads < 1 ? 1 : n_threads);
}
uint64_t orc_last_unique(void* h, uint32_t* rows_out) {
  auto* t = static_cast<Table*>(h);
  if (rows_out) std::memcpy(rows_out, t->last_unique.data(), t->last_unique.size() * 4);
  return t->last_unique.size();
}

// ---- cache ----
void* orc_cache_create(uint64_t capacity, uint32_t ways, uint64_t aging_interval, uint32_t dim) {
  auto* c = new Cache;
  c->capacity = capacity;
  c->ways = ways;
  c->dim = dim;
  c->num_sets = capacity / ways;
  if (aging_interval == 0) aging_interval = 10 * capacity;  // SPEC.md:118 default
  c->aging_period = std::max<uint64_t>(1, aging_interval / c->num_sets);
  c->key.assign(capacity, 0);
  c->version.assign(capacity, 0);
  c->last_touch.assign(capacity, 0);
  c->freq.assign(capacity, 0);
  c->set_acc.assign(c->num_sets, 0);
  c->vec.assign(capacity * dim, 0.f);
  return c;
}
void orc_cache_destroy(void* h) { delete static_cast<Cache*>(h); }
void orc_cache_set_dtype(void* h, int dtype) { static_cast<Cache*>(h)->f16 = dtype == 1; }
// binary16 conversions (the restatement above), element-wise
void orc_f32_to_f16(const float* src, uint16_t* dst, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t b;
    std::memcpy(&b, src + i, 4);
    dst[i] = f32_to_f16_bits(b);
  }
}
void orc_f16_to_f32(const uint16_t* src, float* dst, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t b = f16_to_f32_bits(src[i]);
    std::memcpy(dst + i, &b, 4);
  }
}
// SPEC.md:131-139
void orc_cache_query(void* h, const uint64_t* keys, uint64_t n, float* found_vecs, uint32_t* found_idx,
                     uint32_t* missing_idx, uint64_t* counts) {
  auto* c = static_cast<Cache*>(h);
  uint64_t nf = 0, nm = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t s = c->set_of(keys[i]);
    c->access(s);
    const uint64_t t = ++c->clock;
    const int w = c->find(s, keys[i]);
    c->st[0]++;
    if (w >= 0) {
      const uint64_t e = s * c->ways + w;
      c->freq[e] = static_cast<uint8_t>(std::min<int>(255, c->freq[e] + 1));
      c->last_touch[e] = t;
      if (found_vecs) std::memcpy(found_vecs + nf * c->dim, &c->vec[e * c->dim], c->dim * 4);
      if (found_idx) found_idx[nf] = static_cast<uint32_t>(i);
      ++nf;
      c->st[1]++;
    } else {
      if (missing_idx) missing_idx[nm] = static_cast<uint32_t>(i);
      ++nm;
      c->st[2]++;
    }
  }
  if (counts) counts[0] = nf, counts[1] = nm;
}
// SPEC.md:140-148
uint64_t orc_cache_insert(void* h, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                          uint64_t n, int* status) {
  auto* c = static_cast<Cache*>(h);
  uint64_t admitted = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const float* v = vecs + i * c->dim;
    if (const int e = c->check(v)) {
      if (status && !*status) *status = e;
      continue;
    }
    const uint64_t s = c->set_of(keys[i]);
    c->access(s);
    const uint64_t t = ++c->clock;
    const int w = c->find(s, keys[i]);
    if (w >= 0) {  // resident: refresh semantics
      const uint64_t e = s * c->ways + w;
      if (versions[i] > c->version[e]) {
        c->store(e, v);
        c->version[e] = versions[i];
        c->st[5]++;
      }
      continue;
    }
    int slot = -1;
    for (uint32_t q = 0; q < c->ways; ++q)
      if (!c->freq[s * c->ways + q]) {
        slot = static_cast<int>(q);
        break;
      }
    if (slot < 0) {  // evict min (freq, last_touch)
      slot = 0;
      for (uint32_t q = 1; q < c->ways; ++q) {
        const uint64_t a = s * c->ways + q, b = s * c->ways + slot;
        if (c->freq[a] < c->freq[b] || (c->freq[a] == c->freq[b] && c->last_touch[a] < c->last_touch[b]))
          slot = static_cast<int>(q);
      }
      c->st[6]++;
    }
    const uint64_t e = s * c->ways + slot;
    c->key[e] = keys[i];
    c->version[e] = versions[i];
    c->freq[e] = 1;
    c->last_touch[e] = t;
    c->store(e, v);
    c->st[3]++;
    ++admitted;
  }
  return admitted;
}
// SPEC.md:149-157
uint64_t orc_cache_refresh(void* h, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                           uint64_t n, int* status) {
  auto* c = static_cast<Cache*>(h);
  uint64_t replaced = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const float* v = vecs + i * c->dim;
    if (const int e = c->check(v)) {
      if (status && !*status) *status = e;
      continue;
    }
    const uint64_t s = c->set_of(keys[i]);
    const int w = c->find(s, keys[i]);
    if (w < 0) continue;
    const uint64_t e = s * c->ways + w;
    if (versions[i] > c->version[e]) {
      c->store(e, v);
      c->version[e] = versions[i];
      c->st[5]++;
      ++replaced;
    }
  }
  return replaced;
}
void orc_cache_stats(void* h, uint64_t* out7) { std::memcpy(out7, static_cast<Cache*>(h)->st, 56); }
void orc_cache_reset_stats(void* h) { std::memset(static_cast<Cache*>(h)->st, 0, 56); }
uint64_t orc_cache_size(void* h) {
  auto* c = static_cast<Cache*>(h);
  uint64_t n = 0;
  for (auto f : c->freq) n += f != 0;
  return n;
}
// Snapshot of a set's metadata for white-box parity: key, version, freq, last_touch per way.
void orc_cache_set_state(void* h, uint64_t set, uint64_t* keys, uint64_t* versions, uint8_t* freq,
                         uint64_t* last_touch) {
  auto* c = static_cast<Cache*>(h);
  const uint64_t b = set * c->ways;
  std::memcpy(keys, &c->key[b], c->ways * 8);
  std::memcpy(versions, &c->version[b], c->ways * 8);
  std::memcpy(freq, &c->freq[b], c->ways);
  std::memcpy(last_touch, &c->last_touch[b], c->ways * 8);
}

// The whole cache state (white-box parity with hps_gpu_cache_debug_export); NULL skips.
void orc_cache_export(void* h, uint64_t* keys, uint64_t* versions, uint8_t* freq, uint64_t* last_touch,
                      uint64_t* set_access, float* vecs) {
  auto* c = static_cast<Cache*>(h);
  if (keys) std::memcpy(keys, c->key.data(), c->capacity * 8);
  if (versions) std::memcpy(versions, c->version.data(), c->capacity * 8);
  if (freq) std::memcpy(freq, c->freq.data(), c->capacity);
  if (last_touch) std::memcpy(last_touch, c->last_touch.data(), c->capacity * 8);
  if (set_access) std::memcpy(set_access, c->set_acc.data(), c->num_sets * 8);
  if (vecs) std::memcpy(vecs, c->vec.data(), c->capacity * c->dim * 4);
}

// ---- sparse CPU step (baseline timing; same math as the table model) ----
void* orc_sparse_create(uint32_t n_tables, uint32_t dim, const uint32_t* slot_table, uint32_t n_slots, int optimizer,
                        uint64_t seed, float a0) {
  auto* s = new Sparse;
  s->n_tables = n_tables;
  s->dim = dim;
  s->n_slots = n_slots;
  s->optimizer = optimizer;
  s->seed = seed;
  s->a0 = a0;
  s->slot_table.assign(slot_table, slot_table + n_slots);
  s->index.resize(n_tables);
  return s;
}
void orc_sparse_destroy(void* h) { delete static_cast<Sparse*>(h); }
// One fwd+bwd+update step: keys sample-major, offsets==nullptr => one key per bag.
int orc_sparse_step(void* h, const uint64_t* keys, const uint32_t* offsets, uint32_t n_samples, int combiner,
                    const float* dout, const float* opt7, float* out, int n_threads) {
  auto* s = static_cast<Sparse*>(h);
  const uint32_t D = s->dim, S = s->n_slots;
  const uint64_t n_bags = static_cast<uint64_t>(n_samples) * S;
  const uint64_t N = offsets ? offsets[n_bags] : n_bags;
  s->occ_row.resize(N);
  s->occ_bag.resize(N);
  s->bag_len.resize(n_bags);
  for (uint64_t b = 0; b < n_bags; ++b) {  // index probe (serial: std::unordered_map)
    const uint32_t table = s->slot_table[b % S];
    const uint64_t lo = offsets ? offsets[b] : b, hi = offsets ? offsets[b + 1] : b + 1;
    s->bag_len[b] = static_cast<uint32_t>(hi - lo);
    for (uint64_t i = lo; i < hi; ++i) {
      s->occ_row[i] = s->touch(table, keys[i]);
      s->occ_bag[i] = static_cast<uint32_t>(b);
    }
  }
  const float* W = s->w.data();
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(n_threads)
#endif
  for (int64_t b = 0; b < static_cast<int64_t>(n_bags); ++b) {
    const uint64_t lo = offsets ? offsets[b] : b, hi = offsets ? offsets[b + 1] : b + 1;
    float* o = out + b * D;
    for (uint32_t j = 0; j < D; ++j) o[j] = 0.0f;
    for (uint64_t i = lo; i < hi; ++i) {
      const float* src = W + s->occ_row[i] * D;
      for (uint32_t j = 0; j < D; ++j) o[j] = o[j] + src[j];
    }
    if (combiner == 1 && hi > lo) {
      const float fl = static_cast<float>(hi - lo);
      for (uint32_t j = 0; j < D; ++j) o[j] = o[j] / fl;
    }
  }
  OptParams p{opt7[0], opt7[1], opt7[2], opt7[3], opt7[4], opt7[5], opt7[6]};
  reduce_and_update(s->occ_row, s->occ_bag, s->bag_len, combiner == 1, dout, D, s->optimizer, p, n_threads, nullptr,
                    [&](uint64_t r, int k) -> float* {
                      if (k == 0) return &s->w[r * D];
                      if (k == 1) return s->s0.empty() ? nullptr : &s->s0[r * D];
                      return s->s1.empty() ? nullptr : &s->s1[r * D];
                    });
  return 0;
}

}  // extern "C"
