// tiers.cpp — the lower tiers of the miss path:
//
//   VDB (L2)  sharded in-memory store: shard = partition_of(key, num_shards)
//        (proj/include/hps/hash.hpp:52-54), bounded per-shard capacity with an explicit overflow
//        policy (RejectNew | EvictOldestVersion), version-gated puts (stored iff newer), a
//        shared_mutex per shard (single writer, many readers), shards worked in parallel.
//   PDB (L3)  durable per-table namespaces on disk: <root>/<table>/MANIFEST
//        (dim, dtype, default vector) + numbered append-only log segments of LogRecords
//          key u64 | version u64 | dim u16 | dtype u8 | payload dim x f32 | crc32c u32
//        (little-endian; the checksum is CRC-32C over the preceding record bytes — the
//        reference's crc32c, proj/src/kernels/kernels_scalar.cpp:89-108, SSE4.2 crc32 here);
//        open() rebuilds a key -> (segment, offset, version) index keeping the highest version,
//        drops (and truncates) a torn tail of the LAST segment with a warning count, and fails
//        with Corruption on a bad record anywhere else; put appends iff newer; segments rotate
//        at 64 MiB with a file flush; compact() rewrites the latest versions into fresh segments.
//
// Host code: these tiers live in CPU memory and on disk by definition (the paper's VDB is
// Redis, its PDB RocksDB); the GPU reaches them through the tiered orchestrator (tiered.cu).
#include <dirent.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <shared_mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "hps/hash.hpp"
#include "hps_gpu.h"

namespace hpsg {
void set_last_error(const std::string& msg);
}
using hpsg::set_last_error;

// ---- CRC-32C (Castagnoli, reflected 0x82F63B78, init/xorout 0xFFFFFFFF) -----------------
namespace {
uint32_t g_crc_table[8][256];
std::once_flag g_crc_once;
void crc_init() {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0x82F63B78u & (0u - (c & 1u)));
    g_crc_table[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; ++i)
    for (int t = 1; t < 8; ++t) g_crc_table[t][i] = (g_crc_table[t - 1][i] >> 8) ^ g_crc_table[0][g_crc_table[t - 1][i] & 255u];
}
__attribute__((target("sse4.2"))) uint32_t crc_hw(uint32_t c, const uint8_t* p, size_t n) {
  uint64_t c64 = c;
  for (; n >= 8; n -= 8, p += 8) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    c64 = __builtin_ia32_crc32di(c64, v);
  }
  c = static_cast<uint32_t>(c64);
  for (; n; --n, ++p) c = __builtin_ia32_crc32qi(c, *p);
  return c;
}
uint32_t crc_sw(uint32_t c, const uint8_t* p, size_t n) {
  for (; n >= 8; n -= 8, p += 8) {
    uint32_t lo, hi;
    std::memcpy(&lo, p, 4);
    std::memcpy(&hi, p + 4, 4);
    lo ^= c;
    c = g_crc_table[7][lo & 255u] ^ g_crc_table[6][(lo >> 8) & 255u] ^ g_crc_table[5][(lo >> 16) & 255u] ^
        g_crc_table[4][lo >> 24] ^ g_crc_table[3][hi & 255u] ^ g_crc_table[2][(hi >> 8) & 255u] ^
        g_crc_table[1][(hi >> 16) & 255u] ^ g_crc_table[0][hi >> 24];
  }
  for (; n; --n, ++p) c = (c >> 8) ^ g_crc_table[0][(c ^ *p) & 255u];
  return c;
}
}  // namespace

extern "C" uint32_t hps_crc32c_host(uint32_t crc, const void* data, size_t len) {
  std::call_once(g_crc_once, crc_init);
  static const bool hw = __builtin_cpu_supports("sse4.2");
  const uint32_t c = ~crc;
  return ~(hw ? crc_hw(c, static_cast<const uint8_t*>(data), len) : crc_sw(c, static_cast<const uint8_t*>(data), len));
}

// ---- VDB ---------------------------------------------------------------------------------
namespace {
struct VdbShard {
  mutable std::shared_mutex mu;
  std::unordered_map<uint64_t, uint32_t> index;  // key -> slot
  std::vector<uint64_t> keys, versions;
  std::vector<float> vecs;                       // [slots x dim]
  std::vector<uint32_t> free_slots;
  std::set<std::pair<uint64_t, uint64_t>> by_version;  // (version, key): EvictOldestVersion
};

// Workers over `n` independent items (shards): min(n, hardware threads) threads, or the
// calling thread alone when the batch is small (`work` entries: thread start-up would cost
// more than the shards' work — a lookup's few misses).
template <class F>
void parallel_for(size_t n, F&& f, uint64_t work) {
  const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
  const size_t T = work < 16384 ? 1 : std::min(n, hw);
  if (T <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (size_t t = 0; t < T; ++t)
    th.emplace_back([&, t]() {
      for (size_t i = t; i < n; i += T) f(i);
    });
  for (auto& x : th) x.join();
}
}  // namespace

struct hps_vdb_s {
  uint32_t num_shards = 1, dim = 0;
  uint64_t cap = 0;
  int policy = HPS_VDB_REJECT_NEW;
  std::vector<std::unique_ptr<VdbShard>> shards;
};

namespace {
// Entries of a batch grouped by shard, each group in input order (sequential semantics per key).
std::vector<std::vector<uint32_t>> by_shard(const hps_vdb_s* v, const uint64_t* keys, uint64_t n) {
  std::vector<std::vector<uint32_t>> g(v->num_shards);
  for (uint64_t i = 0; i < n; ++i) g[hps::partition_of(keys[i], v->num_shards)].push_back(static_cast<uint32_t>(i));
  return g;
}
}  // namespace

extern "C" {

int hps_vdb_create(uint32_t num_shards, uint64_t per_shard_capacity, int overflow_policy, uint32_t dim, hps_vdb* out) {
  if (!out || num_shards == 0 || per_shard_capacity == 0 || per_shard_capacity >= (1ull << 32) || dim == 0 ||
      dim > 4096 || (overflow_policy != HPS_VDB_REJECT_NEW && overflow_policy != HPS_VDB_EVICT_OLDEST_VERSION)) {
    set_last_error("vdb: need num_shards >= 1, 1 <= per_shard_capacity < 2^32, 1 <= dim <= 4096, a known policy");
    return HPS_GPU_E_INVALID_ARGUMENT;
  }
  auto v = new hps_vdb_s;
  v->num_shards = num_shards;
  v->cap = per_shard_capacity;
  v->policy = overflow_policy;
  v->dim = dim;
  for (uint32_t s = 0; s < num_shards; ++s) v->shards.emplace_back(new VdbShard);
  *out = v;
  return HPS_GPU_OK;
}

int hps_vdb_destroy(hps_vdb v) {
  delete v;
  return HPS_GPU_OK;
}

int hps_vdb_put_batch(hps_vdb v, const uint64_t* keys, const float* vecs, const uint64_t* versions, uint64_t n,
                      uint64_t* stored_out) {
  if (!v || (n && (!keys || !vecs || !versions))) return HPS_GPU_E_INVALID_ARGUMENT;
  const auto groups = by_shard(v, keys, n);
  std::vector<uint64_t> stored(v->num_shards, 0);
  const uint32_t D = v->dim;
  parallel_for(v->num_shards, [&](size_t s) {
    VdbShard& sh = *v->shards[s];
    std::unique_lock<std::shared_mutex> lk(sh.mu);
    for (uint32_t i : groups[s]) {
      const uint64_t k = keys[i], ver = versions[i];
      auto it = sh.index.find(k);
      uint32_t slot;
      if (it != sh.index.end()) {
        slot = it->second;
        if (ver <= sh.versions[slot]) continue;  // stored iff newer
        sh.by_version.erase({sh.versions[slot], k});
      } else {
        if (sh.index.size() >= v->cap) {
          if (v->policy == HPS_VDB_REJECT_NEW || sh.by_version.empty()) continue;
          const auto oldest = *sh.by_version.begin();  // the resident entry with the smallest version
          sh.by_version.erase(sh.by_version.begin());
          const uint32_t vs = sh.index[oldest.second];
          sh.index.erase(oldest.second);
          sh.free_slots.push_back(vs);
        }
        if (!sh.free_slots.empty()) {
          slot = sh.free_slots.back();
          sh.free_slots.pop_back();
        } else {
          slot = static_cast<uint32_t>(sh.keys.size());
          sh.keys.push_back(0);
          sh.versions.push_back(0);
          sh.vecs.resize(sh.vecs.size() + D);
        }
        sh.index.emplace(k, slot);
      }
      sh.keys[slot] = k;
      sh.versions[slot] = ver;
      std::memcpy(&sh.vecs[size_t(slot) * D], vecs + size_t(i) * D, D * sizeof(float));
      sh.by_version.insert({ver, k});
      ++stored[s];
    }
  }, n);
  if (stored_out) {
    uint64_t t = 0;
    for (uint64_t x : stored) t += x;
    *stored_out = t;
  }
  return HPS_GPU_OK;
}

// found[i] = 1 and (vecs, versions)[i] filled for resident keys; no side effects.
int hps_vdb_get_batch(hps_vdb v, const uint64_t* keys, uint64_t n, float* vecs_out, uint64_t* versions_out,
                      uint8_t* found_out, uint64_t* n_found_out) {
  if (!v || (n && (!keys || !found_out))) return HPS_GPU_E_INVALID_ARGUMENT;
  const auto groups = by_shard(v, keys, n);
  std::vector<uint64_t> nf(v->num_shards, 0);
  const uint32_t D = v->dim;
  parallel_for(v->num_shards, [&](size_t s) {
    const VdbShard& sh = *v->shards[s];
    std::shared_lock<std::shared_mutex> lk(sh.mu);
    for (uint32_t i : groups[s]) {
      auto it = sh.index.find(keys[i]);
      found_out[i] = it != sh.index.end();
      if (!found_out[i]) continue;
      ++nf[s];
      if (vecs_out) std::memcpy(vecs_out + size_t(i) * D, &sh.vecs[size_t(it->second) * D], D * sizeof(float));
      if (versions_out) versions_out[i] = sh.versions[it->second];
    }
  }, n);
  if (n_found_out) {
    uint64_t t = 0;
    for (uint64_t x : nf) t += x;
    *n_found_out = t;
  }
  return HPS_GPU_OK;
}

// A point-in-time listing of shard `idx`, ascending by key. *n_out = entries; with cap below
// it only the count is returned (call again with room).
int hps_vdb_shard_snapshot(hps_vdb v, uint32_t idx, uint64_t* keys, float* vecs, uint64_t* versions, uint64_t cap,
                           uint64_t* n_out) {
  if (!v || !n_out) return HPS_GPU_E_INVALID_ARGUMENT;
  if (idx >= v->num_shards) return HPS_GPU_E_BAD_SHARD;
  const VdbShard& sh = *v->shards[idx];
  std::shared_lock<std::shared_mutex> lk(sh.mu);
  *n_out = sh.index.size();
  if (cap < sh.index.size() || sh.index.empty()) return HPS_GPU_OK;
  if (!keys) return HPS_GPU_E_INVALID_ARGUMENT;
  std::vector<std::pair<uint64_t, uint32_t>> e(sh.index.begin(), sh.index.end());
  std::sort(e.begin(), e.end());
  for (size_t j = 0; j < e.size(); ++j) {
    keys[j] = e[j].first;
    if (versions) versions[j] = sh.versions[e[j].second];
    if (vecs) std::memcpy(vecs + j * v->dim, &sh.vecs[size_t(e[j].second) * v->dim], v->dim * sizeof(float));
  }
  return HPS_GPU_OK;
}

int hps_vdb_size(hps_vdb v, uint64_t* n_out) {
  if (!v || !n_out) return HPS_GPU_E_INVALID_ARGUMENT;
  uint64_t t = 0;
  for (auto& s : v->shards) {
    std::shared_lock<std::shared_mutex> lk(s->mu);
    t += s->index.size();
  }
  *n_out = t;
  return HPS_GPU_OK;
}

}  // extern "C"

// ---- PDB ---------------------------------------------------------------------------------
namespace {
constexpr char kManifestMagic[8] = {'H', 'P', 'S', 'P', 'D', 'B', '1', '\0'};
constexpr size_t kRecHead = 8 + 8 + 2 + 1;  // key, version, dim, dtype
constexpr uint8_t kDtypeF32 = 0;

struct PdbLoc {
  uint32_t seg;      // index into Table::segs
  uint64_t off;      // record start
  uint64_t version;
};
struct PdbSeg {
  uint32_t num = 0;
  int fd = -1;
  uint64_t size = 0;
};
struct PdbTable {
  std::string name, dir;
  uint32_t dim = 0;
  std::vector<float> default_vec;  // empty: zeros
  std::vector<PdbSeg> segs;
  std::unordered_map<uint64_t, PdbLoc> index;
  mutable std::shared_mutex mu;
  size_t rec_bytes() const { return kRecHead + 4ull * dim + 4; }
};

std::string seg_path(const PdbTable& t, uint32_t num) {
  char b[32];
  std::snprintf(b, sizeof(b), "seg_%08u.log", num);
  return t.dir + "/" + b;
}

bool write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::write(fd, c, n);
    if (w <= 0) return false;
    c += w;
    n -= static_cast<size_t>(w);
  }
  return true;
}

bool read_file(const std::string& path, std::vector<uint8_t>* out) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) return false;
  struct stat st;
  if (fstat(fd, &st) != 0) {
    ::close(fd);
    return false;
  }
  out->resize(static_cast<size_t>(st.st_size));
  size_t got = 0;
  while (got < out->size()) {
    const ssize_t r = ::pread(fd, out->data() + got, out->size() - got, static_cast<off_t>(got));
    if (r <= 0) break;
    got += static_cast<size_t>(r);
  }
  ::close(fd);
  return got == out->size();
}

void encode_record(uint8_t* p, uint64_t key, uint64_t version, uint32_t dim, const float* vec) {
  std::memcpy(p, &key, 8);
  std::memcpy(p + 8, &version, 8);
  const uint16_t d16 = static_cast<uint16_t>(dim);
  std::memcpy(p + 16, &d16, 2);
  p[18] = kDtypeF32;
  std::memcpy(p + kRecHead, vec, 4ull * dim);
  const uint32_t crc = hps_crc32c_host(0, p, kRecHead + 4ull * dim);
  std::memcpy(p + kRecHead + 4ull * dim, &crc, 4);
}

bool valid_name(const char* name) {
  if (!name || !*name) return false;
  const std::string s(name);
  if (s == "." || s == ".." || s.size() > 255) return false;
  return s.find('/') == std::string::npos && s.find('\0') == std::string::npos;
}
}  // namespace

struct hps_pdb_s {
  std::string root;
  uint64_t seg_limit = 64ull << 20;
  bool sync_every_batch = false;
  uint64_t dropped_tail = 0;
  std::mutex tables_mu;
  std::map<std::string, std::unique_ptr<PdbTable>> tables;
};

namespace {
int open_segment_for_append(PdbTable& t, uint32_t num) {
  const std::string p = seg_path(t, num);
  const int fd = ::open(p.c_str(), O_RDWR | O_CREAT | O_APPEND, 0644);
  if (fd < 0) {
    set_last_error("pdb: cannot open segment " + p);
    return HPS_GPU_E_IO;
  }
  struct stat st;
  fstat(fd, &st);
  t.segs.push_back(PdbSeg{num, fd, static_cast<uint64_t>(st.st_size)});
  return HPS_GPU_OK;
}

// Rebuild a table's index from its segments (open): highest version per key.
int load_table(hps_pdb_s* db, PdbTable& t) {
  std::vector<uint8_t> m;
  if (!read_file(t.dir + "/MANIFEST", &m) || m.size() < 8 + 4 + 1 + 1 || std::memcmp(m.data(), kManifestMagic, 8) != 0) {
    set_last_error("pdb: unreadable manifest in " + t.dir);
    return HPS_GPU_E_IO;
  }
  std::memcpy(&t.dim, m.data() + 8, 4);
  const uint8_t dtype = m[12], has_def = m[13];
  if (dtype != kDtypeF32 || t.dim == 0 || t.dim > 4096 || m.size() != 14 + (has_def ? 4ull * t.dim : 0)) {
    set_last_error("pdb: malformed manifest in " + t.dir);
    return HPS_GPU_E_IO;
  }
  if (has_def) {
    t.default_vec.resize(t.dim);
    std::memcpy(t.default_vec.data(), m.data() + 14, 4ull * t.dim);
  }
  std::vector<uint32_t> nums;
  if (DIR* d = ::opendir(t.dir.c_str())) {
    while (dirent* e = ::readdir(d)) {
      unsigned num;
      char tail;
      if (std::sscanf(e->d_name, "seg_%8u.lo%c", &num, &tail) == 2 && tail == 'g') nums.push_back(num);
    }
    ::closedir(d);
  }
  std::sort(nums.begin(), nums.end());
  const size_t R = t.rec_bytes();
  for (size_t si = 0; si < nums.size(); ++si) {
    const bool last = si + 1 == nums.size();
    std::vector<uint8_t> buf;
    if (!read_file(seg_path(t, nums[si]), &buf)) {
      set_last_error("pdb: cannot read " + seg_path(t, nums[si]));
      return HPS_GPU_E_IO;
    }
    uint64_t off = 0;
    bool torn = false;
    while (off < buf.size()) {
      bool ok = buf.size() - off >= R;
      if (ok) {
        uint16_t d16;
        std::memcpy(&d16, buf.data() + off + 16, 2);
        uint32_t crc;
        std::memcpy(&crc, buf.data() + off + R - 4, 4);
        ok = d16 == t.dim && buf[off + 18] == kDtypeF32 && crc == hps_crc32c_host(0, buf.data() + off, R - 4);
      }
      if (!ok) {
        if (!last) {
          set_last_error("pdb: corrupt record inside " + seg_path(t, nums[si]) + " (not its tail)");
          return HPS_GPU_E_CORRUPTION;
        }
        torn = true;  // crash semantics: a torn tail of the newest segment is dropped
        break;
      }
      uint64_t key, ver;
      std::memcpy(&key, buf.data() + off, 8);
      std::memcpy(&ver, buf.data() + off + 8, 8);
      auto it = t.index.find(key);
      if (it == t.index.end() || ver > it->second.version)
        t.index[key] = PdbLoc{static_cast<uint32_t>(t.segs.size()), off, ver};
      off += R;
    }
    if (int s = open_segment_for_append(t, nums[si])) return s;
    if (torn) {
      ++db->dropped_tail;
      if (::ftruncate(t.segs.back().fd, static_cast<off_t>(off)) != 0) return HPS_GPU_E_IO;
      t.segs.back().size = off;
    }
  }
  if (t.segs.empty())
    if (int s = open_segment_for_append(t, 0)) return s;
  return HPS_GPU_OK;
}

PdbTable* find_table(hps_pdb db, const char* name) {
  if (!db || !name) return nullptr;
  std::lock_guard<std::mutex> lk(db->tables_mu);
  auto it = db->tables.find(name);
  return it == db->tables.end() ? nullptr : it->second.get();
}

void close_table(PdbTable& t) {
  for (auto& s : t.segs)
    if (s.fd >= 0) {
      ::fdatasync(s.fd);
      ::close(s.fd);
      s.fd = -1;
    }
}
}  // namespace

extern "C" {

int hps_pdb_open(const char* root, hps_pdb* out, uint64_t* dropped_tail_out) {
  if (!root || !*root || !out) return HPS_GPU_E_INVALID_ARGUMENT;
  *out = nullptr;
  ::mkdir(root, 0755);
  struct stat st;
  if (::stat(root, &st) != 0 || !S_ISDIR(st.st_mode)) {
    set_last_error(std::string("pdb: root is not a directory: ") + root);
    return HPS_GPU_E_IO;
  }
  auto db = new hps_pdb_s;
  db->root = root;
  if (const char* e = std::getenv("HPS_PDB_SEGMENT_BYTES")) db->seg_limit = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  std::vector<std::string> names;
  if (DIR* d = ::opendir(root)) {
    while (dirent* e = ::readdir(d)) {
      const std::string n = e->d_name;
      if (n == "." || n == "..") continue;
      if (::stat((db->root + "/" + n + "/MANIFEST").c_str(), &st) == 0) names.push_back(n);
    }
    ::closedir(d);
  }
  std::sort(names.begin(), names.end());
  for (const auto& n : names) {
    auto t = std::make_unique<PdbTable>();
    t->name = n;
    t->dir = db->root + "/" + n;
    if (int s = load_table(db, *t)) {
      close_table(*t);
      hps_pdb_close(db);
      return s;
    }
    db->tables.emplace(n, std::move(t));
  }
  if (dropped_tail_out) *dropped_tail_out = db->dropped_tail;
  *out = db;
  return HPS_GPU_OK;
}

int hps_pdb_close(hps_pdb db) {
  if (!db) return HPS_GPU_OK;
  for (auto& kv : db->tables) close_table(*kv.second);
  delete db;
  return HPS_GPU_OK;
}

int hps_pdb_table_count(hps_pdb db, uint64_t* n_out) {
  if (!db || !n_out) return HPS_GPU_E_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(db->tables_mu);
  *n_out = db->tables.size();
  return HPS_GPU_OK;
}

// Registers a table namespace (manifest written and flushed before any segment). An existing
// table with the same dim is kept as it is; a different dim -> DimMismatch.
int hps_pdb_create_table(hps_pdb db, const char* name, uint32_t dim, const float* default_vec) {
  if (!db || !valid_name(name) || dim == 0 || dim > 4096) return HPS_GPU_E_INVALID_ARGUMENT;
  if (PdbTable* t = find_table(db, name)) return t->dim == dim ? HPS_GPU_OK : HPS_GPU_E_DIM_MISMATCH;
  auto t = std::make_unique<PdbTable>();
  t->name = name;
  t->dir = db->root + "/" + name;
  t->dim = dim;
  if (default_vec) t->default_vec.assign(default_vec, default_vec + dim);
  ::mkdir(t->dir.c_str(), 0755);
  std::vector<uint8_t> m(14 + (default_vec ? 4ull * dim : 0));
  std::memcpy(m.data(), kManifestMagic, 8);
  std::memcpy(m.data() + 8, &dim, 4);
  m[12] = kDtypeF32;
  m[13] = default_vec ? 1 : 0;
  if (default_vec) std::memcpy(m.data() + 14, default_vec, 4ull * dim);
  const std::string tmp = t->dir + "/MANIFEST.tmp";
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0 || !write_all(fd, m.data(), m.size()) || ::fsync(fd) != 0) {
    if (fd >= 0) ::close(fd);
    set_last_error("pdb: cannot write manifest in " + t->dir);
    return HPS_GPU_E_IO;
  }
  ::close(fd);
  if (::rename(tmp.c_str(), (t->dir + "/MANIFEST").c_str()) != 0) return HPS_GPU_E_IO;
  if (int s = open_segment_for_append(*t, 0)) return s;
  std::lock_guard<std::mutex> lk(db->tables_mu);
  db->tables.emplace(name, std::move(t));
  return HPS_GPU_OK;
}

// Appends a LogRecord per entry whose version is newer than the key's latest (in input order,
// so a batch holding a key twice keeps the newer); the index follows.
int hps_pdb_put_batch(hps_pdb db, const char* table, const uint64_t* keys, const float* vecs, const uint64_t* versions,
                      uint64_t n, uint64_t* stored_out) {
  PdbTable* t = find_table(db, table);
  if (!t) return db && table ? HPS_GPU_E_UNKNOWN_TABLE : HPS_GPU_E_INVALID_ARGUMENT;
  if (n && (!keys || !vecs || !versions)) return HPS_GPU_E_INVALID_ARGUMENT;
  std::unique_lock<std::shared_mutex> lk(t->mu);
  const size_t R = t->rec_bytes();
  std::vector<uint8_t> buf;
  uint64_t stored = 0;
  auto flush = [&]() -> int {
    if (buf.empty()) return HPS_GPU_OK;
    PdbSeg& s = t->segs.back();
    if (!write_all(s.fd, buf.data(), buf.size())) {
      set_last_error("pdb: write failed in " + t->dir);
      return HPS_GPU_E_IO;
    }
    s.size += buf.size();
    buf.clear();
    if (db->sync_every_batch) ::fdatasync(s.fd);
    return HPS_GPU_OK;
  };
  for (uint64_t i = 0; i < n; ++i) {
    auto it = t->index.find(keys[i]);
    if (it != t->index.end() && versions[i] <= it->second.version) continue;  // stale
    if (t->segs.back().size + buf.size() + R > db->seg_limit && t->segs.back().size + buf.size() > 0) {
      if (int s = flush()) return s;
      ::fdatasync(t->segs.back().fd);  // file-level flush at rotation
      if (int s = open_segment_for_append(*t, t->segs.back().num + 1)) return s;
    }
    const uint64_t off = t->segs.back().size + buf.size();
    buf.resize(buf.size() + R);
    encode_record(buf.data() + buf.size() - R, keys[i], versions[i], t->dim, vecs + size_t(i) * t->dim);
    t->index[keys[i]] = PdbLoc{static_cast<uint32_t>(t->segs.size() - 1), off, versions[i]};
    ++stored;
  }
  if (int s = flush()) return s;
  if (stored_out) *stored_out = stored;
  return HPS_GPU_OK;
}

// found[i] = 1 and (vecs, versions)[i] = the latest record of keys[i] (read from its segment).
int hps_pdb_get_batch(hps_pdb db, const char* table, const uint64_t* keys, uint64_t n, float* vecs_out,
                      uint64_t* versions_out, uint8_t* found_out, uint64_t* n_found_out) {
  PdbTable* t = find_table(db, table);
  if (!t) return db && table ? HPS_GPU_E_UNKNOWN_TABLE : HPS_GPU_E_INVALID_ARGUMENT;
  if (n && (!keys || !found_out)) return HPS_GPU_E_INVALID_ARGUMENT;
  std::shared_lock<std::shared_mutex> lk(t->mu);
  const uint64_t D = t->dim;
  // key chunks on parallel host threads for large batches (index reads + one pread per key;
  // the segments are usually in the page cache, so the syscalls, not the device, bound it)
  constexpr uint64_t kChunkKeys = 512;
  const uint64_t chunks = (n + kChunkKeys - 1) / kChunkKeys;
  std::vector<uint64_t> nf(chunks, 0);
  std::vector<uint8_t> bad(chunks, 0);
  parallel_for(chunks, [&](size_t c) {
    for (uint64_t i = c * kChunkKeys; i < std::min(n, (c + 1) * kChunkKeys); ++i) {
      auto it = t->index.find(keys[i]);
      found_out[i] = it != t->index.end();
      if (!found_out[i]) continue;
      ++nf[c];
      if (versions_out) versions_out[i] = it->second.version;
      if (vecs_out) {
        const PdbSeg& s = t->segs[it->second.seg];
        const ssize_t r = ::pread(s.fd, vecs_out + i * D, 4 * D, static_cast<off_t>(it->second.off + kRecHead));
        if (r != static_cast<ssize_t>(4 * D)) bad[c] = 1;
      }
    }
  }, n >= 2048 ? uint64_t(1) << 20 : 0);
  for (uint8_t b : bad)
    if (b) {
      set_last_error("pdb: short read in " + t->dir);
      return HPS_GPU_E_IO;
    }
  if (n_found_out) {
    uint64_t tot = 0;
    for (uint64_t x : nf) tot += x;
    *n_found_out = tot;
  }
  return HPS_GPU_OK;
}

// The table's default vector (zeros when its manifest has none) into vec_out[dim].
int hps_pdb_table_info(hps_pdb db, const char* table, uint32_t* dim_out, float* default_vec_out, uint64_t* keys_out) {
  PdbTable* t = find_table(db, table);
  if (!t) return db && table ? HPS_GPU_E_UNKNOWN_TABLE : HPS_GPU_E_INVALID_ARGUMENT;
  std::shared_lock<std::shared_mutex> lk(t->mu);
  if (dim_out) *dim_out = t->dim;
  if (keys_out) *keys_out = t->index.size();
  if (default_vec_out) {
    if (t->default_vec.empty())
      std::memset(default_vec_out, 0, 4ull * t->dim);
    else
      std::memcpy(default_vec_out, t->default_vec.data(), 4ull * t->dim);
  }
  return HPS_GPU_OK;
}

// Latest version of every key, ascending by key (a snapshot of the index taken at the call).
// *n_out = keys; with cap below it only the count is returned.
int hps_pdb_scan(hps_pdb db, const char* table, uint64_t* keys, float* vecs, uint64_t* versions, uint64_t cap,
                 uint64_t* n_out) {
  PdbTable* t = find_table(db, table);
  if (!t) return db && table ? HPS_GPU_E_UNKNOWN_TABLE : HPS_GPU_E_INVALID_ARGUMENT;
  if (!n_out) return HPS_GPU_E_INVALID_ARGUMENT;
  std::vector<uint64_t> ks;
  {
    std::shared_lock<std::shared_mutex> lk(t->mu);
    *n_out = t->index.size();
    if (cap < t->index.size() || t->index.empty()) return HPS_GPU_OK;
    for (const auto& kv : t->index) ks.push_back(kv.first);
  }
  if (!keys) return HPS_GPU_E_INVALID_ARGUMENT;
  std::sort(ks.begin(), ks.end());
  std::memcpy(keys, ks.data(), ks.size() * 8);
  std::vector<uint8_t> found(ks.size());
  return hps_pdb_get_batch(db, table, ks.data(), ks.size(), vecs, versions, found.data(), nullptr);
}

// Rewrites the latest version of every key into fresh segments (ascending key order), then
// removes the old ones: *reclaimed_out = old bytes - new bytes. Lookups are unchanged.
int hps_pdb_compact(hps_pdb db, const char* table, uint64_t* reclaimed_out) {
  PdbTable* t = find_table(db, table);
  if (!t) return db && table ? HPS_GPU_E_UNKNOWN_TABLE : HPS_GPU_E_INVALID_ARGUMENT;
  std::unique_lock<std::shared_mutex> lk(t->mu);
  const size_t R = t->rec_bytes();
  uint64_t old_bytes = 0;
  for (const auto& s : t->segs) old_bytes += s.size;
  std::vector<std::pair<uint64_t, PdbLoc>> live(t->index.begin(), t->index.end());
  std::sort(live.begin(), live.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<PdbSeg> old = std::move(t->segs);
  t->segs.clear();
  if (int s = open_segment_for_append(*t, old.back().num + 1)) {
    t->segs = std::move(old);
    return s;
  }
  std::unordered_map<uint64_t, PdbLoc> index;
  std::vector<uint8_t> rec(R), buf;
  for (const auto& kv : live) {
    const PdbSeg& from = old[kv.second.seg];
    if (::pread(from.fd, rec.data(), R, static_cast<off_t>(kv.second.off)) != static_cast<ssize_t>(R)) return HPS_GPU_E_IO;
    if (t->segs.back().size + buf.size() + R > db->seg_limit && t->segs.back().size + buf.size() > 0) {
      if (!write_all(t->segs.back().fd, buf.data(), buf.size())) return HPS_GPU_E_IO;
      t->segs.back().size += buf.size();
      buf.clear();
      ::fdatasync(t->segs.back().fd);
      if (int s = open_segment_for_append(*t, t->segs.back().num + 1)) return s;
    }
    index[kv.first] = PdbLoc{static_cast<uint32_t>(t->segs.size() - 1), t->segs.back().size + buf.size(), kv.second.version};
    buf.insert(buf.end(), rec.begin(), rec.end());
  }
  if (!buf.empty()) {
    if (!write_all(t->segs.back().fd, buf.data(), buf.size())) return HPS_GPU_E_IO;
    t->segs.back().size += buf.size();
  }
  for (const auto& s : t->segs) ::fdatasync(s.fd);
  for (auto& s : old) {
    ::close(s.fd);
    ::unlink(seg_path(*t, s.num).c_str());
  }
  t->index = std::move(index);
  uint64_t new_bytes = 0;
  for (const auto& s : t->segs) new_bytes += s.size;
  if (reclaimed_out) *reclaimed_out = old_bytes > new_bytes ? old_bytes - new_bytes : 0;
  return HPS_GPU_OK;
}

}  // extern "C"
