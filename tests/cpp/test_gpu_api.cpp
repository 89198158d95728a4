// C++ host API test on the GPU (hps::gpu wrappers over the C-ABI), mirroring the SPEC's
// hot-cache examples and the table insert/find contract. Exit 0 = pass.
#include <cmath>
#include <cstdio>
#include <vector>

#include <hps/gpu.hpp>

#define REQUIRE(c)                                                        \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                           \
    }                                                                     \
  } while (0)

static hps::EmbeddingVector vec(float a, uint16_t dim = 4) {
  std::vector<float> v(dim);
  for (uint16_t j = 0; j < dim; ++j) v[j] = a + j;
  return hps::EmbeddingVector::f32(v);
}

int main() {
  hps::gpu::Context ctx(0);
  // ---- hot cache ----
  hps::gpu::HotCache cache(ctx, hps::TableMeta::make("ads", 4), 64);
  std::vector<hps::EmbeddingKey> k123{1, 2, 3};
  auto r = cache.query(k123);
  REQUIRE(r.found.empty() && r.missing == k123);
  std::vector<hps::VersionedEntry> e7{{7, vec(1.f), 3}};
  REQUIRE(cache.insert(e7) == 1);
  std::vector<hps::EmbeddingKey> k7{7};
  r = cache.query(k7);
  REQUIRE(r.found.size() == 1 && r.found[0].first == 7 && r.found[0].second == vec(1.f));
  std::vector<hps::VersionedEntry> newer{{7, vec(5.f), 5}}, older{{7, vec(9.f), 4}}, absent{{8, vec(0.f), 9}};
  REQUIRE(cache.refresh(newer) == 1);
  REQUIRE(cache.refresh(older) == 0);
  REQUIRE(cache.refresh(absent) == 0);
  r = cache.query(k7);
  REQUIRE(r.found[0].second == vec(5.f));
  auto s = cache.stats();
  REQUIRE(s.queries == 5 && s.hits + s.misses == s.queries && s.hits == 2);
  REQUIRE(cache.size() == 1);
  // an encoded UpdateBatch frame refreshes resident keys at version = seq
  {
    const uint64_t fk[2] = {7, 12345};
    std::vector<float> fv(8);
    for (int j = 0; j < 8; ++j) fv[j] = 40.f + j;
    uint64_t len = 0;
    REQUIRE(hps_update_batch_encode("ads", 3, /*seq=*/9, 2, 4, 0, fk, fv.data(), nullptr, 0, &len) == 0);
    REQUIRE(len == 25 + 2 * (8 + 16));
    std::vector<std::byte> frame(len);
    REQUIRE(hps_update_batch_encode("ads", 3, 9, 2, 4, 0, fk, fv.data(), reinterpret_cast<uint8_t*>(frame.data()), len,
                                    &len) == 0);
    REQUIRE(cache.apply_update(frame) == 1);  // key 7 (version 5 -> 9); 12345 is not resident
    r = cache.query(k7);
    REQUIRE(r.found[0].second == vec(40.f));
    frame[0] = std::byte{0};  // bad magic
    try {
      cache.apply_update(frame);
      REQUIRE(false);
    } catch (const hps::Error& e) {
      REQUIRE(e.code() == hps::ErrorCode::BadMagic);
    }
  }
  // a dim mismatch is a DimMismatch, like the reference's entry validation
  std::vector<hps::VersionedEntry> bad{{9, vec(0.f, 8), 1}};
  try {
    cache.insert(bad);
    REQUIRE(false);
  } catch (const hps::Error& e) {
    REQUIRE(e.code() == hps::ErrorCode::DimMismatch);
  }
  // ---- F16 table: rows held as binary16 on the device ----
  {
    hps::gpu::HotCache c16(ctx, hps::TableMeta::make("h", 4, hps::Dtype::F16), 64);
    const std::vector<uint16_t> bits{0x3c00, 0xbc00, 0x3555, 0x7bff};  // 1, -1, ~1/3, 65504
    std::vector<hps::VersionedEntry> e{{5, hps::EmbeddingVector::f16(bits), 1}};
    REQUIRE(c16.insert(e) == 1);
    std::vector<hps::EmbeddingKey> k5{5};
    auto r16 = c16.query(k5);
    REQUIRE(r16.found.size() == 1 && r16.found[0].second == hps::EmbeddingVector::f16(bits));
    std::vector<hps::VersionedEntry> wrong{{6, vec(1.f), 1}};  // an F32 vector for an F16 table
    try {
      c16.insert(wrong);
      REQUIRE(false);
    } catch (const hps::Error& ex) {
      REQUIRE(ex.code() == hps::ErrorCode::DtypeMismatch);
    }
  }
  // ---- embedding table ----
  std::vector<hps::TableMeta> metas{hps::TableMeta::make("a", 4), hps::TableMeta::make("b", 4)};
  hps::gpu::EmbeddingTable tbl(ctx, metas, {100, 10}, {0, 1});
  std::vector<hps::EmbeddingKey> keys{5, 6, 5, 0xffffffffffffffffull};
  auto rows = tbl.insert(0, keys);
  REQUIRE(rows[0] == 0 && rows[1] == 1 && rows[2] == 0 && rows[3] == 2 && tbl.size(0) == 3);
  auto found = tbl.find(0, keys);
  REQUIRE(found[0].has_value() && found[3].has_value());
  std::vector<hps::EmbeddingKey> none{5};
  REQUIRE(!tbl.find(1, none)[0].has_value());  // separate namespace
  std::vector<hps::VersionedEntry> ents{{11, vec(2.f), 0}};
  tbl.insert(1, ents);
  REQUIRE(tbl.find(1, std::vector<hps::EmbeddingKey>{11})[0].value() == vec(2.f));
  // capacity exhaustion surfaces as Infeasible and leaves the table unchanged
  std::vector<hps::EmbeddingKey> many;
  for (uint64_t i = 100; i < 120; ++i) many.push_back(i);
  try {
    tbl.insert(1, many);
    REQUIRE(false);
  } catch (const hps::Error& e) {
    REQUIRE(e.code() == hps::ErrorCode::Infeasible);
  }
  REQUIRE(tbl.size(1) == 1);
  std::printf("hps::gpu C++ API test passed\n");
  return 0;
}
