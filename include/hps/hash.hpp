// hps/hash.hpp — the placement authority, usable from host C++20 and from sm_100a device code.
//
// Same declarations and bit-exact results as the reference
// (proj/include/hps/hash.hpp:27-54): FNV-1a 64 over the little-endian key bytes.
// key_hash / partition_of are additionally __host__ __device__ so the CUDA
// kernels (table home slot, cache set, destination shard) call the very same
// definition; the reference's `u64 % n` is kept as a true 64-bit modulo (the
// device side uses hps::FastMod64, an exact multiply-high division, verified
// against % in tests/test_hash_golden.py).
#pragma once

#include <cstddef>
#include <cstdint>
#if !defined(__CUDACC_RTC__)
#include <span>
#endif

#include <hps/types.hpp>

#if defined(__CUDACC__)
#define HPS_HD __host__ __device__ __forceinline__
#else
#define HPS_HD inline
#endif

namespace hps {

constexpr std::uint64_t kFnv1a64OffsetBasis = 0xcbf29ce484222325ull;
constexpr std::uint64_t kFnv1a64Prime = 0x100000001b3ull;

/// FNV-1a 64 over an arbitrary byte string (host only; used for known-answer tests).
constexpr std::uint64_t fnv1a64(std::span<const std::byte> data) {
  std::uint64_t acc = kFnv1a64OffsetBasis;
  for (std::size_t i = 0; i < data.size(); ++i) {
    acc = (acc ^ static_cast<std::uint64_t>(data[i])) * kFnv1a64Prime;
  }
  return acc;
}

/// FNV-1a 64 of the 8-byte little-endian encoding of `key`. Unrolled: 8 xor/multiply
/// rounds, one per byte, least significant byte first.
HPS_HD constexpr std::uint64_t key_hash(EmbeddingKey key) {
  std::uint64_t acc = kFnv1a64OffsetBasis;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (unsigned shift = 0; shift < 64; shift += 8) {
    acc = (acc ^ ((key >> shift) & 0xffull)) * kFnv1a64Prime;
  }
  return acc;
}

/// Hash partition of `key` among `num_shards` shards: key_hash(key) mod num_shards,
/// computed in 64 bits and then narrowed. num_shards == 0 is a caller error (as in the
/// reference, which does not guard it).
HPS_HD constexpr std::uint32_t partition_of(EmbeddingKey key, std::uint32_t num_shards) {
  return static_cast<std::uint32_t>(key_hash(key) % num_shards);
}

/// Exact u64 % d for a runtime divisor d >= 1 without the software 64-bit division
/// (~70 instructions on the GPU): Lemire's direct remainder with a 128-bit magic
/// M = ceil(2^128 / d), exact for every 64-bit numerator and divisor. Used for cache
/// set indices (key_hash mod num_sets) and non-power-of-two shard counts.
struct FastMod64 {
  std::uint64_t m_hi = 0, m_lo = 0;  // M = ceil(2^128 / d) (mod 2^128)
  std::uint64_t d = 1;

  FastMod64() = default;
  explicit FastMod64(std::uint64_t divisor) : d(divisor) {
    // M = floor((2^128 - 1) / d) + 1 computed with 128-bit host arithmetic.
    unsigned __int128 all_ones = ~static_cast<unsigned __int128>(0);
    unsigned __int128 m = all_ones / divisor + 1;
    m_hi = static_cast<std::uint64_t>(m >> 64);
    m_lo = static_cast<std::uint64_t>(m);
  }

  // a mod d = high 64 bits of ((M * a mod 2^128) * d) >> 128 — all in 64-bit limbs.
  HPS_HD std::uint64_t mod(std::uint64_t a) const {
    if (d == 1) return 0;
    // lowbits = (M * a) mod 2^128
    std::uint64_t lo = m_lo * a;
    std::uint64_t hi = mulhi(m_lo, a) + m_hi * a;
    // result = floor(lowbits * d / 2^128)
    std::uint64_t t_lo_hi = mulhi(lo, d);  // high part of lo*d
    std::uint64_t p_lo = hi * d;
    std::uint64_t p_hi = mulhi(hi, d);
    std::uint64_t sum = p_lo + t_lo_hi;
    p_hi += (sum < p_lo) ? 1u : 0u;
    return p_hi;
  }

  HPS_HD static std::uint64_t mulhi(std::uint64_t a, std::uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
  }
};

}  // namespace hps
