// philox.cuh -- the method's counter-based RNG on the device.
//
// Algorithm 2 step 1 "randomly select k columns and k rows" is
// realised as Floyd's sampling without replacement driven by Lemire bounded
// integers over a Philox4x32-10 word stream.  Integer only: the result is
// bit-identical to any other implementation of the same specification.
#pragma once
#include <stdint.h>

namespace cabsk {

__device__ __forceinline__ uint4 philox_round(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
  uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
  return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    c = philox_round(c, k);
    k.x += W0;
    k.y += W1;
  }
  return philox_round(c, k);
}

__device__ __forceinline__ uint2 seed_key(uint64_t seed) {
  return make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// Sequential word stream w(q) = Philox((q/4 lo, q/4 hi, tag, 0), key)[q % 4].
struct WordStream {
  uint2 key;
  uint32_t tag;
  uint64_t q;
  uint64_t blk_id;
  uint4 blk;
  __device__ WordStream(uint64_t seed, uint32_t tag_) : key(seed_key(seed)), tag(tag_), q(0), blk_id(~0ull) {}
  __device__ uint32_t next() {
    uint64_t b = q >> 2;
    if (b != blk_id) {
      blk = philox4x32_10(make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32), tag, 0u), key);
      blk_id = b;
    }
    uint32_t i = static_cast<uint32_t>(q & 3);
    ++q;
    return i == 0 ? blk.x : (i == 1 ? blk.y : (i == 2 ? blk.z : blk.w));
  }
};

// Lemire multiply-shift: uniform in [0, s), 1 <= s <= 2^32, rejection draws more words.
__device__ __forceinline__ uint64_t lemire_bounded(WordStream& ws, uint64_t s) {
  for (;;) {
    uint64_t m = static_cast<uint64_t>(ws.next()) * s;
    uint64_t lo = m & 0xFFFFFFFFull;
    if (lo < s) {
      uint64_t thresh = ((1ull << 32) - s) % s;
      if (lo < thresh) continue;
    }
    return m >> 32;
  }
}

}  // namespace cabsk
