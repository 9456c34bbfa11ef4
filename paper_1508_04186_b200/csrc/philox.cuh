// philox.cuh — device Philox4x32-10 and the integer-only slot mapping of the
// replay sampler (a1; A11). Independent of the oracle's implementation; both
// follow Salmon et al. (Random123) and are checked against its known answers.
#pragma once
#include <cstdint>

namespace dqn {

__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                              uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// slot = floor(u * size / 2^64), u = x0:x1 of Philox(ctr = (j, T_lo, T_hi, rank), key = seed)
__device__ __forceinline__ long long sample_slot(unsigned long long seed, unsigned rank, unsigned long long T,
                                                 unsigned j, long long size) {
  uint32_t c0 = j, c1 = (uint32_t)T, c2 = (uint32_t)(T >> 32), c3 = rank;
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const unsigned long long u = ((unsigned long long)c0 << 32) | c1;
  return (long long)__umul64hi(u, (unsigned long long)size);
}

}  // namespace dqn
