// K1: in-register Gaussian generator for G (never stored in HBM).
//
// Definition (DESIGN.md "Readings" C9; the paper's G = randn(s, m), Alg. 1 step 2,
// P:483-485, and G = randn(n, s), Alg. 2 step 2):
//   key = (seed & 0xffffffff, seed >> 32), counter = (i >> 1, lo32(j), hi32(j), 0)
//   o = Philox4x32-10(counter, key)               (Salmon et al., SC'11)
//   u1 = ((w0 >> 11) + 1) 2^-53 in (0,1], u2 = (w1 >> 11) 2^-53 in [0,1),
//   w0 = o.x | o.y << 32, w1 = o.z | o.w << 32
//   G[2q, j] = sqrt(-2 ln u1) cos(2 pi u2),  G[2q+1, j] = sqrt(-2 ln u1) sin(2 pi u2).
// The paper generated G with a threaded Ziggurat on CPUs; a
// counter-based stream lets every CTA (and every GPU) regenerate exactly the
// tile it needs from (seed, i, j), so the sketch is tiling- and shard-invariant.
#pragma once
#include "common.cuh"

namespace lsrn {

LSRN_DEV uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

LSRN_DEV uint2 philox_key(uint64_t seed) {
  return make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// u = (x >> 11) * 2^-53 for a 64-bit word split as (lo, hi), built from the
// bits without an integer->double conversion: with t = x >> 11 (53 bits),
// bit 52 of t chooses between [0.5, 1) (exact bit pattern) and [0, 0.5)
// (the same pattern minus 0.5, exact by Sterbenz).
LSRN_DEV double u53_from_words(uint32_t lo, uint32_t hi) {
  // t = (hi:lo) >> 11; t52 = bit 63 of x; mantissa bits = bits 62..11 of x
  const uint32_t mant_hi = (hi >> 11) & 0xFFFFFu;           // x bits 62..43 -> 20 bits
  const uint32_t mant_lo = (lo >> 11) | (hi << 21);         // x bits 42..11 -> 32 bits
  const double half_plus = __hiloint2double(static_cast<int>(0x3FE00000u | mant_hi),
                                            static_cast<int>(mant_lo));  // 0.5 + mant * 2^-53
  return (hi & 0x80000000u) ? half_plus : (half_plus - 0.5);
}

// Box-Muller pair for Philox output o.
LSRN_DEV void box_muller(uint4 o, double& z0, double& z1) {
  const double u2 = u53_from_words(o.z, o.w);
  const double u1 = u53_from_words(o.x, o.y) + 0x1.0p-53;   // ((w0>>11)+1) 2^-53, exact
  const double rho = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  z0 = rho * cs;
  z1 = rho * sn;
}

// The normal pair (G[2q, j], G[2q+1, j]).
LSRN_DEV void gaussian_pair(uint2 key, uint64_t q, uint64_t j, double& z0, double& z1) {
  const uint4 o = philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(j),
                                           static_cast<uint32_t>(j >> 32), 0u), key);
  box_muller(o, z0, z1);
}

}  // namespace lsrn
