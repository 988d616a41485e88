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
#include "bm_int_tables.h"
#include "bm_tables.h"
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

// Box-Muller pair for Philox output o with CUDA's libm (log, sqrt, sincospi):
// about 77 FP64-pipe instructions per pair on sm_100a.  Kept as the reference
// implementation for lsrn_debug_box_muller (tests compare the two).
LSRN_DEV void box_muller_libm(uint4 o, double& z0, double& z1) {
  const double u2 = u53_from_words(o.z, o.w);
  const double u1 = u53_from_words(o.x, o.y) + 0x1.0p-53;   // ((w0>>11)+1) 2^-53, exact
  const double rho = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  z0 = rho * cs;
  z1 = rho * sn;
}

// ---- table-driven Box-Muller (K1 v2) -------------------------------------------
// The same transform in ~40 FP64 instructions instead of ~77: the RNG shares the
// FP64 pipe with DMMA in the dense sketch and is the whole cost of the CSR
// sketch.  Tables and coefficients: bm_tables.h (tools/gen_bm_tables.py); the
// caller stages bm::kTable (4 KB) in shared memory (bm_load_table) and passes it.
//
// ln u1, u1 = n 2^-53, n = (w0 >> 11) + 1 in [1, 2^53]:  n = 2^e m, m in [1, 2);
//   i = top 7 bits of m's fraction; r = m invc_i - 1 is exact (invc_i has 9
//   significant bits, |r| < 2^-7); ln u1 = (e - 53) ln2 - ln(invc_i) + log1p(r),
//   with ln2 and -ln(invc_i) as 42-bit heads + tails so the head sum is exact;
//   invc_127 = 1/2 makes u1 -> 1 come out as log1p(r) with no cancellation.
// sin / cos (2 pi u2): 4 u2 = k + f (quadrant k, f exact), f = j / 64 + d / 64;
//   table sin / cos (pi/2 j/64), polynomials in d for (pi/128) d, angle addition,
//   quadrant rotation.
// Accuracy (host model of the same operations vs 40-digit references over 3e4
// random and edge words): ln u1 within 1.4e-16 relative, sin / cos within 1.5e-16,
// normals within 4.5e-16 max(1, |z|).

LSRN_DEV void bm_load_table(double* Ts) {
  for (int i = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); i < bm::TAB_SIZE;
       i += blockDim.x * blockDim.y * blockDim.z)
    Ts[i] = bm::kTable[i];
}

// x = -2 ln u1 >= 0 (the square of the Box-Muller radius).  The polynomial is
// evaluated in Estrin form and the -2 is folded into the table terms: the
// transform shares the FP64 pipe with DMMA in the dense sketch, where each
// dependent FP64 instruction waits behind the queued DMMAs, so the length of the
// dependency chain (not the instruction count) sets the producers' rate.
LSRN_DEV double bm_m2ln_u1(uint32_t lo, uint32_t hi, const double* T) {
  const uint64_t w0 = (static_cast<uint64_t>(hi) << 32) | lo;
  const uint64_t n1 = (w0 >> 11) + 1ull;                        // 1 .. 2^53
  const int e = 63 - __clzll(static_cast<long long>(n1));      // 0 .. 53
  const uint64_t mant = (e <= 52) ? ((n1 << (52 - e)) & 0xFFFFFFFFFFFFFull) : 0ull;
  const double m = __longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | mant));
  const int i = static_cast<int>(mant >> 45);
  const double r = fma(m, T[i], -1.0);                          // exact, |r| < 2^-7
  // log1p(r) = r + r^2 p(r), p = C2 + C3 r + ... + C8 r^6 (Estrin)
  const double r2 = r * r;
  const double m2r = -2.0 * r;
  const double a0 = fma(bm::LOG1P_C3, r, bm::LOG1P_C2);
  const double a1 = fma(bm::LOG1P_C5, r, bm::LOG1P_C4);
  const double a2 = fma(bm::LOG1P_C7, r, bm::LOG1P_C6);
  const double r4 = r2 * r2;
  const double q1 = fma(a1, r2, a0);
  const double q2 = fma(bm::LOG1P_C8, r2, a2);
  const double p = fma(q2, r4, q1);
  const double poly = fma(-2.0 * r2, p, m2r);                   // -2 log1p(r)
  const double E = static_cast<double>(e - 53);
  const double thi = fma(E, -2.0 * bm::LN2_HI, -2.0 * T[128 + i]);   // exact (42-bit heads, x2 exact)
  const double tlo = fma(E, -2.0 * bm::LN2_LO, -2.0 * T[256 + i]);
  return thi + (tlo + poly);
}

// ln u1 (kept for reference / tests): -x / 2, exact scaling.
LSRN_DEV double bm_ln_u1(uint32_t lo, uint32_t hi, const double* T) { return -0.5 * bm_m2ln_u1(lo, hi, T); }

LSRN_DEV void bm_sincos_2pi(uint32_t lo, uint32_t hi, const double* T, double& sn, double& cs) {
  const uint64_t w1 = (static_cast<uint64_t>(hi) << 32) | lo;
  const uint64_t n2 = w1 >> 11;                                 // u2 = n2 2^-53
  const int k = static_cast<int>(n2 >> 51);
  const int j = static_cast<int>((n2 >> 45) & 63);
  const uint64_t dm = n2 & ((1ull << 45) - 1);
  const double d = __longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | (dm << 7))) - 1.0;
  const double d2 = d * d;
  const double d4 = d2 * d2;
  // sin b = d (S1 + S3 d^2 + ... + S9 d^8), cos b = 1 + d^2 (C2 + C4 d^2 + ... + C10 d^8) (Estrin)
  const double b0 = fma(bm::SIN_C3, d2, bm::SIN_C1);
  const double b1 = fma(bm::SIN_C7, d2, bm::SIN_C5);
  const double c0 = fma(bm::COS_C4, d2, bm::COS_C2);
  const double c1 = fma(bm::COS_C8, d2, bm::COS_C6);
  const double b1b = fma(bm::SIN_C9, d4, b1);
  const double c1b = fma(bm::COS_C10, d4, c1);
  const double sp = fma(b1b, d4, b0);
  const double cp = fma(c1b, d4, c0);
  const double sb = sp * d;
  const double cb = fma(cp, d2, 1.0);
  const double sa = T[384 + j], ca = T[448 + j];
  const double s = fma(sa, cb, ca * sb);
  const double c = fma(ca, cb, -(sa * sb));
  // rotate by k quarter turns
  sn = (k == 0) ? s : (k == 1) ? c : (k == 2) ? -s : -c;
  cs = (k == 0) ? c : (k == 1) ? -s : (k == 2) ? -c : s;
}

// sqrt(x) for x in [0, 74] with a short chain: y0 = rsqrt.approx (MUFU.RSQ64H),
// s0 = x y0, e = 1 - s0 y0, sqrt(x) = s0 (1 + e/2 + 3 e^2 / 8 + O(e^3)); x = 0 -> 0.
LSRN_DEV double bm_sqrt(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double s0 = x * y0;
  const double e = fma(-s0, y0, 1.0);
  const double t = fma(e, 0.375, 0.5);
  const double u = s0 * e;
  const double r = fma(u, t, s0);
  return x > 0.0 ? r : 0.0;
}

LSRN_DEV void box_muller_tab(uint4 o, const double* T, double& z0, double& z1) {
  const double rho = bm_sqrt(bm_m2ln_u1(o.x, o.y, T));
  double sn, cs;
  bm_sincos_2pi(o.z, o.w, T, sn, cs);
  z0 = rho * cs;
  z1 = rho * sn;
}

// ---- integer (fixed-point) Box-Muller (K1 v3, measured and not used by the sketch) --
// The same transform with the polynomial work on the integer pipe, meant to take
// the Box-Muller FP64 instructions off the pipe the dense sketch's DMMAs use:
// there the table-driven transform's ~49 FP64-pipe instructions per pair cost 15 %
// of the sketch (c5 shard: 1.75 s with it, 1.53 s with Philox only, 1.47 s with
// neither).  This version needs only 8 FP64 instructions + 1 MUFU per pair, but ~250
// integer multiply instructions (64-bit products as IMAD.WIDE chains), and the
// sketch got slower: 2.02 s (1.95 s with only sin / cos in integers)
// (profiles/r02_rng_cost.jsonl).  It stays as lsrn_debug_box_muller mode 2, tested
// against the oracle.  Tables / constants: bm_int_tables.h
// (tools/gen_bm_int_tables.py, 60 digits).  An integer model of these exact
// operations is within 3e-16 max(1, |z|) of 60-digit references on random and
// edge-case words.
//   sin / cos (2 pi u2): u2 = n2 2^-53; quadrant k = n2 >> 51, table j = next 6 bits,
//     d = low 45 bits, b = (pi/2) d 2^-51 < pi/128 in Q64 (umulhi(d << 14, K_B));
//     sin b, cos b by Horner in Q64 (degree 7 / 8); angle addition with the Q63
//     table values; the quadrant rotation on the results' signs.
//   x = -2 ln u1, n1 = (w0 >> 11) + 1 = 2^e m: r = m invc_i - 1 exact in Q61
//     (invc_i = CI_i / 512, the fp64 transform's table); x = A + B with
//     A = 2 (53 - e) ln 2 + 2 ln invc_i (Q57 integers, A = 0 exactly when u1 -> 1)
//     and B = -2 r log1p(r)/r, the series log1p(r)/r = sum (-r)^k / (k + 1) in Q62;
//     B is formed in fp64 from the exact integer r, so x keeps its relative
//     precision as u1 -> 1.
LSRN_DEV void bm_int_load_table(uint64_t* Ts) {
  for (int i = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); i < bmi::TAB_WORDS;
       i += blockDim.x * blockDim.y * blockDim.z)
    Ts[i] = bmi::kTable[i];
}

// v 2^-scale for an unsigned 64-bit v, rounded to nearest (ties to even), built from
// the bits (no integer -> double conversion on the FP64 pipe).  v = 0 -> 0.
LSRN_DEV double bmi_u64_to_double(uint64_t v, int scale) {
  const int lz = __clzll(static_cast<long long>(v));
  const uint64_t t = v << (lz & 63);
  uint64_t m = t >> 11;                                          // 53 bits, bit 52 set
  const uint64_t rem = t & 0x7FFull;
  m += (rem > 0x400ull) | ((rem == 0x400ull) & (m & 1ull));      // a carry to 2^53 bumps the exponent
  const uint64_t ex = static_cast<uint64_t>(63 - lz - scale + 1023);
  const uint64_t bits = (ex << 52) + (m - (1ull << 52));
  return v == 0 ? 0.0 : __longlong_as_double(static_cast<long long>(bits));
}

// the same with the sign bit set when neg (a sign flip without an FP64 instruction)
LSRN_DEV double bmi_u64_to_double_sgn(uint64_t v, int scale, bool neg) {
  const double d = bmi_u64_to_double(v, scale);
  return __longlong_as_double(__double_as_longlong(d) | (static_cast<long long>(neg) << 63));
}

LSRN_DEV uint64_t bmi_mul63(uint64_t a, uint64_t b) {            // (a b) >> 63
  return (__umul64hi(a, b) << 1) | ((a * b) >> 63);
}

LSRN_DEV void box_muller_int(uint4 o, const uint64_t* T, double& z0, double& z1) {
  // ---- sin / cos (2 pi u2)
  const uint64_t w1 = (static_cast<uint64_t>(o.w) << 32) | o.z;
  const uint64_t n2 = w1 >> 11;
  const int k = static_cast<int>(n2 >> 51);
  const int j = static_cast<int>((n2 >> 45) & 63);
  const uint64_t dm = n2 & ((1ull << 45) - 1);
  const uint64_t bq = __umul64hi(dm << 14, bmi::K_B);           // b in Q64
  const uint64_t b2 = __umul64hi(bq, bq);
  uint64_t t = bmi::S5 - __umul64hi(b2, bmi::S7);
  t = bmi::S3 - __umul64hi(b2, t);
  t = __umul64hi(b2, t);
  const uint64_t sb = (bq - __umul64hi(bq, t)) >> 1;             // sin b, Q63
  uint64_t u = bmi::C6 - __umul64hi(b2, bmi::C8);
  u = bmi::C4 - __umul64hi(b2, u);
  u = bmi::C2 - __umul64hi(b2, u);
  u = __umul64hi(b2, u);
  const uint64_t cb = (1ull << 63) - (u >> 1);                   // cos b, Q63
  const uint64_t sa = T[j], ca = T[64 + j];
  const uint64_t S = bmi_mul63(sa, cb) + bmi_mul63(ca, sb);      // sin(a + b), Q63
  const uint64_t C = bmi_mul63(ca, cb) - bmi_mul63(sa, sb);      // cos(a + b) > 0, Q63
  // rotate by k quarter turns: (sin, cos) = (S, C), (C, -S), (-S, -C), (-C, S)
  const double sn = bmi_u64_to_double_sgn((k & 1) ? C : S, 63, k >= 2);
  const double cs = bmi_u64_to_double_sgn((k & 1) ? S : C, 63, k == 1 || k == 2);
  // ---- x = -2 ln u1
  const uint64_t w0 = (static_cast<uint64_t>(o.y) << 32) | o.x;
  const uint64_t n1 = (w0 >> 11) + 1ull;                        // 1 .. 2^53
  const int e = 63 - __clzll(static_cast<long long>(n1));      // 0 .. 53
  const uint64_t mant = (n1 << ((52 - e) & 63)) & ((1ull << 52) - 1);
  const int i = static_cast<int>(mant >> 45);
  const int64_t R = static_cast<int64_t>(((1ull << 52) + mant) * T[256 + i]) - (1ll << 61);   // r in Q61, exact
  const int64_t R8 = R * 8;                                      // r in Q64 (|R8| < 2^57)
  int64_t p = bmi::PK8;                                          // log1p(r)/r by Horner, Q62
  p = bmi::PK7 - __mul64hi(R8, p);
  p = bmi::PK6 - __mul64hi(R8, p);
  p = bmi::PK5 - __mul64hi(R8, p);
  p = bmi::PK4 - __mul64hi(R8, p);
  p = bmi::PK3 - __mul64hi(R8, p);
  p = bmi::PK2 - __mul64hi(R8, p);
  p = bmi::PK1 - __mul64hi(R8, p);
  p = bmi::PK0 - __mul64hi(R8, p);
  const uint64_t A = static_cast<uint64_t>(53 - e) * bmi::TWO_LN2_Q57 + T[128 + i];   // Q57, >= 0
  const uint64_t aR = static_cast<uint64_t>(R < 0 ? -R : R);
  const double mRd = bmi_u64_to_double_sgn(aR, 0, R > 0);        // -r 2^61, exact (or 1 ulp if |R| >= 2^53)
  const double x = fma(mRd, bmi_u64_to_double(static_cast<uint64_t>(p), 122), bmi_u64_to_double(A, 57));
  // u1 = 1 (n1 = 2^53): x = 0 -> rho = 0; bm_sqrt's own zero test replaced by an integer one
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double s0 = x * y0;
  const double ee = fma(-s0, y0, 1.0);
  const double rho0 = fma(s0 * ee, fma(ee, 0.375, 0.5), s0);    // sqrt(x), as bm_sqrt
  const double rho = (e == 53 || __double_as_longlong(x) == 0) ? 0.0 : rho0;
  z0 = rho * cs;
  z1 = rho * sn;
}

LSRN_DEV uint4 philox_counter(uint2 key, uint64_t q, uint64_t j) {
  return philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(j),
                                  static_cast<uint32_t>(j >> 32), 0u), key);
}

// The normal pair (G[2q, j], G[2q+1, j]); T = shared-memory copy of bm::kTable.
LSRN_DEV void gaussian_pair(uint2 key, uint64_t q, uint64_t j, const double* T, double& z0, double& z1) {
  box_muller_tab(philox_counter(key, q, j), T, z0, z1);
}

// The same pair through the integer transform; T = shared-memory copy of bmi::kTable.
LSRN_DEV void gaussian_pair_int(uint2 key, uint64_t q, uint64_t j, const uint64_t* T, double& z0, double& z1) {
  box_muller_int(philox_counter(key, q, j), T, z0, z1);
}

}  // namespace lsrn
