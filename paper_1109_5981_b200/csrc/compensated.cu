// Compensated row pass: the precision = 1 option (LSRN_COMPENSATED, DESIGN.md
// reading C18(ii)).
//
// Same contract as the fp64 row pass (rowpass.cu: K5 on N^T, K6 on X), but the
// vectors that cross between the two products are carried as unevaluated sums
// hi + lo (double-double) and every dot product and column sum is accumulated
// with error-free transformations (TwoProd by FMA, TwoSum; the Dot2 scheme of
// Ogita, Rump and Oishi), so each product is as accurate as if computed in about
// twice the working precision and rounded once:
//     z_j <- c1 z_j + c2 sx (Y_j . (t_hi + t_lo))       (z: fp64 Krylov vector)
//     acc_j += ca z_j
//     (out_hi + out_lo) = sx Y^T z (+ sI zI, zI <- c1 zI + c2 sI t)   out_hi[C] = ||z||^2 (+ ||zI||^2)
// Why: with t = N v rounded to fp64, A t carries an absolute
// error ~ u ||A|| ||t||, and t's large components (the small-sigma directions,
// ||N|| ~ 1 / sigma_min) cancel in A t, so x has a relative error ~ kappa(A) u:
// 1.7e-9 at kappa = 1e6 on c1's shape, above the 1e-9 bar.  Carrying t (and
// A^T u, whose small-sigma components N^T amplifies) in double-double removes
// that term; the Krylov recurrences stay fp64.  The oracle's counterpart is its
// long-double product mode (oracle/lsrn.py LongOperator(extended=True)).
//
// Two launches per pass: ext_rowpass_kernel (block b owns a contiguous row range:
// warp-per-row compensated dots, then thread-per-column compensated sums of the
// block's rows into the partial (s, c)[b][:]) and ext_colreduce_kernel (fixed-
// order double-double sum of the partials, the Tikhonov block, the norm).
// Deterministic (fixed ranges and reduction trees, no atomics).  Not tuned for
// speed: each row of Y is read twice (the second time mostly from L2) and the
// arithmetic is ~10x the fp64 pass; it is an accuracy mode for ill-conditioned
// problems, measured in DESIGN.md §8.
#include "common.cuh"
#include "kernels.h"

namespace lsrn {

namespace {
constexpr int EXT_THREADS = 256;

LSRN_DEV void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

LSRN_DEV void two_prod(double a, double b, double& p, double& e) {
  p = a * b;
  e = fma(a, b, -p);
}

// (s, c) += a * (th + tl)
LSRN_DEV void dot2_step(double a, double th, double tl, double& s, double& c) {
  double p, q, r, sn;
  two_prod(a, th, p, q);
  two_sum(s, p, sn, r);
  s = sn;
  c += q + r;
  c = fma(a, tl, c);
}

// (s, c) += (s2, c2)
LSRN_DEV void dd_add(double& s, double& c, double s2, double c2) {
  double sn, r;
  two_sum(s, s2, sn, r);
  s = sn;
  c += c2 + r;
}

// round (s, c) to a normalised pair (hi = fl(s + c))
LSRN_DEV void dd_norm(double s, double c, double& hi, double& lo) {
  hi = s + c;
  lo = c - (hi - s);
}

LSRN_DEV void warp_dd_sum(double& s, double& c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const double c2 = __shfl_xor_sync(0xffffffffu, c, o);
    // the lower lane's pair first on both lanes: identical results
    const int lane = threadIdx.x & 31;
    const double a = (lane & o) ? s2 : s, ac = (lane & o) ? c2 : c;
    const double b = (lane & o) ? s : s2, bc = (lane & o) ? c : c2;
    s = a;
    c = ac;
    dd_add(s, c, b, bc);
  }
}

// c1 z + c2 (ds + dc), evaluated with one rounding of the compensated sum
LSRN_DEV double axpy_dd(double c1, double z, double c2, double ds, double dc) {
  double p1, e1, p2, e2, s, r;
  two_prod(c1, z, p1, e1);
  two_prod(c2, ds, p2, e2);
  two_sum(p1, p2, s, r);
  return s + (((e1 + e2) + r) + c2 * dc);
}
}  // namespace

__global__ void __launch_bounds__(EXT_THREADS)
ext_rowpass_kernel(ExtRowPassArgs a, int64_t rows_per_block) {
  __shared__ double sh[EXT_THREADS / 32];
  if (a.done != nullptr && *a.done != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(a.R, r0 + rows_per_block);
  const double c1 = a.coef[0], c2 = a.coef[1] * a.sx;
  const double ca = (a.acc != nullptr) ? a.coef[2] : 0.0;
  // phase 1: z_j for the block's rows (warp per row)
  double nrm = 0.0;
  for (int64_t j = r0 + warp; j < r1; j += EXT_THREADS / 32) {
    const double* yr = a.Y + j * a.ld;
    double s = 0.0, c = 0.0;
    for (int64_t q = lane; q < a.C; q += 32) dot2_step(yr[q], a.t_hi[q], a.t_lo[q], s, c);
    warp_dd_sum(s, c);
    if (lane == 0) {
      const double zn = axpy_dd(c1, a.z[j], c2, s, c);
      a.z[j] = zn;
      if (a.acc != nullptr) a.acc[j] = fma(ca, zn, a.acc[j]);
      nrm = fma(zn, zn, nrm);
    }
  }
  // fixed-order block sum of the norm (warp 0 lane 0 of each warp holds a partial)
  if (lane == 0) sh[warp] = nrm;
  __threadfence_block();
  __syncthreads();                      // the block's new z visible to all its threads
  if (threadIdx.x == 0) {
    double b = 0.0;
#pragma unroll
    for (int w = 0; w < EXT_THREADS / 32; ++w) b += sh[w];
    a.npart[blockIdx.x] = b;
  }
  // phase 2: partial (s, c) of sx Y^T z over the block's rows (thread per column)
  for (int64_t q = threadIdx.x; q < a.C; q += EXT_THREADS) {
    double s = 0.0, c = 0.0;
    for (int64_t j = r0; j < r1; ++j) dot2_step(a.Y[j * a.ld + q], a.z[j], 0.0, s, c);
    double ps, pe;
    two_prod(a.sx, s, ps, pe);
    a.part_s[(int64_t)blockIdx.x * a.C + q] = ps;
    a.part_c[(int64_t)blockIdx.x * a.C + q] = fma(a.sx, c, pe);
  }
}

__global__ void __launch_bounds__(1024)
ext_colreduce_kernel(ExtColReduceArgs a) {
  __shared__ double sh[32];
  if (a.done != nullptr && *a.done != 0) return;
  double nI = 0.0;
  for (int64_t q = threadIdx.x; q < a.C; q += blockDim.x) {
    double s = 0.0, c = 0.0;
    for (int g = 0; g < a.nparts; ++g) dd_add(s, c, a.part_s[(int64_t)g * a.C + q], a.part_c[(int64_t)g * a.C + q]);
    if (a.zI != nullptr) {
      // zI <- c1 zI + c2 sI t  (t = t_hi + t_lo), then out += sI zI
      double p, e;
      two_prod(a.sI, a.t_hi[q], p, e);
      const double zn = axpy_dd(a.coef[0], a.zI[q], a.coef[1], p, fma(a.sI, a.t_lo[q], e));
      a.zI[q] = zn;
      two_prod(a.sI, zn, p, e);
      dd_add(s, c, p, e);
      nI = fma(zn, zn, nI);
    }
    double hi, lo;
    dd_norm(s, c, hi, lo);
    a.out_hi[q] = hi;
    a.out_lo[q] = lo;
  }
  // ||z||^2: the row blocks' partials (fixed order) + the I block (fixed tree)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  nI = warp_sum(nI);
  if (lane == 0) sh[warp] = nI;
  __syncthreads();
  if (threadIdx.x == 0) {
    double n = 0.0;
    for (int g = 0; g < a.nparts; ++g) n += a.npart[g];
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) n += sh[w];
    a.out_hi[a.C] = n;
    a.out_lo[a.C] = 0.0;
  }
}

int ext_rowpass_blocks(int64_t R, int nsm) {
  // about 2 blocks per SM, at least 32 rows each
  int64_t nb = std::min<int64_t>(2 * (int64_t)(nsm > 0 ? nsm : 148), (R + 31) / 32);
  return (int)std::max<int64_t>(nb, 1);
}

cudaError_t launch_ext_rowpass(const ExtRowPassArgs& a, int nblocks, cudaStream_t st) {
  if (a.R <= 0 || nblocks <= 0) return cudaSuccess;
  const int64_t per = (a.R + nblocks - 1) / nblocks;
  ext_rowpass_kernel<<<nblocks, EXT_THREADS, 0, st>>>(a, per);
  return cudaGetLastError();
}

cudaError_t launch_ext_colreduce(const ExtColReduceArgs& a, cudaStream_t st) {
  ext_colreduce_kernel<<<1, 1024, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace lsrn
