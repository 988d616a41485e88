/*
 * lsrn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow CPU pieces of the LSRN oracle that the north star names
 * explicitly: "naive loops for GA" and "a one-sided Jacobi SVD".  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load this (through
 * oracle/_c.py).  It shares no code, header, table or constant generator with
 * the CUDA product (paper_1109_5981_b200/); the product never loads it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; C9 etc. = the readings in
 * DESIGN.md §3.
 *
 *   orc_philox4x32_10   Philox4x32-10 (Salmon et al., SC'11), the counter-based
 *                       generator of reading C9.
 *   orc_gaussian        G[i, j] (C9): u1 = ((w0 >> 11) + 1) 2^-53, u2 = (w1 >> 11) 2^-53,
 *                       rho = sqrt(-2 ln u1), G[2q, j] = rho cos 2 pi u2,
 *                       G[2q+1, j] = rho sin 2 pi u2, evaluated in long double
 *                       (x87 80-bit) and rounded once to double.
 *   orc_sketch_dense    Alg. 1/2 step 3 with the §5 blocks
 *                       in the tall form: At[i][c] = sx sum_j G[i, j] X[j][c]
 *                       + si G[i, L + c], by naive loops -- for each sketch row i
 *                       and column c the sum over the long index j in increasing
 *                       order, accumulated in fixed blocks of 256 consecutive j
 *                       (block partial first, then added to the running total;
 *                       SURVEY §8(c) O3, reading C17).  Sketch rows are processed
 *                       four Box-Muller pairs at a time (independent outputs, no
 *                       effect on any result bit) so X is streamed s/8 times.
 *   orc_jacobi_svd      Alg. 1 step 4: one-sided (Hestenes) Jacobi SVD
 *                       of an s x k matrix.  Cyclic sweeps in the round-robin
 *                       (tournament) ordering, each round's k/2 disjoint column
 *                       pairs rotated in parallel; a pair (p, q) is rotated when
 *                       |a_p . a_q| > s u |a_p| |a_q| (u = 2^-53),
 *                       the rotation zeroing a_p . a_q (t = sign(zeta) / (|zeta| +
 *                       sqrt(1 + zeta^2)), zeta = (|a_q|^2 - |a_p|^2) / (2 a_p . a_q));
 *                       the squared norms are recomputed at the start of every
 *                       sweep and updated by the rotation in between
 *                       (|a_p|^2 -= t g, |a_q|^2 += t g, exact in exact arithmetic);
 *                       converged when a sweep rotates nothing.  sigma_c = |a_c|
 *                       (recomputed), V accumulates the rotations; sorted descending.
 *
 * Every function is deterministic and independent of the OpenMP thread count
 * (each output element is computed by exactly one thread in a fixed order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ Philox */
void orc_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* ------------------------------------------------------------ Box-Muller (C9) */
static void gauss_pair(uint64_t seed, uint64_t q, uint64_t j, double* z0, double* z1) {
  const uint32_t ctr[4] = {(uint32_t)q, (uint32_t)j, (uint32_t)(j >> 32), 0u};
  uint32_t o[4];
  orc_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), o);
  const uint64_t w0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  const uint64_t w1 = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
  const long double u1 = (long double)((w0 >> 11) + 1) * 0x1p-53L;   /* (0, 1] */
  const long double u2 = (long double)(w1 >> 11) * 0x1p-53L;         /* [0, 1) */
  const long double two_pi = 8.0L * atanl(1.0L);
  const long double rho = sqrtl(-2.0L * logl(u1));
  *z0 = (double)(rho * cosl(two_pi * u2));
  *z1 = (double)(rho * sinl(two_pi * u2));
}

void orc_gaussian(uint64_t seed, const int64_t* rows, const int64_t* cols, int64_t n, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    double z0, z1;
    gauss_pair(seed, (uint64_t)(rows[t] >> 1), (uint64_t)cols[t], &z0, &z1);
    out[t] = (rows[t] & 1) ? z1 : z0;
  }
}

/* --------------------------------------------------------------- naive G A */
#define ORC_BLOCK 256   /* fixed summation blocks along the long index (C17) */
#define ORC_QB 4        /* Box-Muller pairs (8 sketch rows) per pass over X */

int orc_sketch_dense(const double* X, int64_t L, int64_t k, int64_t ld, int64_t s, uint64_t seed, double sx,
                     double si, double* At) {
  if (L < 0 || k <= 0 || s <= 0 || ld < k) return -1;
  const int64_t npair = (s + 1) / 2;
  const int64_t ntask = (npair + ORC_QB - 1) / ORC_QB;
  int fail = 0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * 2 * ORC_QB * k);
    double* blk = (double*)malloc(sizeof(double) * 2 * ORC_QB * k);
    if (!acc || !blk) {
#pragma omp atomic write
      fail = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t task = 0; task < ntask; ++task) {
      if (!acc || !blk) continue;
      const int64_t q0 = task * ORC_QB;
      const int64_t nq = (npair - q0) < ORC_QB ? (npair - q0) : ORC_QB;
      memset(acc, 0, sizeof(double) * 2 * ORC_QB * k);
      for (int64_t j0 = 0; j0 < L; j0 += ORC_BLOCK) {
        const int64_t j1 = (j0 + ORC_BLOCK < L) ? j0 + ORC_BLOCK : L;
        memset(blk, 0, sizeof(double) * 2 * ORC_QB * k);
        for (int64_t j = j0; j < j1; ++j) {
          const double* xj = X + j * ld;
          for (int64_t qq = 0; qq < nq; ++qq) {
            double z0, z1;
            gauss_pair(seed, (uint64_t)(q0 + qq), (uint64_t)j, &z0, &z1);
            double* b0 = blk + (2 * qq) * k;
            double* b1 = blk + (2 * qq + 1) * k;
            for (int64_t c = 0; c < k; ++c) {
              b0[c] += z0 * xj[c];
              b1[c] += z1 * xj[c];
            }
          }
        }
        for (int64_t e = 0; e < 2 * nq * k; ++e) acc[e] += blk[e];
      }
      for (int64_t qq = 0; qq < nq; ++qq) {
        for (int h = 0; h < 2; ++h) {
          const int64_t i = 2 * (q0 + qq) + h;
          if (i >= s) continue;
          for (int64_t c = 0; c < k; ++c) {
            double v = sx * acc[(2 * qq + h) * k + c];
            if (si != 0.0) {
              double z0, z1;
              gauss_pair(seed, (uint64_t)(q0 + qq), (uint64_t)(L + c), &z0, &z1);
              v += si * (h ? z1 : z0);
            }
            At[i * k + c] = v;
          }
        }
      }
    }
    free(acc);
    free(blk);
  }
  return fail ? -2 : 0;
}

/* CSR X (rowptr[L + 1] from 0, colind, val): the same sums as orc_sketch_dense, the
 * nonzeros of row j scattered into the block partials (row-wise scatter, O3). */
int orc_sketch_csr(const int64_t* rowptr, const int32_t* colind, const double* val, int64_t L, int64_t k, int64_t s,
                   uint64_t seed, double sx, double si, double* At) {
  if (L < 0 || k <= 0 || s <= 0) return -1;
  const int64_t npair = (s + 1) / 2;
  const int64_t ntask = (npair + ORC_QB - 1) / ORC_QB;
  int fail = 0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * 2 * ORC_QB * k);
    double* blk = (double*)malloc(sizeof(double) * 2 * ORC_QB * k);
    if (!acc || !blk) {
#pragma omp atomic write
      fail = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t task = 0; task < ntask; ++task) {
      if (!acc || !blk) continue;
      const int64_t q0 = task * ORC_QB;
      const int64_t nq = (npair - q0) < ORC_QB ? (npair - q0) : ORC_QB;
      memset(acc, 0, sizeof(double) * 2 * ORC_QB * k);
      for (int64_t j0 = 0; j0 < L; j0 += ORC_BLOCK) {
        const int64_t j1 = (j0 + ORC_BLOCK < L) ? j0 + ORC_BLOCK : L;
        memset(blk, 0, sizeof(double) * 2 * ORC_QB * k);
        for (int64_t j = j0; j < j1; ++j) {
          if (rowptr[j + 1] == rowptr[j]) continue;
          for (int64_t qq = 0; qq < nq; ++qq) {
            double z0, z1;
            gauss_pair(seed, (uint64_t)(q0 + qq), (uint64_t)j, &z0, &z1);
            double* b0 = blk + (2 * qq) * k;
            double* b1 = blk + (2 * qq + 1) * k;
            for (int64_t e = rowptr[j]; e < rowptr[j + 1]; ++e) {
              b0[colind[e]] += z0 * val[e];
              b1[colind[e]] += z1 * val[e];
            }
          }
        }
        for (int64_t e = 0; e < 2 * nq * k; ++e) acc[e] += blk[e];
      }
      for (int64_t qq = 0; qq < nq; ++qq) {
        for (int h = 0; h < 2; ++h) {
          const int64_t i = 2 * (q0 + qq) + h;
          if (i >= s) continue;
          for (int64_t c = 0; c < k; ++c) {
            double v = sx * acc[(2 * qq + h) * k + c];
            if (si != 0.0) {
              double z0, z1;
              gauss_pair(seed, (uint64_t)(q0 + qq), (uint64_t)(L + c), &z0, &z1);
              v += si * (h ? z1 : z0);
            }
            At[i * k + c] = v;
          }
        }
      }
    }
    free(acc);
    free(blk);
  }
  return fail ? -2 : 0;
}

/* ------------------------------------------------------- one-sided Jacobi */
/* A: s x k row-major (not modified).  sig: k (descending).  V: k x k row-major,
 * column c (V[j * k + c], j < k) = right singular vector c.  Returns the number
 * of sweeps (> 0), or -1 on bad arguments / no memory, -2 if max_sweeps ran out. */
int orc_jacobi_svd(const double* A, int64_t s, int64_t k, int max_sweeps, double* sig, double* V) {
  if (s <= 0 || k <= 0 || max_sweeps <= 0) return -1;
  /* column-major working copies: W (s x k) and Vc (k x k) */
  double* W = (double*)malloc(sizeof(double) * s * k);
  double* Vc = (double*)malloc(sizeof(double) * k * k);
  double* nrm = (double*)malloc(sizeof(double) * k);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (k + 1));
  if (!W || !Vc || !nrm || !perm) {
    free(W);
    free(Vc);
    free(nrm);
    free(perm);
    return -1;
  }
  for (int64_t i = 0; i < s; ++i)
    for (int64_t c = 0; c < k; ++c) W[c * s + i] = A[i * k + c];
  memset(Vc, 0, sizeof(double) * k * k);
  for (int64_t c = 0; c < k; ++c) Vc[c * k + c] = 1.0;
  const double tol = (double)s * 0x1p-53;
  /* round-robin tournament on an even number of players (a dummy when k is odd) */
  const int64_t np = (k + 1) / 2 * 2;
  for (int64_t t = 0; t < np; ++t) perm[t] = t;
  int sweeps = 0, converged = 0;
  while (!converged && sweeps < max_sweeps) {
    ++sweeps;
    int64_t rotated = 0;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < k; ++c) {
      double a = 0.0;
      for (int64_t i = 0; i < s; ++i) a += W[c * s + i] * W[c * s + i];
      nrm[c] = a;
    }
    for (int64_t round = 0; round < np - 1; ++round) {
#pragma omp parallel for schedule(static) reduction(+ : rotated)
      for (int64_t m = 0; m < np / 2; ++m) {
        int64_t p = perm[m], q = perm[np - 1 - m];
        if (p >= k || q >= k) continue;            /* dummy player */
        if (p > q) {
          const int64_t tmp = p;
          p = q;
          q = tmp;
        }
        double* wp = W + p * s;
        double* wq = W + q * s;
        const double a = nrm[p], b = nrm[q];
        double g = 0.0;
        for (int64_t i = 0; i < s; ++i) g += wp[i] * wq[i];
        if (g == 0.0 || fabs(g) <= tol * sqrt(a * b)) continue;
        ++rotated;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        nrm[p] = a - t * g;
        nrm[q] = b + t * g;
        for (int64_t i = 0; i < s; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = cs * x - sn * y;
          wq[i] = sn * x + cs * y;
        }
        double* vp = Vc + p * k;
        double* vq = Vc + q * k;
        for (int64_t i = 0; i < k; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
      /* rotate the tournament: player 0 fixed, the others move one seat */
      const int64_t last = perm[np - 1];
      for (int64_t t = np - 1; t > 1; --t) perm[t] = perm[t - 1];
      perm[1] = last;
    }
    converged = rotated == 0;
  }
  for (int64_t c = 0; c < k; ++c) {
    double a = 0.0;
    for (int64_t i = 0; i < s; ++i) a += W[c * s + i] * W[c * s + i];
    nrm[c] = sqrt(a);
  }
  /* sort descending (stable selection by index on ties) */
  for (int64_t c = 0; c < k; ++c) perm[c] = c;
  for (int64_t a = 1; a < k; ++a) {                /* insertion sort: k <= a few thousand */
    const int64_t v = perm[a];
    int64_t b = a - 1;
    while (b >= 0 && nrm[perm[b]] < nrm[v]) {
      perm[b + 1] = perm[b];
      --b;
    }
    perm[b + 1] = v;
  }
  for (int64_t c = 0; c < k; ++c) {
    sig[c] = nrm[perm[c]];
    for (int64_t j = 0; j < k; ++j) V[j * k + c] = Vc[perm[c] * k + j];
  }
  free(W);
  free(Vc);
  free(nrm);
  free(perm);
  return converged ? sweeps : -2;
}
