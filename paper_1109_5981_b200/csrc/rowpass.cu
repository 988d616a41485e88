// K5 / K6: the fused single-pass preconditioned matvec of LSQR and CS.
//
// One launch streams a row-major R x C matrix Y exactly once and computes, for
// every row j,
//     z_j <- c1 z_j + c2 (Y_j . t)        (the new Krylov vector entry)
//     acc_j += ca z_j                     (optional fused x/y update, CS)
//     norm2 += z_j^2,   w += Y_j z_j      (Y^T z, the transposed product)
// Long pass (K6): Y = X (A, or A^T for Alg. 2) -- "u = A t - c u ; w = A^T u" in
// one read of A instead of two (the paper
// counts flops(Av) + flops(A^T u) per iteration).
// Short pass (K5): Y = N^T (N column-major) -- "v = c1 v + c2 N^T w ; t = N v".
//
// Layout: each CTA owns a column slice of 512 * VPT columns (two per thread per
// VPT step, 16-byte loads) and a contiguous chunk of rows (per cluster).  When
// C > 512 * VPT the row is split over a thread-block cluster of CL CTAs that
// exchange their partial dot products through distributed shared memory
// (one cluster barrier per row tile); every CTA of the cluster then knows z_j
// and accumulates its slice of w in registers.  Rows are processed TR at a time
// with the next tile's loads issued before the current tile's reduction.
// Deterministic: fixed row chunks, fixed reduction trees, no atomics.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace lsrn {

template <int VPT, int TR, int VEC>
__global__ void __launch_bounds__(256, 1)
rowpass_kernel(RowPassArgs a, int64_t rows_per_cluster, int CL) {
  __shared__ double red[2][8][TR];
  __shared__ double xs[2][8][TR];
  if (a.done != nullptr && *a.done != 0) return;     // uniform over the grid
  const int q = (CL > 1) ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t g = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t C = a.C;
  const int64_t cbase = (int64_t)q * (512 * VPT);
  const double c1 = a.coef[0], c2 = a.coef[1] * a.sx;
  const double ca = (a.acc != nullptr) ? a.coef[2] : 0.0;

  double2 tv[VPT], wv[VPT];
#pragma unroll
  for (int p = 0; p < VPT; ++p) {
    const int64_t c = cbase + 2 * (tid + 256 * p);
    tv[p].x = (c < C) ? a.t[c] : 0.0;
    tv[p].y = (c + 1 < C) ? a.t[c + 1] : 0.0;
    wv[p] = make_double2(0.0, 0.0);
  }
  const int64_t r0 = g * rows_per_cluster;
  const int64_t r1 = min(a.R, r0 + rows_per_cluster);
  const int64_t ntiles = (r1 > r0) ? (r1 - r0 + TR - 1) / TR : 0;

  auto load_tile = [&](int64_t tile, double2 (&y)[TR][VPT], double (&zo)[TR]) {
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const int64_t row = r0 + tile * TR + tr;
      const bool rok = row < r1;
      zo[tr] = rok ? a.z[row] : 0.0;
      const double* yr = a.Y + row * a.ld;
#pragma unroll
      for (int p = 0; p < VPT; ++p) {
        const int64_t c = cbase + 2 * (tid + 256 * p);
        if (VEC == 2) {
          if (rok && c + 1 < C) {
            y[tr][p] = ldg_stream2(yr + c);
          } else {
            y[tr][p].x = (rok && c < C) ? ldg_stream1(yr + c) : 0.0;
            y[tr][p].y = 0.0;
          }
        } else {
          y[tr][p].x = (rok && c < C) ? ldg_stream1(yr + c) : 0.0;
          y[tr][p].y = (rok && c + 1 < C) ? ldg_stream1(yr + c + 1) : 0.0;
        }
      }
    }
  };

  double2 y[TR][VPT], yn[TR][VPT];
  double zo[TR], zon[TR];
  double norm = 0.0;
  if (ntiles > 0) load_tile(0, y, zo);
  int buf = 0;
  for (int64_t tile = 0; tile < ntiles; ++tile) {
    double d[TR];
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < VPT; ++p) s = fma(y[tr][p].x, tv[p].x, fma(y[tr][p].y, tv[p].y, s));
      d[tr] = s;
    }
    if (tile + 1 < ntiles) load_tile(tile + 1, yn, zon);
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const double s = warp_sum(d[tr]);
      if (lane == 0) red[buf][warp][tr] = s;
    }
    __syncthreads();
    double dot[TR];
    if (CL > 1) {
      cg::cluster_group cluster = cg::this_cluster();
      if (tid < TR) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[buf][w][tid];
        for (int rr = 0; rr < CL; ++rr) {
          double* remote = cluster.map_shared_rank(&xs[buf][q][tid], rr);
          *remote = s;
        }
      }
      cluster.sync();
#pragma unroll
      for (int tr = 0; tr < TR; ++tr) {
        double s = 0.0;
        for (int qq = 0; qq < CL; ++qq) s += xs[buf][qq][tr];
        dot[tr] = s;
      }
    } else {
#pragma unroll
      for (int tr = 0; tr < TR; ++tr) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[buf][w][tr];
        dot[tr] = s;
      }
    }
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const int64_t row = r0 + tile * TR + tr;
      double zn = 0.0;
      if (row < r1) {
        zn = fma(c1, zo[tr], c2 * dot[tr]);
        norm = fma(zn, zn, norm);
        if (q == 0 && tid == 0) {
          a.z[row] = zn;
          if (a.acc != nullptr) a.acc[row] = fma(ca, zn, a.acc[row]);
        }
      }
#pragma unroll
      for (int p = 0; p < VPT; ++p) {
        wv[p].x = fma(y[tr][p].x, zn, wv[p].x);
        wv[p].y = fma(y[tr][p].y, zn, wv[p].y);
      }
    }
    if (tile + 1 < ntiles) {
#pragma unroll
      for (int tr = 0; tr < TR; ++tr) {
        zo[tr] = zon[tr];
#pragma unroll
        for (int p = 0; p < VPT; ++p) y[tr][p] = yn[tr][p];
      }
    }
    buf ^= 1;
  }
  double* wp = a.wpart + g * C;
#pragma unroll
  for (int p = 0; p < VPT; ++p) {
    const int64_t c = cbase + 2 * (tid + 256 * p);
    if (c < C) wp[c] = a.sx * wv[p].x;
    if (c + 1 < C) wp[c + 1] = a.sx * wv[p].y;
  }
  if (q == 0 && tid == 0) a.npart[g] = norm;
  if (CL > 1) cg::this_cluster().sync();   // keep smem alive until remote stores land
}

// --------------------------------------------------------------- col reduce
// Block (16 columns) x (32 partial groups): thread (x, y) sums partials g = y,
// y + 32, ... of column c = 16 blockIdx.x + x (two accumulators, fixed order);
// the 32 group sums are added in fixed order.  The last block to finish adds the
// norm partials (one warp, fixed order).  Deterministic.  History on c2 (2000
// columns, 296 partials): one thread per column ~28 us; 32 x 16 blocks 13.6 us
// (63 blocks: fewer than one per SM); 16 x 32 blocks twice the blocks and half
// the serial chain per thread.
constexpr int CR_X = 16, CR_Y = 32;

__global__ void __launch_bounds__(CR_X * CR_Y)
colreduce_kernel(ColReduceArgs a) {
  __shared__ double sh[CR_Y][CR_X + 1];
  __shared__ bool last;
  if (a.done != nullptr && *a.done != 0) return;
  const int tid = threadIdx.x;                 // 1-D block (warp_sum_l2 takes its lane from threadIdx.x)
  const int x = tid % CR_X, y = tid / CR_X;
  const int64_t c = (int64_t)blockIdx.x * CR_X + x;
  double w0 = 0.0, w1 = 0.0;
  if (c < a.C) {
    int g = y;
    for (; g + CR_Y < a.nparts; g += 2 * CR_Y) {
      w0 += a.wpart[(int64_t)g * a.C + c];
      w1 += a.wpart[(int64_t)(g + CR_Y) * a.C + c];
    }
    if (g < a.nparts) w0 += a.wpart[(int64_t)g * a.C + c];
  }
  sh[y][x] = w0 + w1;
  __syncthreads();
  double nI = 0.0;
  if (y == 0 && c < a.C) {
    double t = 0.0;
#pragma unroll
    for (int yy = 0; yy < CR_Y; ++yy) t += sh[yy][x];
    if (a.zI != nullptr) {
      const double zn = fma(a.coef[0], a.zI[c], a.coef[1] * (a.sI * a.t[c]));
      a.zI[c] = zn;
      t = fma(a.sI, zn, t);
      nI = zn * zn;
    }
    a.out[c] = t;
  }
  if (tid < 32) {                            // warp 0 holds the y == 0 row (CR_X <= 32)
    const double bsum = warp_sum(nI);
    if (tid == 0) {
      a.blockpart[blockIdx.x] = bsum;
      __threadfence();
      last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (last && tid < 32) {
    __threadfence();
    const double n = warp_sum_l2(a.npart, a.nparts) + warp_sum_l2(a.blockpart, gridDim.x);
    if (tid == 0) {
      a.out[a.C] = n;
      *a.counter = 0u;
    }
  }
}

int colreduce_blocks(int64_t C) { return (int)((C + CR_X - 1) / CR_X); }

cudaError_t launch_colreduce(const ColReduceArgs& a, cudaStream_t st) {
  colreduce_kernel<<<colreduce_blocks(a.C), CR_X * CR_Y, 0, st>>>(a);
  return cudaGetLastError();
}

// --------------------------------------------------------------- planning
RowPassPlan plan_rowpass(int64_t R, int64_t C, int64_t ld, const double* Y, int nsm, bool allow_bulk) {
  RowPassPlan p{};
  if (allow_bulk && plan_rowpass_bulk(R, C, ld, Y, nsm, &p)) return p;
  p.vec = ((ld % 2) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0) ? 2 : 1;
  if (C <= 512) p.vpt = 1;
  else if (C <= 1024) p.vpt = 2;
  else if (C <= 2048) p.vpt = 4;
  else p.vpt = 8;
  p.cl = (int)((C + 512 * p.vpt - 1) / (512 * p.vpt));
  if (p.cl < 1) p.cl = 1;
  p.tr = 8 / p.vpt;
  int nclusters = nsm / p.cl;
  if (nclusters < 1) nclusters = 1;
  const int64_t rows_needed = (R + p.tr - 1) / p.tr;   // at least one tile per cluster
  if ((int64_t)nclusters > rows_needed) nclusters = (int)(rows_needed > 0 ? rows_needed : 1);
  p.nclusters = nclusters;
  p.rows_per_cluster = (R + nclusters - 1) / nclusters;
  if (p.rows_per_cluster < 1) p.rows_per_cluster = 1;
  return p;
}

template <int VPT, int TR, int VEC>
static cudaError_t launch_t(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.nclusters * p.cl));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.cl > 8) {
    cudaError_t e = cudaFuncSetAttribute(rowpass_kernel<VPT, TR, VEC>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchKernelEx(&cfg, rowpass_kernel<VPT, TR, VEC>, a, p.rows_per_cluster, p.cl);
}

cudaError_t launch_rowpass(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  if (p.bulk) return launch_rowpass_bulk(a, p, st);
  if (p.cl > 16) return cudaErrorInvalidValue;
  if (p.vec == 2) {
    switch (p.vpt) {
      case 1: return launch_t<1, 8, 2>(a, p, st);
      case 2: return launch_t<2, 4, 2>(a, p, st);
      case 4: return launch_t<4, 2, 2>(a, p, st);
      default: return launch_t<8, 1, 2>(a, p, st);
    }
  }
  switch (p.vpt) {
    case 1: return launch_t<1, 8, 1>(a, p, st);
    case 2: return launch_t<2, 4, 1>(a, p, st);
    case 4: return launch_t<4, 2, 1>(a, p, st);
    default: return launch_t<8, 1, 1>(a, p, st);
  }
}

}  // namespace lsrn
