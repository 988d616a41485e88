// K5 / K6 on the TMA bulk-copy engine: the fused single-pass matvec of
// rowpass.cu, with the rows of Y streamed into a shared-memory ring by
// cp.async.bulk (1-D TMA) and mbarrier completion instead of per-thread loads.
//
// Same contract as rowpass_kernel (kernels.h RowPassArgs): for every row j
//     z_j <- c1 z_j + c2 sx (Y_j . t);  acc_j += ca z_j;  norm2 += z_j^2;  w += sx Y_j z_j.
// The paper counts flops(Av) + flops(A^T u) per iteration; this
// pass reads each row of A (or N^T) from HBM exactly once.
//
// Why bulk copies: the pass is HBM-bound and needs ~40 KB in flight per SM to
// cover DRAM latency at 6.5 TB/s.  Per-thread 16-byte loads kept only one row
// tile (32 KB) in flight and reached ~48 % of the measured copy bandwidth
// (profiles/r01_ncu_full_sketch_rowpass.json).  Here one elected thread keeps
// NST - 1 stages of TR rows (32-64 KB each) in flight while the CTA reduces the
// current stage out of shared memory.
//
// Layout: cluster g owns a contiguous chunk of rows; CTA q of the cluster owns
// the column slice [q Cq, (q+1) Cq); thread tid owns columns 2 (tid + NT p) +
// {0, 1} of the slice, p < P, and keeps t and w for them in registers.  Plans
// (plan_rowpass_bulk): rows <= 8192 doubles in one 256-thread CTA (two CTAs per
// SM); 8192-10240 in one 512-thread CTA with two 1-row stages (c5); wider rows in
// clusters whose partial row dots are exchanged through distributed shared
// memory (rowpass_cluster_kernel, asynchronous st.async exchange; 2-CTA clusters
// of 512 threads up to 20480, c4's N-pass).  Deterministic: fixed row chunks and
// reduction trees, no atomics.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace lsrn {

namespace {

constexpr int THREADS = 256;
constexpr int kMaxStages = 8;

}  // namespace

// TR rows per stage; P column pairs per thread (slice width <= 512 P).
// KEEP: hold the staged row tile in registers between the two phases (2 P TR
// doubles per thread) instead of re-reading shared memory; OCC: CTAs per SM.
template <int P, int TR, bool KEEP, int OCC, int NT = THREADS>
__global__ void __launch_bounds__(NT, OCC)
rowpass_bulk_kernel(RowPassArgs a, int64_t rows_per_cluster, int CL, int64_t Cq, int nst, int pf) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kMaxStages];
  constexpr int NWARP_ = NT / 32;
  __shared__ double red[2][NWARP_][TR];
  __shared__ double xs[2][16][TR];
  if (a.done != nullptr && *a.done != 0) return;     // uniform over the grid

  const int q = (CL > 1) ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t g = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t C = a.C;
  const int64_t c0 = (int64_t)q * Cq;
  const int64_t ncol = max((int64_t)0, min(Cq, C - c0));       // this CTA's slice width (even)
  const unsigned row_bytes = (unsigned)(ncol * 8);
  const int64_t stage_ld = Cq;                                   // doubles per staged row
  double* stage = reinterpret_cast<double*>(smem_raw);           // [nst][TR][stage_ld]

  const double c1 = a.coef[0], c2 = a.coef[1] * a.sx;
  const double ca = (a.acc != nullptr) ? a.coef[2] : 0.0;

  const int64_t r0 = g * rows_per_cluster;
  const int64_t r1 = min(a.R, r0 + rows_per_cluster);
  const int64_t ntiles = (r1 > r0) ? (r1 - r0 + TR - 1) / TR : 0;

  auto issue = [&](int64_t tile) {     // one thread: stage tile % nst <- rows of `tile`
    const int st = (int)(tile % nst);
    const int64_t rb = r0 + tile * TR;
    const int nr = (int)min((int64_t)TR, r1 - rb);
    if (row_bytes == 0) {
      mbar_arrive(&full[st]);
      return;
    }
    mbar_arrive_expect_tx(&full[st], row_bytes * (unsigned)nr);
    for (int tr = 0; tr < nr; ++tr)
      bulk_g2s(stage + ((int64_t)st * TR + tr) * stage_ld, a.Y + (rb + tr) * a.ld + c0, row_bytes, &full[st]);
    // L2 prefetch `pf` tiles beyond the one just issued: with only two shared-memory
    // stages of 80 KB rows (c5) the DRAM latency of the next refill is otherwise exposed
    if (pf > 0) {
      const int64_t pb = rb + (int64_t)pf * TR;
      for (int tr = 0; tr < TR && pb + tr < r1; ++tr) bulk_prefetch_l2(a.Y + (pb + tr) * a.ld + c0, row_bytes);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {       // prime every stage; stage of tile t-1 is refilled after tile t's barrier
    for (int64_t t = 0; t < min((int64_t)nst, ntiles); ++t) issue(t);
  }

  double2 tv[P], wv[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = 2 * (tid + NT * p);
    const int64_t c = c0 + cl;
    tv[p].x = (cl < ncol) ? a.t[c] : 0.0;
    tv[p].y = (cl + 1 < ncol) ? a.t[c + 1] : 0.0;
    wv[p] = make_double2(0.0, 0.0);
  }

  double norm = 0.0;
  int buf = 0;
  for (int64_t tile = 0; tile < ntiles; ++tile) {
    const int st = (int)(tile % nst);
    const unsigned parity = (unsigned)((tile / nst) & 1);
    const int64_t rb = r0 + tile * TR;
    double zo[TR];
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) zo[tr] = (rb + tr < r1) ? a.z[rb + tr] : 0.0;
    mbar_wait(&full[st], parity);

    // phase 1: partial row dots from shared memory (rows past r1 are zero-weighted)
    double d[TR];
    double2 yk[KEEP ? TR : 1][KEEP ? P : 1];
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const double* row = stage + ((int64_t)st * TR + tr) * stage_ld;
      double s = 0.0;
      const bool rok = rb + tr < r1;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t cl = 2 * (tid + NT * p);
        const double2 y = (rok && cl < ncol) ? *reinterpret_cast<const double2*>(row + cl) : make_double2(0.0, 0.0);
        if constexpr (KEEP) yk[tr][p] = y;
        s = fma(y.x, tv[p].x, fma(y.y, tv[p].y, s));
      }
      d[tr] = s;
    }
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const double s = warp_sum(d[tr]);
      if (lane == 0) red[buf][warp][tr] = s;
    }
    __syncthreads();                       // partial dots visible; stage of tile-1 fully consumed
    // refill the stage the previous tile used (its phase-2 reads finished before this barrier)
    if (tid == 0 && tile >= 1 && tile - 1 + nst < ntiles) issue(tile - 1 + nst);
    double dot[TR];
    if (CL > 1) {
      cg::cluster_group cluster = cg::this_cluster();
      if (tid < TR) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NWARP_; ++w) s += red[buf][w][tid];
        for (int rr = 0; rr < CL; ++rr) *cluster.map_shared_rank(&xs[buf][q][tid], rr) = s;
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
        for (int w = 0; w < NWARP_; ++w) s += red[buf][w][tr];
        dot[tr] = s;
      }
    }
    // phase 2: new z entries, norm, and w += y z re-read from shared memory
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const int64_t row = rb + tr;
      if (row < r1) {
        const double zn = fma(c1, zo[tr], c2 * dot[tr]);
        norm = fma(zn, zn, norm);
        if (q == 0 && tid == 0) {
          a.z[row] = zn;
          if (a.acc != nullptr) a.acc[row] = fma(ca, zn, a.acc[row]);
        }
        const double* rowp = stage + ((int64_t)st * TR + tr) * stage_ld;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int64_t cl = 2 * (tid + NT * p);
          if (cl < ncol) {
            double2 y;
            if constexpr (KEEP)
              y = yk[tr][p];
            else
              y = *reinterpret_cast<const double2*>(rowp + cl);
            wv[p].x = fma(y.x, zn, wv[p].x);
            wv[p].y = fma(y.y, zn, wv[p].y);
          }
        }
      }
    }
    buf ^= 1;
  }
  double* wp = a.wpart + g * C;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = 2 * (tid + NT * p);
    if (cl < ncol) wp[c0 + cl] = a.sx * wv[p].x;
    if (cl + 1 < ncol) wp[c0 + cl + 1] = a.sx * wv[p].y;
  }
  if (q == 0 && tid == 0) a.npart[g] = norm;
  if (CL > 1) cg::this_cluster().sync();   // keep smem alive until remote stores land
}

// ----------------------------------------------------------- wide rows (CL > 1)
// Rows wider than one CTA slice are split over a cluster of CL CTAs that must
// exchange partial row dots.  With one cluster barrier per tile the c5 long pass
// (k = 1e4, 3-CTA clusters, one 80 KB row per tile) ran at 1.8 TB/s.  Here the
// exchange is asynchronous and software-pipelined: after the block reduction of
// tile t each CTA pushes its TR partials into every peer's `xs` slot with
// st.async (completing on the peer's `xbar` mbarrier) and goes on to finish tile
// t-1, whose peer partials were sent one tile earlier.  Four exchange slots: a
// peer sends tile t only after finishing tile t-2, which needs our tile t-2
// partials, which we send after our wait on tile t-4 and after reading tile
// t-3's slot -- so slot t % 4 (and its barrier phase) is free when t arrives.
namespace {
LSRN_DEV unsigned cl_map(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
LSRN_DEV void st_async_f64(unsigned addr, double v, unsigned bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(addr), "d"(v),
               "r"(bar)
               : "memory");
}
LSRN_DEV void cluster_sync_all2() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
}  // namespace

template <int P, int TR, int OCC, int NT>
__global__ void __launch_bounds__(NT, OCC)
rowpass_cluster_kernel(RowPassArgs a, int64_t rows_per_cluster, int CL, int64_t Cq, int nst) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kMaxStages];
  __shared__ uint64_t xbar[4];
  constexpr int NWARP_ = NT / 32;
  __shared__ double red[2][NWARP_][TR];
  __shared__ double xs[4][16][TR];
  __shared__ double zs[4][TR];                       // old z of the tile, read before the exchange
  if (a.done != nullptr && *a.done != 0) return;     // uniform over the grid

  const unsigned q = cg::this_cluster().block_rank();
  const int64_t g = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t C = a.C;
  const int64_t c0 = (int64_t)q * Cq;
  const int64_t ncol = max((int64_t)0, min(Cq, C - c0));
  const unsigned row_bytes = (unsigned)(ncol * 8);
  const int64_t stage_ld = Cq;
  double* stage = reinterpret_cast<double*>(smem_raw);           // [nst][TR][stage_ld]
  const double c1 = a.coef[0], c2 = a.coef[1] * a.sx;
  const double ca = (a.acc != nullptr) ? a.coef[2] : 0.0;
  const int64_t r0 = g * rows_per_cluster;
  const int64_t r1 = min(a.R, r0 + rows_per_cluster);
  const int64_t ntiles = (r1 > r0) ? (r1 - r0 + TR - 1) / TR : 0;

  auto issue = [&](int64_t tile) {
    const int st = (int)(tile % nst);
    const int64_t rb = r0 + tile * TR;
    const int nr = (int)min((int64_t)TR, r1 - rb);
    if (row_bytes == 0) {
      mbar_arrive(&full[st]);
      return;
    }
    mbar_arrive_expect_tx(&full[st], row_bytes * (unsigned)nr);
    for (int tr = 0; tr < nr; ++tr)
      bulk_g2s(stage + ((int64_t)st * TR + tr) * stage_ld, a.Y + (rb + tr) * a.ld + c0, row_bytes, &full[st]);
  };

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < 4; ++s) mbar_init(&xbar[s], 1);
    mbar_fence_init();
  }
  cluster_sync_all2();                       // peers' xbar exist before any st.async
  if (tid == 0)
    for (int64_t t = 0; t < min((int64_t)nst, ntiles); ++t) issue(t);

  double2 tv[P], wv[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = 2 * (tid + NT * p);
    tv[p].x = (cl < ncol) ? a.t[c0 + cl] : 0.0;
    tv[p].y = (cl + 1 < ncol) ? a.t[c0 + cl + 1] : 0.0;
    wv[p] = make_double2(0.0, 0.0);
  }
  double norm = 0.0;

  // phase 1 of `tile`: partial dots, block reduction, push to every CTA of the cluster
  auto phase1 = [&](int64_t tile) {
    const int st = (int)(tile % nst);
    const int64_t rb = r0 + tile * TR;
    // old z of row rb + tid, fetched before the stage wait so its latency overlaps it
    const double zpre = (tid < TR && rb + tid < r1) ? a.z[rb + tid] : 0.0;
    mbar_wait(&full[st], (unsigned)((tile / nst) & 1));
    double d[TR];
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const double* row = stage + ((int64_t)st * TR + tr) * stage_ld;
      const bool rok = rb + tr < r1;
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t cl = 2 * (tid + NT * p);
        if (rok && cl < ncol) {
          const double2 y = *reinterpret_cast<const double2*>(row + cl);
          s = fma(y.x, tv[p].x, fma(y.y, tv[p].y, s));
        }
      }
      d[tr] = s;
    }
    const int rb2 = (int)(tile & 1), xb = (int)(tile & 3);
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const double s = warp_sum(d[tr]);
      if (lane == 0) red[rb2][warp][tr] = s;
    }
    __syncthreads();
    if (tid == 0) mbar_arrive_expect_tx(&xbar[xb], (unsigned)(CL * TR * 8));
    if (tid < TR) {
      // the old z of this row is read (and consumed) before our partial leaves: CTA 0
      // of the cluster overwrites z only after receiving every CTA's partial
      zs[xb][tid] = zpre;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP_; ++w) s += red[rb2][w][tid];
      for (int rr = 0; rr < CL; ++rr)
        st_async_f64(cl_map(&xs[xb][q][tid], (unsigned)rr), s, cl_map(&xbar[xb], (unsigned)rr));
    }
  };
  // phase 2 of `tile`: totals from the exchange slot, new z, norm, w += y z (y re-read)
  auto phase2 = [&](int64_t tile) {
    const int st = (int)(tile % nst);
    const int64_t rb = r0 + tile * TR;
    const int xb = (int)(tile & 3);
    mbar_wait(&xbar[xb], (unsigned)((tile >> 2) & 1));
#pragma unroll
    for (int tr = 0; tr < TR; ++tr) {
      const int64_t row = rb + tr;
      if (row >= r1) continue;
      double dot = 0.0;
      for (int qq = 0; qq < CL; ++qq) dot += xs[xb][qq][tr];
      const double zn = fma(c1, zs[xb][tr], c2 * dot);
      norm = fma(zn, zn, norm);
      if (q == 0 && tid == 0) {
        a.z[row] = zn;
        if (a.acc != nullptr) a.acc[row] = fma(ca, zn, a.acc[row]);
      }
      const double* rowp = stage + ((int64_t)st * TR + tr) * stage_ld;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t cl = 2 * (tid + NT * p);
        if (cl < ncol) {
          const double2 y = *reinterpret_cast<const double2*>(rowp + cl);
          wv[p].x = fma(y.x, zn, wv[p].x);
          wv[p].y = fma(y.y, zn, wv[p].y);
        }
      }
    }
  };

  for (int64_t tile = 0; tile < ntiles; ++tile) {
    phase1(tile);
    if (tile >= 1) {
      phase2(tile - 1);
      __syncthreads();                       // stage of tile-1 fully read by every thread
      if (tid == 0 && tile - 1 + nst < ntiles) issue(tile - 1 + nst);
    }
  }
  if (ntiles >= 1) phase2(ntiles - 1);

  double* wp = a.wpart + g * C;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = 2 * (tid + NT * p);
    if (cl < ncol) wp[c0 + cl] = a.sx * wv[p].x;
    if (cl + 1 < ncol) wp[c0 + cl + 1] = a.sx * wv[p].y;
  }
  if (q == 0 && tid == 0) a.npart[g] = norm;
  cluster_sync_all2();                       // no CTA exits while peers may still address it
}

// ------------------------------------------------------------------ planning
namespace {
constexpr int64_t kMaxSlice = 4096;        // doubles per CTA slice (32 KB per staged row)
constexpr size_t kStageBudget = 192 * 1024;
constexpr size_t kWideBudget = 224 * 1024;   // + ~2.5 KB static shared memory <= 227 KB
}  // namespace

// Overrides (lsrn_ctx_set_option): rowpass_occ = 1 (one CTA per SM, the whole
// stage budget), rowpass_keep = 0/1 (force re-read / register tile), ...
bool plan_rowpass_bulk(int64_t R, int64_t C, int64_t ld, const double* Y, int nsm, RowPassPlan* p) {
  // 16-byte aligned rows and an even slice width: every bulk copy is a multiple of 16 bytes
  if (C <= 0 || (C & 1) || (ld & 1) || (reinterpret_cast<uintptr_t>(Y) & 15)) return false;
  // Rows up to 4096 doubles: one CTA per row slice, two CTAs per SM (while one CTA
  // sits in its per-tile barrier and row reductions the other streams; c2 long pass
  // 5.0 -> 6.4 TB/s, 99 % of the measured copy bandwidth, profiles/r01_rowpass_tune.jsonl).
  // Wider rows (c5 k = 1e4, c4's N-pass k = 2e4): clusters of CTAs with slices of
  // up to 8192 doubles, one CTA per SM (deeper rings), asynchronous partial-dot exchange.
  const bool wide = C > kMaxSlice;
  int64_t max_slice = wide ? 2 * kMaxSlice : kMaxSlice;
  const Overrides& ov = ovr();
  if (ov.rowpass_wide_slice > 0 && wide) max_slice = std::max<int64_t>(512, ov.rowpass_wide_slice);
  auto vpt_for = [](int64_t q) {
    int v = 1;
    while (512 * v < q) v = (v < 8) ? v * 2 : v + 4;              // 1, 2, 4, 8, 12, 16
    return v;
  };
  auto slice = [&](int n) { return (((C + n - 1) / n) + 1) & ~int64_t(1); };
  int cl = (int)((C + max_slice - 1) / max_slice);
  // Rows wider than two 5120-double slices (c4's N-pass, k = 2e4): the smallest
  // cluster whose slice fills >= 90 % of the threads' column pairs (masked pairs
  // cost issue slots, and the 16-pair instance spills).  Measured with
  // lsrn_debug_rowpass on 2e4 x 2e4 (profiles/r01_rowpass_shape.log): 3-CTA
  // clusters (6668-double slices, 16 pairs) 2.04 TB/s, 5-CTA (4000, 8 pairs)
  // 3.09 TB/s.  Up to 10240 (c5) the 2-CTA cluster stays best (4.44 TB/s against
  // <= 2.7 for 3-10 CTAs).
  // Rows of 16384-20480 doubles (c4's N-pass, k = 2e4): 2-CTA clusters of 512
  // threads x 10 column pairs (slices up to 10240 doubles), one CTA per SM, two
  // 1-row stages: 2e4 x 2e4 3.09 -> 3.99 TB/s (profiles/r01_rowpass_shape.log);
  // below 16384 the 256-thread 2-CTA plan is faster (16000: 5.77 vs 4.91 TB/s).
  // The rowpass_wide2 = 0 override disables it.
  // Rows of 8192-10240 doubles (c5, k = 1e4): ONE CTA of 512 threads x 10 column
  // pairs per row, no cluster and no partial-dot exchange, two 1-row stages (80 KB
  // each): 125000 x 1e4 4.44 -> 5.80 TB/s against the 2-CTA cluster pass
  // (profiles/r01_rowpass_shape.log).  The rowpass_wide1 = 0 override disables it.
  const bool wide1 = wide && C > 8192 && C <= 10240 && ov.rowpass_wide1 != 0;
  if (wide1) cl = 1;
  const bool wide2 = wide && C > 16384 && C <= 20480 && ov.rowpass_wide2 != 0;
  if (wide2) cl = 2;
  if (wide && C > 10240 && !wide2 && ov.rowpass_wide_slice <= 0) {
    for (int n = cl; n <= 16; ++n) {
      const int64_t q = slice(n);
      if ((double)q >= 0.9 * 512.0 * vpt_for(q)) {
        cl = n;
        break;
      }
    }
  }
  if (cl > 16) return false;
  const int64_t cq = slice(cl);
  const int vpt = (wide2 || wide1) ? 16 : vpt_for(cq);            // replaced by the 512-thread plans below
  if (vpt > 16) return false;                                     // no kernel instance: fallback
  // Wide rows: two CTAs (clusters) per SM with two 1-row stages each when two
  // slices fit in half of shared memory.  Each CTA's per-tile chain (block
  // reduction, exchange, stage release) is latency-bound, and the second CTA
  // hides it: c5 4.05 -> 4.43 TB/s (profiles/r01_rowpass_tune_c5c.jsonl) against
  // one CTA per SM with 4-5 stages.  Otherwise one CTA with (almost) all of shared
  // memory so that >= 3 stages stay in flight.  Overrides: rowpass_occ,
  // rowpass_budget_kb.
  int occ = 2;
  if (wide && 2 * (size_t)cq * 8 > kWideBudget / 2) occ = 1;
  if (wide2 || wide1) occ = 1;
  if (ov.rowpass_occ >= 1) occ = ov.rowpass_occ == 1 ? 1 : 2;
  size_t budget = wide ? (occ == 1 ? kWideBudget : kWideBudget / 2) : kStageBudget / occ;
  if (ov.rowpass_budget_kb > 0) budget = (size_t)ov.rowpass_budget_kb * 1024;
  int tr = (int)std::max<int64_t>(1, std::min<int64_t>(8, (int64_t)(budget / 3) / (cq * 8)));
  int t2 = 1;
  while (t2 * 2 <= tr) t2 *= 2;
  tr = t2;
  if (ov.rowpass_tr >= 1 && wide) tr = ov.rowpass_tr == 2 ? 2 : 1;   // wide rows: 1 or 2
  const size_t stage_bytes = (size_t)tr * cq * 8;
  int nst = (int)std::min<size_t>(kMaxStages, budget / stage_bytes);
  // one stage being reduced, one waiting for its refill, >= 1 in flight; with two
  // CTAs per SM on wide rows (tuning aid) two stages each still keep two in flight per SM
  if (nst < 3 && !(wide && (occ == 2 || wide2 || wide1 || tr == 2) && nst == 2)) return false;
  bool keep = vpt * tr <= (occ == 2 ? 4 : 16);
  if (ov.rowpass_keep >= 0) keep = ov.rowpass_keep != 0 && vpt * tr <= 16;
  p->keep = keep ? 1 : 0;
  p->occ = occ;
  // L2 prefetch distance (tiles beyond the shared-memory ring) for two-stage rings:
  // c5's 80 KB rows, 125000 x 1e4 through lsrn_debug_rowpass: pf 0 / 1 / 2 / 3 ->
  // 5.80 / 7.04 / 6.99 / 6.27 TB/s (profiles/r02_rowpass_pf.jsonl; a read-only stream
  // exceeds the 6.46 TB/s measured for a copy); deeper rings gain nothing (c2: 6.49 either way)
  p->pf = nst <= 2 ? 1 : 0;
  if (ov.rowpass_pf >= 0) p->pf = ov.rowpass_pf;
  p->nt = 256;
  // wide rows: pipelined asynchronous partial-dot exchange (override rowpass_asyncx = 0: cluster barrier per tile)
  p->async_x = 1;
  if (ov.rowpass_asyncx >= 0) p->async_x = ov.rowpass_asyncx != 0;
  int nclusters = (nsm * occ) / cl;
  if (nclusters < 1) nclusters = 1;
  const int64_t tiles = (R + tr - 1) / tr;
  if ((int64_t)nclusters > tiles) nclusters = (int)(tiles > 0 ? tiles : 1);
  p->vpt = vpt;
  p->cl = cl;
  p->tr = tr;
  p->nclusters = nclusters;
  p->vec = 2;
  p->rows_per_cluster = std::max<int64_t>(1, (R + nclusters - 1) / nclusters);
  p->bulk = 1;
  p->cq = cq;
  p->nst = nst;
  // Wide rows, override rowpass_nt = 512: 16 warps per CTA.  The c5 pass is
  // latency-bound (ncu: 12.5 % warps active; stalls on fixed-latency dependencies,
  // shared loads and the per-tile barrier, profiles/r01_ncu_c5_cluster.txt), but
  // neither 512 threads (3.76 TB/s) nor an mbarrier-only tile flow without the two
  // per-tile __syncthreads (3.50 TB/s) beat this kernel (4.05 TB/s,
  // profiles/r01_rowpass_tune_c5c.jsonl).
  if (wide1 && p->tr == 1) {
    p->nt = 512;
    p->vpt = 10;
    return true;
  }
  if (wide2 && p->async_x && p->tr == 1) {
    p->nt = 512;
    p->vpt = 10;
    return true;
  }
  if (cl > 1 && p->async_x) {
    int nt = 256;
    if (ov.rowpass_nt > 0) nt = ov.rowpass_nt == 512 ? 512 : 256;
    if (nt == 512) {
      int v = 4;
      while (v < 8 && 1024 * v < cq) v += 2;                     // 4, 6, 8 pairs per thread
      if (1024 * v >= cq && p->tr <= 2) {
        p->nt = 512;
        p->vpt = v;
      }
    }
  }
  return true;
}

template <int P, int TR, bool KEEP, int OCC, int NT = THREADS>
static cudaError_t launch_bulk_k(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  const size_t smem = (size_t)p.nst * TR * p.cq * 8;
  auto kern = rowpass_bulk_kernel<P, TR, KEEP, OCC, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p.cl > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.nclusters * p.cl));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, p.rows_per_cluster, p.cl, p.cq, p.nst, p.pf);
}

template <int P, int TR, int OCC, int NT = THREADS>
static cudaError_t launch_cluster_k(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  const size_t smem = (size_t)p.nst * TR * p.cq * 8;
  auto kern = rowpass_cluster_kernel<P, TR, OCC, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p.cl > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.nclusters * p.cl));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, p.rows_per_cluster, p.cl, p.cq, p.nst);
}

template <int P, int TR>
static cudaError_t launch_bulk_t(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  if (p.cl > 1 && p.async_x) {
    if (p.occ == 2) return launch_cluster_k<P, TR, 2>(a, p, st);
    return launch_cluster_k<P, TR, 1>(a, p, st);
  }
  if (p.occ == 2) {
    if constexpr (P * TR <= 4) {
      if (p.keep) return launch_bulk_k<P, TR, true, 2>(a, p, st);
    }
    return launch_bulk_k<P, TR, false, 2>(a, p, st);
  }
  if constexpr (P * TR <= 16) {
    if (p.keep) return launch_bulk_k<P, TR, true, 1>(a, p, st);
  }
  return launch_bulk_k<P, TR, false, 1>(a, p, st);
}

template <int P>
static cudaError_t launch_bulk_p(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  if constexpr (P >= 12) {     // slices > 4096 doubles: at most 2 rows per stage
    return p.tr == 1 ? launch_bulk_t<P, 1>(a, p, st) : launch_bulk_t<P, 2>(a, p, st);
  } else {
    switch (p.tr) {
      case 1: return launch_bulk_t<P, 1>(a, p, st);
      case 2: return launch_bulk_t<P, 2>(a, p, st);
      case 4: return launch_bulk_t<P, 4>(a, p, st);
      default: return launch_bulk_t<P, 8>(a, p, st);
    }
  }
}

template <int P>
static cudaError_t launch_cluster512(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  return p.tr == 1 ? launch_cluster_k<P, 1, 1, 512>(a, p, st) : launch_cluster_k<P, 2, 1, 512>(a, p, st);
}

cudaError_t launch_rowpass_bulk(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st) {
  if (p.nt == 512 && p.cl == 1) return launch_bulk_k<10, 1, false, 1, 512>(a, p, st);
  if (p.nt == 512) {
    switch (p.vpt) {
      case 4: return launch_cluster512<4>(a, p, st);
      case 6: return launch_cluster512<6>(a, p, st);
      case 10: return launch_cluster512<10>(a, p, st);
      default: return launch_cluster512<8>(a, p, st);
    }
  }
  switch (p.vpt) {
    case 1: return launch_bulk_p<1>(a, p, st);
    case 2: return launch_bulk_p<2>(a, p, st);
    case 4: return launch_bulk_p<4>(a, p, st);
    case 8: return launch_bulk_p<8>(a, p, st);
    case 12: return launch_bulk_p<12>(a, p, st);
    default: return launch_bulk_p<16>(a, p, st);
  }
}

}  // namespace lsrn
