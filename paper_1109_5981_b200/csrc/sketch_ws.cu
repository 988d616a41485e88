// K2 v2: warp-specialized dense Gaussian sketch on the fp64 tensor cores.
//
// Same contract as sketch_dense_kernel (kernels.h SketchDenseArgs): the split-K
// partial  P[split][i][c] = sum_{j in split} G[i, lo + j] X[j][c]  of Alg. 1
// step 3 "Ã = G A" / Alg. 2 step 3 "Ã = A G" in the tall form,
// with G generated in-kernel (philox_bm.cuh, C9) and never stored.
//
// Why a second kernel: the first one (every warp loads, generates G and runs
// DMMA, one __syncthreads per k-block) kept the tensor pipe 62 % active on c2
// (profiles/r01_ncu_full_sketch_rowpass.json): after each barrier all warps sat
// in the latency-bound Box-Muller phase together.  Here the roles are split:
//   warpgroups 0-1 (8 producer warps, setmaxnreg 56): one lane streams X tiles
//     into a shared-memory ring with 1-D TMA bulk copies; all 256 threads
//     generate the 64 x 16 G tile of each k-block into a second ring;
//   warpgroups 2-3 (8 consumer warps, setmaxnreg 200): DMMA.8x8x4 on 32 x 64
//     warp tiles, never touching RNG, released stage by stage with mbarriers.
// Measured on c2 (profiles/r01_sketch_tune*.jsonl): with the RNG switched off the
// consumers reach 33.8 TFLOP/s (92 % of the DMMA peak); with it, 25.5 TFLOP/s.
// The Box-Muller FP64 instructions cost far more than their issue count: each
// competes with the consumers' DMMAs for the shared FP64 pipe.  Variants tried
// and rejected: 4 producer warps (66 ms vs 62.7), producers batching 4-8 pairs
// per thread (register-starved), X streamed by a consumer warp (serialises the
// consumers), batched RNG phases in a non-specialized kernel (sketch_batch.cu,
// 73.9 ms).
// The RNG shares the FP64 pipe with DMMA (measured), so each
// normal must be generated as few times as possible: the CTAs of a cluster of
// CL along N (same sketch rows, same k-range, different column tiles) need the
// SAME G tile, so CTA q generates rows [q BM/CL, (q+1) BM/CL) of it into its own
// ring and pushes that slice to the other CL-1 CTAs with async-proxy
// shared->shared bulk copies (cp.async.bulk.shared::cluster.shared::cta) that
// complete on the destination's `gfull` barrier; consumers release a G stage on
// every CTA of the cluster with plain remote arrives.  RNG work per CTA drops by
// CL.  (Without the sharing the consumers waited on the G ring 29 % of the time;
// distributing with st.shared::cluster + release/acquire.cluster barriers cost
// a MEMBAR.GPU / L1 invalidate per stage and ran 2x slower.)
//
// Requirements (else the caller uses sketch_dense_kernel): ld even, X 16-byte
// aligned, k even (every bulk row segment is a multiple of 16 bytes).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "philox_bm.cuh"

namespace lsrn {

namespace ws {
constexpr int BM = 64, BN = 256, BK = 16;
constexpr int NSX = 4, NSG = 4;             // X ring and G ring depth
constexpr int A_LD = BN + 8;                // padded smem row (doubles)
constexpr int G_LD = BK + 4;
constexpr int X_STAGE = BK * A_LD;          // doubles
constexpr int G_STAGE = BM * G_LD;
constexpr int NPROD = 256;                 // producer threads (2 warpgroups)
constexpr int THREADS = NPROD + 256;
constexpr int NCONS_WARPS = 8;
constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)(NSX * X_STAGE + NSG * G_STAGE) + 128;
}  // namespace ws

namespace {
LSRN_DEV unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
LSRN_DEV unsigned map_rank(const void* p, unsigned rank) {     // shared::cluster address in CTA `rank`
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
// remote arrive (default .release.cta semantics: only orders this thread's prior
// shared-memory reads, which is all a consumer release needs)
LSRN_DEV void mbar_arrive_remote(unsigned addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
// async-proxy copy of `bytes` from this CTA's shared memory into CTA-rank shared
// memory (dst, bar: shared::cluster addresses), completing tx on the remote barrier
LSRN_DEV void bulk_s2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar)
      : "memory");
}
LSRN_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
LSRN_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
LSRN_DEV void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
LSRN_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
}  // namespace

template <int CL>
__global__ void __launch_bounds__(ws::THREADS, 1)
sketch_ws_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k, int64_t lo, int64_t s,
                 uint64_t seed, int64_t rows_per_split, double* __restrict__ out, int64_t out_split_stride,
                 int diag, int accumulate) {
  using namespace ws;
  extern __shared__ __align__(128) double smem[];
  double* Xs = smem;                                   // [NSX][BK][A_LD]
  double* Gs = smem + NSX * X_STAGE;                   // [NSG][BM][G_LD]
  __shared__ uint64_t xfull[NSX], xempty[NSX], gfull[NSG], gempty[NSG];
  __shared__ double bmT[bm::TAB_SIZE];                 // Box-Muller tables (producers)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (r_end > r_begin) ? (int)((r_end - r_begin + BK - 1) / BK) : 0;

  const unsigned qrank = (CL > 1) ? cluster_rank() : 0u;
  constexpr int SLICE_ROWS = BM / CL;                  // G rows generated by this CTA
  constexpr unsigned SLICE_BYTES = (unsigned)(SLICE_ROWS * G_LD * sizeof(double));
  if (tid == 0) {
    for (int i = 0; i < NSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], NCONS_WARPS);
    }
    for (int i = 0; i < NSG; ++i) {
      mbar_init(&gfull[i], 1);                          // local producer leader (+ tx of CL-1 remote slices)
      mbar_init(&gempty[i], NCONS_WARPS * CL);          // one per consumer warp of each CTA of the cluster
    }
    mbar_fence_init();
  }
  if (CL > 1)
    cluster_sync_all();                                 // every CTA's barriers exist before remote traffic
  else
    __syncthreads();

  if (warp < NPROD / 32) {
    // ------------------------------------------------------------ producers
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    const uint2 key = philox_key(seed);
    const int ptid = tid;                                // 0..127
    for (int i = ptid; i < bm::TAB_SIZE; i += NPROD) bmT[i] = bm::kTable[i];
    named_bar(1, NPROD);
    const int64_t ncols = min((int64_t)BN, k - n0);      // even (k even, n0 multiple of BN)
    const unsigned seg_bytes = (unsigned)(ncols * 8);
    for (int kb = 0; kb < nk; ++kb) {
      const int sx = kb % NSX, sg = kb % NSG;
      const unsigned px = (unsigned)(((kb / NSX) & 1) ^ 1), pg = (unsigned)(((kb / NSG) & 1) ^ 1);
      const int64_t rbase = r_begin + (int64_t)kb * BK;
      const int nrow = (int)min((int64_t)BK, r_end - rbase);
      // X tile: rows rbase .. rbase + nrow of this N-tile (lane 0 of warp 0)
      if (warp == 0) {
        if (kb >= NSX) mbar_wait(&xempty[sx], px);
        double* dst = Xs + sx * X_STAGE;
        if (nrow < BK) {          // ragged K tail: zero the missing rows (0 x stale would risk NaN)
          for (int e = lane; e < (BK - nrow) * A_LD; e += 32) dst[nrow * A_LD + e] = 0.0;
          __syncwarp();
        }
        if (lane == 0) {
          mbar_arrive_expect_tx(&xfull[sx], seg_bytes * (unsigned)nrow);
          for (int rr = 0; rr < nrow; ++rr) bulk_g2s(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx]);
        }
      }
      // G stage sg must be free on every CTA of the cluster, and (CL > 1) the bulk
      // copies that last read our slice of it must have finished reading
      if (kb >= NSG) mbar_wait(&gempty[sg], pg);
      if (CL > 1) {
        if (ptid == 0) bulk_wait_read<NSG - 1>();
        named_bar(1, NPROD);
      }
      double* gdst = Gs + sg * G_STAGE;
      const int64_t jbase = lo + rbase;
      constexpr int PAIRS = (SLICE_ROWS / 2) * BK;       // pairs per CTA per k-block
#pragma unroll
      for (int t = 0; t < (PAIRS + NPROD - 1) / NPROD; ++t) {
        const int p = ptid + NPROD * t;
        if (PAIRS % NPROD == 0 || p < PAIRS) {
          const int qp = (int)qrank * (SLICE_ROWS / 2) + p / BK, kk = p % BK;
          double z0 = 0.0, z1 = 0.0;
          if (kk < nrow && !(diag & 1)) gaussian_pair(key, (uint64_t)(m0 / 2 + qp), (uint64_t)(jbase + kk), bmT, z0, z1);
          gdst[(2 * qp) * G_LD + kk] = z0;
          gdst[(2 * qp + 1) * G_LD + kk] = z1;
        }
      }
      if (CL > 1) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic -> async proxy
      named_bar(1, NPROD);                                // the whole slice is written
      if (ptid == 0) {
        mbar_arrive_expect_tx(&gfull[sg], SLICE_BYTES * (unsigned)(CL - 1));   // local slice: this arrive
        if (CL > 1) {
          const double* src = gdst + (int64_t)qrank * SLICE_ROWS * G_LD;
#pragma unroll
          for (unsigned r = 1; r < (unsigned)CL; ++r) {
            const unsigned dr = (qrank + r) % (unsigned)CL;
            bulk_s2s(map_rank(src, dr), src, SLICE_BYTES, map_rank(&gfull[sg], dr));
          }
          bulk_commit();
        }
      }
    }
    if (CL > 1) {
      if (ptid == 0) bulk_wait_read<0>();
      cluster_sync_all();                               // no CTA leaves while others may still signal it
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n");
  const int cw = warp - NPROD / 32;                      // 0..7
  const int wm = cw >> 2, wn = cw & 3;                   // 2 x 4 warps
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kb = 0; kb < nk; ++kb) {
    const int sx = kb % NSX, sg = kb % NSG;
    mbar_wait(&xfull[sx], (unsigned)((kb / NSX) & 1));
    mbar_wait(&gfull[sg], (unsigned)((kb / NSG) & 1));
    const double* as = Xs + sx * X_STAGE;
    const double* gs = Gs + sg * G_STAGE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = gs[(wm * 32 + i * 8 + (lane >> 2)) * G_LD + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = as[(ks * 4 + (lane & 3)) * A_LD + wn * 64 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&xempty[sx]);
      if (CL == 1) {
        mbar_arrive(&gempty[sg]);
      } else {
#pragma unroll
        for (unsigned r = 0; r < (unsigned)CL; ++r) mbar_arrive_remote(map_rank(&gempty[sg], r));
      }
    }
  }

  double* o = out + (int64_t)blockIdx.z * out_split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (gi >= s) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gc = n0 + wn * 64 + j * 8 + 2 * (lane & 3);
      if (gc + 1 < k) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (accumulate) {
          const double2 w = *reinterpret_cast<const double2*>(o + gi * k + gc);
          v.x = w.x + v.x;
          v.y = w.y + v.y;
        }
        *reinterpret_cast<double2*>(o + gi * k + gc) = v;
      } else if (gc < k) {
        o[gi * k + gc] = accumulate ? o[gi * k + gc] + acc[i][j][0] : acc[i][j][0];
      }
    }
  }
  if (CL > 1) cluster_sync_all();
}

bool sketch_ws_supported(const SketchDenseArgs& a) {
  return (a.ld % 2 == 0) && (a.k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
}

template <int CL>
static cudaError_t launch_ws_t(const SketchDenseArgs& a, dim3 grid, cudaStream_t st) {
  using namespace ws;
  cudaError_t e = cudaFuncSetAttribute(sketch_ws_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // LSRN_SKETCH_DIAG (timing experiments only, results are wrong): 1 = skip the RNG
  int diag = 0;
  if (const char* e = std::getenv("LSRN_SKETCH_DIAG")) diag = std::atoi(e);
  return cudaLaunchKernelEx(&cfg, sketch_ws_kernel<CL>, a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed,
                            a.rows_per_split, a.out, a.out_split_stride, diag, a.accumulate);
}

// Cluster size along N: the largest of {max_cl, ..., 2} dividing the N-tile count.
// LSRN_SKETCH_MAXCL (tuning aid) caps it.  Default 2, measured on c2
// (profiles/r01_sketch_tune.jsonl): CL = 1/2/4/8 -> 82.6/69.3/72.3/83.0 ms; larger
// clusters cut the RNG further but leave SMs idle (whole clusters must fit in a
// GPC: with CL = 8 only 76 % of the SM-cycles were active).
int sketch_ws_cluster(int64_t k) {
  const int64_t nt = (k + ws::BN - 1) / ws::BN;
  int max_cl = 2;
  if (const char* e = std::getenv("LSRN_SKETCH_MAXCL")) max_cl = std::atoi(e);
  for (int cl : {8, 4, 2})
    if (cl <= max_cl && nt % cl == 0) return cl;
  return 1;
}

cudaError_t launch_sketch_ws(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace ws;
  dim3 grid((unsigned)((a.k + BN - 1) / BN), (unsigned)((a.s + BM - 1) / BM), (unsigned)a.nsplit);
  switch (sketch_ws_cluster(a.k)) {
    case 8: return launch_ws_t<8>(a, grid, st);
    case 4: return launch_ws_t<4>(a, grid, st);
    case 2: return launch_ws_t<2>(a, grid, st);
    default: return launch_ws_t<1>(a, grid, st);
  }
}

}  // namespace lsrn
