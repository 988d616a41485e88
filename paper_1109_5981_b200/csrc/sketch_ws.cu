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
//   warpgroup 0 (4 warps, setmaxnreg 96): one lane streams X tiles into a
//     shared-memory ring with 1-D TMA bulk copies; all 128 threads generate the
//     64 x 16 G tile of each k-block into a second ring (4 pairs per thread);
//   warpgroups 1-2 (8 warps, setmaxnreg 200): DMMA.8x8x4 on 32 x 64 warp tiles,
//     never touching RNG, released stage by stage with mbarriers.
// The RNG still shares the FP64 pipe with DMMA (measured) but now
// runs concurrently with it instead of in a separate phase.
//
// Requirements (else the caller uses sketch_dense_kernel): ld even, X 16-byte
// aligned, k even (every bulk row segment is a multiple of 16 bytes).
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
constexpr int THREADS = 384;
constexpr int NCONS_WARPS = 8;
constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)(NSX * X_STAGE + NSG * G_STAGE) + 128;
}  // namespace ws

__global__ void __launch_bounds__(ws::THREADS, 1)
sketch_ws_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k, int64_t lo, int64_t s,
                 uint64_t seed, int64_t rows_per_split, double* __restrict__ out, int64_t out_split_stride) {
  using namespace ws;
  extern __shared__ __align__(128) double smem[];
  double* Xs = smem;                                   // [NSX][BK][A_LD]
  double* Gs = smem + NSX * X_STAGE;                   // [NSG][BM][G_LD]
  __shared__ uint64_t xfull[NSX], xempty[NSX], gfull[NSG], gempty[NSG];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (r_end > r_begin) ? (int)((r_end - r_begin + BK - 1) / BK) : 0;

  if (tid == 0) {
    for (int i = 0; i < NSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], NCONS_WARPS);
    }
    for (int i = 0; i < NSG; ++i) {
      mbar_init(&gfull[i], 4);                          // one arrival per producer warp
      mbar_init(&gempty[i], NCONS_WARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n");
    const uint2 key = philox_key(seed);
    const int ptid = tid;                                // 0..127
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
      // G tile: 64 x 16 normals = 512 Box-Muller pairs, 4 per producer thread
      if (kb >= NSG) mbar_wait(&gempty[sg], pg);
      double* gdst = Gs + sg * G_STAGE;
      const int64_t jbase = lo + rbase;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int p = ptid + 128 * t;
        const int qp = p / BK, kk = p % BK;
        double z0 = 0.0, z1 = 0.0;
        if (kk < nrow) gaussian_pair(key, (uint64_t)(m0 / 2 + qp), (uint64_t)(jbase + kk), z0, z1);
        gdst[(2 * qp) * G_LD + kk] = z0;
        gdst[(2 * qp + 1) * G_LD + kk] = z1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&gfull[sg]);           // release: this warp's G stores
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n");
  const int cw = warp - 4;                               // 0..7
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
      mbar_arrive(&gempty[sg]);
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
        *reinterpret_cast<double2*>(o + gi * k + gc) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (gc < k) {
        o[gi * k + gc] = acc[i][j][0];
      }
    }
  }
}

bool sketch_ws_supported(const SketchDenseArgs& a) {
  return (a.ld % 2 == 0) && (a.k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
}

cudaError_t launch_sketch_ws(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace ws;
  dim3 grid((unsigned)((a.k + BN - 1) / BN), (unsigned)((a.s + BM - 1) / BM), (unsigned)a.nsplit);
  cudaError_t e = cudaFuncSetAttribute(sketch_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  sketch_ws_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed, a.rows_per_split,
                                                      a.out, a.out_split_stride);
  return cudaGetLastError();
}

}  // namespace lsrn
