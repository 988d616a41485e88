// K2 v3: dense Gaussian sketch with batched G generation phases.
//
// Same contract as sketch_dense_kernel (kernels.h SketchDenseArgs): the split-K
// partial  P[split][i][c] = sum_{j in split} G[i, lo + j] X[j][c]  of Alg. 1
// step 3 "Ã = G A" / Alg. 2 step 3 "Ã = A G" in the tall form,
// G generated in-kernel (philox_bm.cuh, C9) and never stored in HBM.
//
// Why: the Box-Muller arithmetic runs on the same FP64 pipe as DMMA.  Measured
// on c2 (profiles/r01_sketch_tune*.jsonl):
//   * v1 (all warps generate one 64 x 16 G tile per k-block, 2 pairs per
//     thread): the RNG phase after each barrier is latency-bound -> 62 % of peak;
//   * v2 (warp-specialized producers generating concurrently with DMMA): the
//     producers' FP64 instructions starve behind the consumers' DMMAs and the
//     consumers wait on the G ring -> 69 %; with no RNG at all the same kernel
//     reaches 92 % (33.8 TFLOP/s).
// Here all 8 warps generate the G tile of SK = 8 k-blocks at once (16 pairs per
// thread: enough independent chains to keep the FP64 pipe full), then run the
// DMMA loop over those 8 k-blocks with no RNG in it.  X tiles keep streaming
// through a 4-stage cp.async ring across the phases.
//
// CTA tile 64 x 256, BK = 16, 8 warps as 2 x 4, warp tile 32 x 64 (64 fp64
// accumulators per lane).  Requirements: ld even and X 16-byte aligned (else
// sketch_dense_kernel).
#include "common.cuh"
#include "kernels.h"
#include "philox_bm.cuh"

namespace lsrn {

namespace sb {
constexpr int BM = 64, BN = 256, BK = 16, THREADS = 256, STAGES = 4, SK = 8;
constexpr int A_LD = BN + 8;             // padded X row (doubles)
constexpr int G_LD = SK * BK + 4;        // padded G row (doubles): 2 wavefronts per fragment load
constexpr int A_STAGE = BK * A_LD;
constexpr int G_TILE = BM * G_LD;
constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)(STAGES * A_STAGE + G_TILE);
}  // namespace sb

__global__ void __launch_bounds__(sb::THREADS, 1)
sketch_batch_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k, int64_t lo, int64_t s,
                    uint64_t seed, int64_t rows_per_split, double* __restrict__ out, int64_t out_split_stride, int accumulate) {
  using namespace sb;
  extern __shared__ __align__(16) double smem[];
  __shared__ double bmT[bm::TAB_SIZE];
  double* As = smem;                         // [STAGES][BK][A_LD]
  double* Gs = smem + STAGES * A_STAGE;      // [BM][G_LD]: G for SK k-blocks

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (r_end > r_begin) ? (int)((r_end - r_begin + BK - 1) / BK) : 0;
  const uint2 key = philox_key(seed);

  auto load_A = [&](int kb, int stage) {
    double* dst = As + stage * A_STAGE;
    const int64_t rbase = r_begin + (int64_t)kb * BK;
#pragma unroll
    for (int t = 0; t < (BK * BN / 2) / THREADS; ++t) {
      const int chunk = tid + t * THREADS;
      const int rr = chunk / (BN / 2), cc = (chunk % (BN / 2)) * 2;
      const int64_t gr = rbase + rr, gc = n0 + cc;
      int bytes = 0;
      const double* src = X;
      if (gr < r_end && gc < k) {
        bytes = (gc + 1 < k) ? 16 : 8;
        src = X + gr * ld + gc;
      }
      cp_async16(dst + rr * A_LD + cc, src, bytes);
    }
  };

  // G for k-blocks kb0 .. kb0 + SK - 1: BM x SK*BK normals = 4096 pairs, 16 per thread
  auto gen_G = [&](int kb0) {
    const int64_t jbase = lo + r_begin + (int64_t)kb0 * BK;
    const int64_t jmax = lo + r_end;
#pragma unroll 4
    for (int t = 0; t < (BM / 2) * SK * BK / THREADS; ++t) {
      const int p = tid + t * THREADS;
      const int qp = p / (SK * BK), kk = p % (SK * BK);
      double z0 = 0.0, z1 = 0.0;
      if (jbase + kk < jmax) gaussian_pair(key, (uint64_t)(m0 / 2 + qp), (uint64_t)(jbase + kk), bmT, z0, z1);
      Gs[(2 * qp) * G_LD + kk] = z0;
      Gs[(2 * qp + 1) * G_LD + kk] = z1;
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  bm_load_table(bmT);
  if (nk > 0) {
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
      if (st < nk) load_A(st, st);
      cp_async_commit();
    }
    for (int kb = 0; kb < nk; ++kb) {
      if (kb % SK == 0) {
        __syncthreads();                     // previous batch fully consumed (and bmT visible)
        gen_G(kb);
      }
      cp_async_wait<STAGES - 2>();
      __syncthreads();                       // X stage kb landed for all; G batch visible
      {
        const int nxt = kb + STAGES - 1;
        if (nxt < nk) load_A(nxt, nxt % STAGES);
        cp_async_commit();
      }
      const double* as = As + (kb % STAGES) * A_STAGE;
      const double* gs = Gs + (kb % SK) * BK;
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
    }
    cp_async_wait<0>();
  }

  double* o = out + (int64_t)blockIdx.z * out_split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (gi >= s) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gc = n0 + wn * 64 + j * 8 + 2 * (lane & 3);
      double* p = o + gi * k + gc;
      if (gc + 1 < k && (k % 2 == 0)) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (accumulate) {
          const double2 w = *reinterpret_cast<const double2*>(p);
          v.x = w.x + v.x;
          v.y = w.y + v.y;
        }
        *reinterpret_cast<double2*>(p) = v;
      } else {
        if (gc < k) p[0] = accumulate ? p[0] + acc[i][j][0] : acc[i][j][0];
        if (gc + 1 < k) p[1] = accumulate ? p[1] + acc[i][j][1] : acc[i][j][1];
      }
    }
  }
}

bool sketch_batch_supported(const SketchDenseArgs& a) {
  return (a.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
}

cudaError_t launch_sketch_batch(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace sb;
  dim3 grid((unsigned)((a.k + BN - 1) / BN), (unsigned)((a.s + BM - 1) / BM), (unsigned)a.nsplit);
  cudaError_t e = cudaFuncSetAttribute(sketch_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  sketch_batch_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed,
                                                         a.rows_per_split, a.out, a.out_split_stride, a.accumulate);
  return cudaGetLastError();
}

}  // namespace lsrn
