// K2: dense Gaussian sketch on the fp64 tensor cores (DMMA.8x8x4).
//
// Computes the tall-form partial sketch of this shard (Alg. 1 step 3 "Ã = GA",
// P:487; Alg. 2 step 3 "Ã = AG", as Ã^T = G^T... see DESIGN.md "tall form"):
//   P[split][i][c] = sum_{j in split's rows} G[i, lo + j] * X[j][c],   i < s, c < k
// G is generated in-kernel (philox_bm.cuh) one BM x BK tile per k-block, into
// shared memory, and consumed by all warps of the CTA; X tiles are staged with
// cp.async (multi-stage ring).  A deterministic second kernel sums the split-K
// partials in fixed order and applies sigma_X and the sigma_I G_I Tikhonov block
// (§5).  No atomics: the sketch is bitwise run-to-run reproducible.
//
// CTA tile BM x BN = 64 x 256, BK = 16, 8 warps as 2 (M) x 4 (N), warp tile
// 32 x 64 = 4 x 8 DMMA fragments (64 fp64 accumulators per lane).  Every normal
// generated is reused BN = 256 times (RNG overhead ~ cost(normal) / BN of the
// FP64 pipe, which DMMA and DFMA share on sm_100a -- measured).
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "philox_bm.cuh"
#include "kernels.h"

namespace lsrn {

namespace sk {
constexpr int BM = 64, BN = 256, BK = 16, THREADS = 256, STAGES = 4;
constexpr int A_LD = BN + 8;   // padded row stride (doubles): 2 wavefronts per B-frag load
constexpr int G_LD = BK + 4;   // padded row stride (doubles): 2 wavefronts per A-frag load
constexpr int A_STAGE = BK * A_LD;
constexpr int G_TILE = BM * G_LD;
constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)(STAGES * A_STAGE + 2 * G_TILE);
}  // namespace sk

// VEC = 2: 16-byte cp.async (ld even, X 16-byte aligned); VEC = 1: 8-byte path.
template <int VEC>
__global__ void __launch_bounds__(sk::THREADS, 1)
sketch_dense_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k,
                    int64_t lo, int64_t s, uint64_t seed, int64_t rows_per_split,
                    double* __restrict__ out, int64_t out_split_stride, int accumulate) {
  using namespace sk;
  extern __shared__ __align__(16) double smem[];
  __shared__ double bmT[bm::TAB_SIZE];       // Box-Muller tables (philox_bm.cuh)
  double* As = smem;                         // [STAGES][BK][A_LD]
  double* Gs = smem + STAGES * A_STAGE;      // [2][BM][G_LD]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;   // 2 x 4 warps
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (int)((r_end - r_begin + BK - 1) / BK);
  const uint2 key = philox_key(seed);

  auto load_A = [&](int kb, int stage) {
    double* dst = As + stage * A_STAGE;
    const int64_t rbase = r_begin + (int64_t)kb * BK;
    if (VEC == 2) {
      // BK x BN / 2 = 2048 chunks of 16 B, 8 per thread
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
    } else {
#pragma unroll 4
      for (int t = 0; t < (BK * BN) / THREADS; ++t) {
        const int e = tid + t * THREADS;
        const int rr = e / BN, cc = e % BN;
        const int64_t gr = rbase + rr, gc = n0 + cc;
        const bool ok = gr < r_end && gc < k;
        cp_async8(dst + rr * A_LD + cc, ok ? (const void*)(X + gr * ld + gc) : (const void*)X, ok ? 8 : 0);
      }
    }
  };

  // G tile for k-block kb: BM x BK normals = 512 Box-Muller pairs, 2 per thread.
  auto gen_G = [&](int kb, int buf) {
    double* dst = Gs + buf * G_TILE;
    const int64_t jbase = lo + r_begin + (int64_t)kb * BK;
#pragma unroll
    for (int t = 0; t < (BM / 2 * BK) / THREADS; ++t) {
      const int p = tid + t * THREADS;
      const int qp = p / BK, kk = p % BK;
      double z0, z1;
      gaussian_pair(key, (uint64_t)(m0 / 2 + qp), (uint64_t)(jbase + kk), bmT, z0, z1);
      dst[(2 * qp) * G_LD + kk] = z0;
      dst[(2 * qp + 1) * G_LD + kk] = z1;
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  bm_load_table(bmT);
  __syncthreads();
  if (nk > 0) {
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
      if (st < nk) load_A(st, st);
      cp_async_commit();
    }
    gen_G(0, 0);

    for (int kb = 0; kb < nk; ++kb) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nxt = kb + STAGES - 1;
        if (nxt < nk) load_A(nxt, nxt % STAGES);
        cp_async_commit();
      }
      if (kb + 1 < nk) gen_G(kb + 1, (kb + 1) & 1);
      const double* as = As + (kb % STAGES) * A_STAGE;
      const double* gs = Gs + (kb & 1) * G_TILE;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        double a[4], b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          a[i] = gs[(wm * 32 + i * 8 + (lane >> 2)) * G_LD + ks * 4 + (lane & 3)];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          b[j] = as[(ks * 4 + (lane & 3)) * A_LD + wn * 64 + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma884(acc[i][j], a[i], b[j]);
      }
    }
    cp_async_wait<0>();
  }

  // epilogue: D fragment rows l/4, cols 2(l%4) + {0,1}
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

// out[i][c] = sx * sum_split P[split][i][c] + si * G[i, L + c]; thread per row pair.
__global__ void sketch_finish_kernel(const double* __restrict__ part, int nsplit, int64_t split_stride,
                                     int64_t s, int64_t k, double sx, double si, int64_t L,
                                     uint64_t seed, double* __restrict__ out) {
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  __syncthreads();
  const int64_t npair = (s + 1) / 2;
  const uint2 key = philox_key(seed);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npair * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / k, c = e % k;
    const int64_t i0 = 2 * q, i1 = 2 * q + 1;
    double v0 = 0.0, v1 = 0.0;
    for (int p = 0; p < nsplit; ++p) {
      v0 += part[p * split_stride + i0 * k + c];
      if (i1 < s) v1 += part[p * split_stride + i1 * k + c];
    }
    v0 *= sx;
    v1 *= sx;
    if (si != 0.0) {
      double z0, z1;
      gaussian_pair(key, (uint64_t)q, (uint64_t)(L + c), bmT, z0, z1);
      v0 += si * z0;
      v1 += si * z1;
    }
    out[i0 * k + c] = v0;
    if (i1 < s) out[i1 * k + c] = v1;
  }
}

__global__ void debug_gaussian_kernel(uint64_t seed, const int64_t* __restrict__ rows,
                                      const int64_t* __restrict__ cols, int64_t count,
                                      double* __restrict__ out) {
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  __syncthreads();
  const uint2 key = philox_key(seed);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    double z0, z1;
    gaussian_pair(key, (uint64_t)(rows[t] >> 1), (uint64_t)cols[t], bmT, z0, z1);
    out[t] = (rows[t] & 1) ? z1 : z0;
  }
}

// Box-Muller on given Philox words (4 per entry): mode 0 table-driven fp64, 1 libm,
// 2 integer fixed-point (the dense sketch's transform).
__global__ void debug_box_muller_kernel(const uint32_t* __restrict__ words, int64_t count, int mode,
                                        double* __restrict__ out) {
  __shared__ double bmT[bm::TAB_SIZE];
  __shared__ uint64_t bmI[bmi::TAB_WORDS];
  bm_load_table(bmT);
  bm_int_load_table(bmI);
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint4 o = make_uint4(words[4 * t], words[4 * t + 1], words[4 * t + 2], words[4 * t + 3]);
    double z0, z1;
    if (mode == 0)
      box_muller_tab(o, bmT, z0, z1);
    else if (mode == 2)
      box_muller_int(o, bmI, z0, z1);
    else
      box_muller_libm(o, z0, z1);
    out[2 * t] = z0;
    out[2 * t + 1] = z1;
  }
}

// ---------------------------------------------------------------- host side
size_t sketch_dense_smem() { return sk::SMEM_BYTES; }

cudaError_t launch_sketch_dense(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace sk;
  // Variant: the warp-specialized kernel (sketch_ws.cu) whenever its alignment
  // needs hold, else this kernel (odd ld / odd k / unaligned X); override
  // sketch_kernel = 1 forces this kernel (tests compare both).
  if (ovr().sketch_kernel != 1 && sketch_ws_supported(a)) return launch_sketch_ws(a, st);
  dim3 grid((unsigned)((a.k + BN - 1) / BN), (unsigned)((a.s + BM - 1) / BM), (unsigned)a.nsplit);
  const bool vec2 = (a.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
  cudaError_t e;
  if (vec2) {
    e = cudaFuncSetAttribute(sketch_dense_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    sketch_dense_kernel<2><<<grid, THREADS, SMEM_BYTES, st>>>(a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed,
                                                             a.rows_per_split, a.out, a.out_split_stride, a.accumulate);
  } else {
    e = cudaFuncSetAttribute(sketch_dense_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    sketch_dense_kernel<1><<<grid, THREADS, SMEM_BYTES, st>>>(a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed,
                                                             a.rows_per_split, a.out, a.out_split_stride, a.accumulate);
  }
  return cudaGetLastError();
}

cudaError_t launch_sketch_finish(const double* part, int nsplit, int64_t split_stride, int64_t s, int64_t k,
                                 double sx, double si, int64_t L, uint64_t seed, double* out, cudaStream_t st,
                                 int nsm) {
  const int64_t work = ((s + 1) / 2) * k;
  int64_t blocks = (work + 255) / 256;
  if (blocks > (int64_t)nsm * 16) blocks = (int64_t)nsm * 16;
  if (blocks < 1) blocks = 1;
  sketch_finish_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, nsplit, split_stride, s, k, sx, si, L, seed, out);
  return cudaGetLastError();
}

cudaError_t launch_debug_gaussian(uint64_t seed, const int64_t* rows, const int64_t* cols, int64_t count,
                                  double* out, cudaStream_t st) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  debug_gaussian_kernel<<<(unsigned)blocks, 256, 0, st>>>(seed, rows, cols, count, out);
  return cudaGetLastError();
}

cudaError_t launch_debug_box_muller(const uint32_t* words, int64_t count, int mode, double* out, cudaStream_t st) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  debug_box_muller_kernel<<<(unsigned)blocks, 256, 0, st>>>(words, count, mode, out);
  return cudaGetLastError();
}

void sketch_tile_counts(int64_t s, int64_t k, int64_t* mtiles, int64_t* ntiles, int64_t* bk) {
  int64_t bm, bn;
  sketch_ws_tile_dims(&bm, &bn, bk);     // the default (warp-specialized) kernel's tile
  *mtiles = (s + bm - 1) / bm;
  *ntiles = (k + bn - 1) / bn;
}

}  // namespace lsrn
