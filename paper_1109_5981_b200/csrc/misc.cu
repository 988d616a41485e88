// Small helper kernels: fills, copies, the transposes around the SVD and the
// formation of N = V_r Sigma_r^-1 (Alg. 1 step 5; Alg. 2 step 5).
#include "common.cuh"
#include "kernels.h"

namespace lsrn {

namespace {
thread_local const Overrides* g_ovr = nullptr;
const Overrides kNoOverrides{};
}  // namespace
const Overrides& ovr() { return g_ovr ? *g_ovr : kNoOverrides; }
OverrideScope::OverrideScope(const Overrides* o) : prev(g_ovr) { g_ovr = o; }
OverrideScope::~OverrideScope() { g_ovr = prev; }

static unsigned grid_for(int64_t n, int threads = 256, int64_t cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

__global__ void fill_kernel(double* p, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void copy_scale_kernel(double* dst, const double* src, double scale, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = scale * src[i];
}

// 32 x 32 tiled transpose: src row-major rows x cols -> dst column-major rows x cols
__global__ void transpose_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                 double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
  }
}

__global__ void extract_r_kernel(const double* __restrict__ qr, int64_t ld, int64_t k, double* __restrict__ R) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % k, j = e / k;   // column-major (i, j)
    R[e] = (i <= j) ? qr[i + j * ld] : 0.0;
  }
}

// VT column-major k x k (row c = right singular vector c).  Nt row-major r x k.
__global__ void form_nt_kernel(const double* __restrict__ VT, const double* __restrict__ S, int64_t k, int64_t r,
                               double* __restrict__ Nt) {
  __shared__ double tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  // read VT[c, j] = VT[c + j*k]: coalesced along c
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t j = j0 + i, c = c0 + threadIdx.x;
    if (j < k && c < r) tile[i][threadIdx.x] = VT[c + j * k] / S[c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, j = j0 + threadIdx.x;
    if (j < k && c < r) Nt[c * k + j] = tile[threadIdx.x][i];
  }
}

// Jordan-Wielandt matrix of R (the upper triangle of the leading k x k block of
// the column-major QR factor qr, leading dim ld): JW = [[0, R^T], [R, 0]] (2k x 2k,
// column-major).  Only the lower triangle is referenced by syevdx(lower); the
// lower-left block R is written in full, everything else zero.
__global__ void build_jw_kernel(const double* __restrict__ qr, int64_t ld, int64_t k, double* __restrict__ JW) {
  const int64_t n2 = 2 * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2 * n2; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n2, j = e / n2;      // column-major (i, j)
    double v = 0.0;
    if (i >= k && j < k) {
      const int64_t a = i - k;                 // R[a][j], upper triangular
      v = (a <= j) ? qr[a + j * ld] : 0.0;
    }
    JW[e] = v;
  }
}

// N^T from the top-k eigenvectors of JW: eigenvalues ascending, so singular value
// c (descending) is eigenpair k-1-c; its right singular vector is sqrt(2) times
// the first k entries of the eigenvector.  Nt[c][j] = sqrt2 E[j, k-1-c] / S[k-1-c].
__global__ void form_nt_jw_kernel(const double* __restrict__ E, int64_t lde, const double* __restrict__ ev,
                                  int64_t k, int64_t r, double* __restrict__ Nt) {
  __shared__ double tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const double sq2 = 1.4142135623730951;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, j = j0 + threadIdx.x;     // read E[j, k-1-c]: coalesced along j
    if (j < k && c < r) tile[i][threadIdx.x] = sq2 * E[j + (k - 1 - c) * lde] / ev[k - 1 - c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, j = j0 + threadIdx.x;
    if (j < k && c < r) Nt[c * k + j] = tile[i][threadIdx.x];
  }
}

cudaError_t launch_build_jw(const double* qr, int64_t ld, int64_t k, double* JW, cudaStream_t st) {
  build_jw_kernel<<<grid_for(4 * k * k), 256, 0, st>>>(qr, ld, k, JW);
  return cudaGetLastError();
}

cudaError_t launch_form_nt_jw(const double* E, int64_t lde, const double* ev, int64_t k, int64_t r, double* Nt,
                              cudaStream_t st) {
  dim3 grid((unsigned)((k + 31) / 32), (unsigned)((r + 31) / 32));
  form_nt_jw_kernel<<<grid, dim3(32, 8), 0, st>>>(E, lde, ev, k, r, Nt);
  return cudaGetLastError();
}

cudaError_t launch_fill(double* p, double v, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fill_kernel<<<grid_for(n), 256, 0, st>>>(p, v, n);
  return cudaGetLastError();
}

cudaError_t launch_copy_scale(double* dst, const double* src, double scale, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  copy_scale_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, scale, n);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* src, int64_t rows, int64_t cols, double* dst, cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst);
  return cudaGetLastError();
}

cudaError_t launch_extract_r(const double* qr, int64_t ld, int64_t k, double* R, cudaStream_t st) {
  extract_r_kernel<<<grid_for(k * k), 256, 0, st>>>(qr, ld, k, R);
  return cudaGetLastError();
}

cudaError_t launch_form_nt(const double* VT, const double* S, int64_t k, int64_t r, double* Nt, cudaStream_t st) {
  dim3 grid((unsigned)((k + 31) / 32), (unsigned)((r + 31) / 32));
  form_nt_kernel<<<grid, dim3(32, 8), 0, st>>>(VT, S, k, r, Nt);
  return cudaGetLastError();
}

// V column-major k x k (column c = right singular vector c, as gesvdp returns it):
// Nt[c][j] = V[j + c k] / S[c] -- row c of Nt is column c of V, scaled.
__global__ void form_nt_v_kernel(const double* __restrict__ V, const double* __restrict__ S, int64_t k, int64_t r,
                                 double* __restrict__ Nt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < r * k; e += (int64_t)gridDim.x * blockDim.x)
    Nt[e] = V[e] / S[e / k];
}

cudaError_t launch_form_nt_v(const double* V, const double* S, int64_t k, int64_t r, double* Nt, cudaStream_t st) {
  form_nt_v_kernel<<<grid_for(r * k), 256, 0, st>>>(V, S, k, r, Nt);
  return cudaGetLastError();
}

// out[0] = sum A[i]^2, out[1] = sum B[i]^2 (i < n), in a fixed order: per-block partials
// (grid-stride, fixed tree) then one block over the partials.  part: 2 * SUMSQ_BLOCKS doubles.
constexpr int SUMSQ_BLOCKS = 296;
__global__ void sumsq2_part_kernel(const double* __restrict__ A, const double* __restrict__ B, int64_t n,
                                   double* __restrict__ part) {
  __shared__ double sh[2][8];
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a = fma(A[i], A[i], a);
    b = fma(B[i], B[i], b);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = a;
    sh[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      x += sh[0][w];
      y += sh[1][w];
    }
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
}
__global__ void sumsq2_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int b = 0; b < nb; ++b) {
      x += part[2 * b];
      y += part[2 * b + 1];
    }
    out[0] = x;
    out[1] = y;
  }
}

cudaError_t launch_sumsq2(const double* A, const double* B, int64_t n, double* part, double* out, cudaStream_t st) {
  sumsq2_part_kernel<<<SUMSQ_BLOCKS, 256, 0, st>>>(A, B, n, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sumsq2_final_kernel<<<1, 32, 0, st>>>(part, SUMSQ_BLOCKS, out);
  return cudaGetLastError();
}
int sumsq2_part_size() { return 2 * SUMSQ_BLOCKS; }

// flag[0] = 1.0 if any p[i] (i < n) is NaN or +-Inf (flag is only ever set, never
// cleared, so several arrays can be checked into one flag).
__global__ void check_finite_kernel(const double* __restrict__ p, int64_t n, double* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(p[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) flag[0] = 1.0;
}

cudaError_t launch_check_finite(const double* p, int64_t n, double* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  check_finite_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(p, n, flag);
  return cudaGetLastError();
}

}  // namespace lsrn
