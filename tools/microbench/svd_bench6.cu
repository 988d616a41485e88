// SVD routes for the c2 sketch shape (s = 4000, k = 2000, rank 1800, sigma 1 -> 1e-4
// on the first 1800): R from geqrf, then (a) syevdx on the Jordan-Wielandt matrix of
// R (the library's route for k < 4096), (b) gesvdj (one-sided Jacobi) on R, (c) gesvd
// on R.  Time and the relative sigma difference from (a) over the top 1800, and the
// largest of the 200 "null" sigma / sigma_1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench6.cu -lcusolver -lcublas -o svd_bench6
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s line %d code %d\"}\n", #x, __LINE__, (int)e); exit(1);} } while (0)
static cudaEvent_t e0, e1;
static void tstart() { cudaEventRecord(e0); }
static float tstop() { cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms; }

__global__ void gen(double* A, int64_t rows, int64_t cols, unsigned seed, double scale_exp, int64_t nscale) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * cols; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = idx / rows;
    unsigned long long h = (unsigned long long)idx * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    double u = ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double sc = nscale > 1 ? pow(10.0, scale_exp * (double)j / (double)(nscale - 1)) : 1.0;
    A[idx] = (u - 0.5) * sc;
  }
}
__global__ void upper(const double* A, int64_t lda, int64_t k, double* R) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < k * k; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % k, j = idx / k;
    R[idx] = i <= j ? A[j * lda + i] : 0.0;
  }
}
__global__ void build_jw(const double* R, int64_t k, double* J) {
  const int64_t n = 2 * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % n, j = idx / n;
    double v = 0.0;
    if (i >= k && j < k) v = R[j * k + (i - k)];   // lower-left block = R
    J[idx] = v;
  }
}

int main() {
  const int64_t s = 4000, k = 2000, r = 1800;
  cusolverDnHandle_t h; cublasHandle_t cb; cusolverDnParams_t prm;
  CK(cusolverDnCreate(&h)); CK(cublasCreate(&cb)); CK(cusolverDnCreateParams(&prm));
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  double *L, *Rr, *A, *tau, *R, *R2, *J, *S, *U, *V; int* info;
  CK(cudaMalloc(&L, 8 * s * r)); CK(cudaMalloc(&Rr, 8 * r * k)); CK(cudaMalloc(&A, 8 * s * k)); CK(cudaMalloc(&tau, 8 * k));
  CK(cudaMalloc(&R, 8 * k * k)); CK(cudaMalloc(&R2, 8 * k * k)); CK(cudaMalloc(&J, 8 * 4 * k * k)); CK(cudaMalloc(&S, 8 * 2 * k));
  CK(cudaMalloc(&U, 8 * k * k)); CK(cudaMalloc(&V, 8 * 4 * k * k)); CK(cudaMalloc(&info, 16));
  gen<<<4096, 256>>>(L, s, r, 1u, -4.0, r);     // s x r, graded columns
  gen<<<4096, 256>>>(Rr, r, k, 2u, 0.0, 1);     // r x k
  const double one = 1.0, zero = 0.0;
  CK(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, s, k, r, &one, L, s, Rr, r, &zero, A, s));   // rank r
  size_t dws = 0, hws = 0;
  CK(cusolverDnXgeqrf_bufferSize(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws));
  void* dw; CK(cudaMalloc(&dw, dws)); std::vector<char> hw(hws + 16);
  CK(cusolverDnXgeqrf(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, dw, dws, hw.data(), hws, info));
  upper<<<4096, 256>>>(A, s, k, R);
  cudaDeviceSynchronize();
  // (a) JW syevdx, top k eigenpairs
  std::vector<double> sa(k), sb(k), sc(k);
  {
    int64_t meig = 0; double vl = 0, vu = 0; size_t d2 = 0, h2 = 0;
    CK(cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k,
                                    CUDA_R_64F, J, 2 * k, &vl, &vu, k + 1, 2 * k, &meig, CUDA_R_64F, S, CUDA_R_64F, &d2, &h2));
    void* w2; CK(cudaMalloc(&w2, d2)); std::vector<char> hw2(h2 + 16);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      build_jw<<<4096, 256>>>(R, k, J);
      tstart();
      CK(cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k, CUDA_R_64F, J,
                           2 * k, &vl, &vu, k + 1, 2 * k, &meig, CUDA_R_64F, S, CUDA_R_64F, w2, d2, hw2.data(), h2, info));
      best = std::min(best, tstop());
    }
    std::vector<double> ev(k);
    cudaMemcpy(ev.data(), S, 8 * k, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < k; ++i) sa[i] = std::max(0.0, ev[k - 1 - i]);
    printf("{\"route\": \"jw_syevdx\", \"ms\": %.2f}\n", best);
    cudaFree(w2);
  }
  // (b) gesvdj on R
  {
    gesvdjInfo_t gi; CK(cusolverDnCreateGesvdjInfo(&gi));
    int lw = 0;
    CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, R2, k, S, U, k, V, k, &lw, gi));
    double* w3; CK(cudaMalloc(&w3, 8 * (size_t)lw));
    float best = 1e30f;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(R2, R, 8 * k * k, cudaMemcpyDeviceToDevice);
      tstart();
      CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, R2, k, S, U, k, V, k, w3, lw, info, gi));
      best = std::min(best, tstop());
    }
    int inf = 0; cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost);
    double res = 0; int sw = 0; cusolverDnXgesvdjGetResidual(h, gi, &res); cusolverDnXgesvdjGetSweeps(h, gi, &sw);
    cudaMemcpy(sb.data(), S, 8 * k, cudaMemcpyDeviceToHost);
    double md = 0, nul = 0;
    for (int64_t i = 0; i < r; ++i) md = std::max(md, fabs(sb[i] - sa[i]) / sa[i]);
    for (int64_t i = r; i < k; ++i) nul = std::max(nul, sb[i] / sb[0]);
    printf("{\"route\": \"gesvdj_R\", \"ms\": %.2f, \"info\": %d, \"sweeps\": %d, \"residual\": %.3e, \"sigma_maxrel_vs_jw\": %.3e, \"null_max_over_s1\": %.3e}\n",
           best, inf, sw, res, md, nul);
    cudaFree(w3);
  }
  // (c) gesvd on R
  {
    size_t d4 = 0, h4 = 0;
    CK(cusolverDnXgesvd_bufferSize(h, prm, 'N', 'A', k, k, CUDA_R_64F, R2, k, CUDA_R_64F, S, CUDA_R_64F, nullptr, 1, CUDA_R_64F, V, k,
                                   CUDA_R_64F, &d4, &h4));
    void* w4; CK(cudaMalloc(&w4, d4)); std::vector<char> hw4(h4 + 16);
    float best = 1e30f;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(R2, R, 8 * k * k, cudaMemcpyDeviceToDevice);
      tstart();
      CK(cusolverDnXgesvd(h, prm, 'N', 'A', k, k, CUDA_R_64F, R2, k, CUDA_R_64F, S, CUDA_R_64F, nullptr, 1, CUDA_R_64F, V, k, CUDA_R_64F,
                          w4, d4, hw4.data(), h4, info));
      best = std::min(best, tstop());
    }
    cudaMemcpy(sc.data(), S, 8 * k, cudaMemcpyDeviceToHost);
    double md = 0, nul = 0, nula = 0;
    for (int64_t i = 0; i < r; ++i) md = std::max(md, fabs(sc[i] - sa[i]) / sa[i]);
    for (int64_t i = r; i < k; ++i) { nul = std::max(nul, sc[i] / sc[0]); nula = std::max(nula, sa[i] / sa[0]); }
    printf("{\"route\": \"gesvd_R\", \"ms\": %.2f, \"sigma_maxrel_vs_jw\": %.3e, \"null_max_over_s1\": %.3e, \"jw_null_max_over_s1\": %.3e}\n", best, md, nul, nula);
  }
  return 0;
}
