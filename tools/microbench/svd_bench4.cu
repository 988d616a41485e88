// SVD-stage options for the full-rank large-k sketches (c5: k = 1e4, c4: k = 2e4),
// outside the hot path (Alg. 1 step 4; cost 2sn^2 + 11n^3).
// R = the R factor of an s x k (s = 2k) Gaussian with columns scaled 1 -> 1e-5
// (c5's recipe).  Per option: time, and intrinsic accuracy
//   resid = ||R V - U S||_F / ||R||_F,  orth = ||V^T V - I||_F / sqrt(k),
// plus sigma agreement with the Jordan-Wielandt reference where it exists (k <= 16384).
// Options: syevdx on the Jordan-Wielandt matrix (current path), gesvdp (polar
// decomposition + symmetric eigensolver) on R, and the building blocks of a
// hand-rolled QDWH polar iteration (syrk / potrf / trsm / gemm) and a syevd of
// a k x k symmetric matrix.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench4.cu -lcusolver -lcublas -o svd_bench4
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

__global__ void gen(double* A, int64_t s, int64_t k, unsigned seed) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t tot = s * k;
  for (; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = idx / s;
    unsigned long long h = (unsigned long long)idx * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    double u = ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    A[idx] = (u - 0.5) * pow(10.0, -5.0 * (double)j / (double)(k - 1));
  }
}

__global__ void extract_r(const double* A, int64_t lda, int64_t k, double* R) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; idx < k * k; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % k, j = idx / k;
    R[idx] = i <= j ? A[j * lda + i] : 0.0;
  }
}

__global__ void build_jw(const double* R, int64_t k, double* J) {   // lower triangle of [[0, R^T],[R, 0]]
  int64_t n = 2 * k;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; idx < n * n; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % n, j = idx / n;
    double v = 0.0;
    if (i >= k && j < k) v = R[j * k + (i - k)];   // block (2,1) = R
    J[idx] = v;
  }
}

__global__ void scale_cols(double* U, const double* S, int64_t k) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; idx < k * k; idx += (int64_t)gridDim.x * blockDim.x) U[idx] *= S[idx / k];
}

__global__ void sub_eye(double* M, int64_t k) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < k) M[i * k + i] -= 1.0;
}

int main(int argc, char** argv) {
  const int64_t k = argc > 1 ? atoll(argv[1]) : 10000;
  const int64_t s = 2 * k;
  cusolverDnHandle_t h;
  cublasHandle_t cb;
  cusolverDnParams_t prm;
  CK(cusolverDnCreate(&h));
  CK(cublasCreate(&cb));
  CK(cusolverDnCreateParams(&prm));
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double *A, *tau, *R, *W, *S, *U, *V, *M;
  int* info;
  CK(cudaMalloc(&A, sizeof(double) * s * k));
  CK(cudaMalloc(&tau, sizeof(double) * k));
  CK(cudaMalloc(&R, sizeof(double) * k * k));
  CK(cudaMalloc(&S, sizeof(double) * 2 * k));
  CK(cudaMalloc(&U, sizeof(double) * k * k));
  CK(cudaMalloc(&V, sizeof(double) * k * k));
  CK(cudaMalloc(&M, sizeof(double) * k * k));
  CK(cudaMalloc(&info, 16));
  gen<<<4096, 256>>>(A, s, k, 7u);
  size_t dws = 0, hws = 0;
  CK(cusolverDnXgeqrf_bufferSize(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws));
  void* dw;
  CK(cudaMalloc(&dw, dws));
  std::vector<char> hw(hws + 16);
  tstart();
  CK(cusolverDnXgeqrf(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, dw, dws, hw.data(), hws, info));
  printf("{\"k\": %lld, \"geqrf_ms\": %.1f}\n", (long long)k, tstop());
  fflush(stdout);
  cudaFree(dw);
  extract_r<<<4096, 256>>>(A, s, k, R);
  CK(cudaFree(A));
  const double one = 1, zero = 0, mone = -1;
  double rn;
  CK(cublasDnrm2(cb, k * k, R, 1, &rn));
  auto accuracy = [&](const char* name, float ms, const double* Uc, const double* Vc, const std::vector<double>* ref) {
    // resid = ||R V - U S||_F / ||R||_F ; orth = ||V^T V - I||_F / sqrt(k)
    CK(cudaMemcpy(M, Uc, sizeof(double) * k * k, cudaMemcpyDeviceToDevice));
    scale_cols<<<4096, 256>>>(M, S, k);
    CK(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, &one, R, k, Vc, k, &mone, M, k));
    double res;
    CK(cublasDnrm2(cb, k * k, M, 1, &res));
    CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, k, &one, Vc, k, Vc, k, &zero, M, k));
    sub_eye<<<(k + 255) / 256, 256>>>(M, k);
    double orth;
    CK(cublasDnrm2(cb, k * k, M, 1, &orth));
    std::vector<double> sg(k);
    CK(cudaMemcpy(sg.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
    double se = 0.0;
    if (ref)
      for (int64_t i = 0; i < k; ++i) se = std::max(se, fabs(sg[i] - (*ref)[i]) / (*ref)[i]);
    printf("{\"k\": %lld, \"svd\": \"%s\", \"ms\": %.1f, \"resid\": %.3e, \"orth\": %.3e, \"sigma_maxrel_vs_jw\": %.3e, "
           "\"smax\": %.6e, \"smin\": %.6e}\n",
           (long long)k, name, ms, res / rn, orth / sqrt((double)k), se, sg[0], sg[k - 1]);
    fflush(stdout);
  };
  std::vector<double> refS;
  // 1. Jordan-Wielandt syevdx (the current path), k <= 16384
  if (2 * k <= 32768) {
    double* J;
    CK(cudaMalloc(&J, sizeof(double) * 4 * k * k));
    build_jw<<<8192, 256>>>(R, k, J);
    double vl = 0, vu = 0;
    int64_t meig = 0;
    CK(cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k,
                                    CUDA_R_64F, J, 2 * k, &vl, &vu, k + 1, 2 * k, &meig, CUDA_R_64F, S, CUDA_R_64F, &dws,
                                    &hws));
    CK(cudaMalloc(&dw, dws));
    hw.resize(hws + 16);
    tstart();
    CK(cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k, CUDA_R_64F,
                         J, 2 * k, &vl, &vu, k + 1, 2 * k, &meig, CUDA_R_64F, S, CUDA_R_64F, dw, dws, hw.data(), hws,
                         info));
    float ms = tstop();
    cudaFree(dw);
    // eigenvalues ascending -> sigma descending; vectors [v; u]/sqrt2: V = sqrt2 * top half, U = sqrt2 * bottom half
    std::vector<double> ev(k);
    CK(cudaMemcpy(ev.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
    refS.resize(k);
    for (int64_t i = 0; i < k; ++i) refS[i] = ev[k - 1 - i];
    CK(cudaMemcpy(S, refS.data(), sizeof(double) * k, cudaMemcpyHostToDevice));
    const double r2 = sqrt(2.0);
    for (int64_t i = 0; i < k; ++i) {   // column k-1-i of J's eigenvectors -> column i
      CK(cudaMemcpy(V + i * k, J + (k - 1 - i) * 2 * k, sizeof(double) * k, cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(U + i * k, J + (k - 1 - i) * 2 * k + k, sizeof(double) * k, cudaMemcpyDeviceToDevice));
    }
    CK(cublasDscal(cb, k * k, &r2, V, 1));
    CK(cublasDscal(cb, k * k, &r2, U, 1));
    cudaFree(J);
    accuracy("syevdx_JW", ms, U, V, nullptr);
  }
  // 2. gesvdp on R (econ): polar decomposition + eigensolver
  {
    CK(cudaMemcpy(M, R, sizeof(double) * k * k, cudaMemcpyDeviceToDevice));
    CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, M, k, CUDA_R_64F, S, CUDA_R_64F,
                                    U, k, CUDA_R_64F, V, k, CUDA_R_64F, &dws, &hws));
    CK(cudaMalloc(&dw, dws));
    hw.resize(hws + 16);
    double herr = 0;
    tstart();
    CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, M, k, CUDA_R_64F, S, CUDA_R_64F, U, k,
                         CUDA_R_64F, V, k, CUDA_R_64F, dw, dws, hw.data(), hws, info, &herr));
    float ms = tstop();
    int hi = 0;
    CK(cudaMemcpy(&hi, info, sizeof(int), cudaMemcpyDeviceToHost));
    printf("{\"k\": %lld, \"gesvdp_info\": %d, \"h_err_sigma\": %.3e, \"dws_gb\": %.2f}\n", (long long)k, hi, herr, dws / 1e9);
    cudaFree(dw);
    accuracy("gesvdp_R", ms, U, V, refS.empty() ? nullptr : &refS);
  }
  // 3. building blocks: syrk, potrf, trsm, gemm, syevd of a k x k symmetric matrix
  {
    float ms;
    tstart();
    CK(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, k, k, &one, R, k, &zero, M, k));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"syrk\", \"ms\": %.1f, \"tflops\": %.1f}\n", (long long)k, ms, 1.0 * k * k * k / ms / 1e9);
    tstart();
    CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, k, &one, R, k, R, k, &zero, U, k));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"gemm\", \"ms\": %.1f, \"tflops\": %.1f}\n", (long long)k, ms, 2.0 * k * k * k / ms / 1e9);
    // SPD: M = R^T R + I
    CK(cudaMemcpy(M, U, sizeof(double) * k * k, cudaMemcpyDeviceToDevice));
    CK(cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_LOWER, k, CUDA_R_64F, M, k, CUDA_R_64F, &dws, &hws));
    CK(cudaMalloc(&dw, dws));
    hw.resize(hws + 16);
    tstart();
    CK(cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_LOWER, k, CUDA_R_64F, M, k, CUDA_R_64F, dw, dws, hw.data(), hws, info));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"potrf\", \"ms\": %.1f, \"tflops\": %.1f}\n", (long long)k, ms, k * k * k / 3.0 / ms / 1e9);
    cudaFree(dw);
    tstart();
    CK(cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, k, k, &one, M, k, V, k));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"trsm\", \"ms\": %.1f, \"tflops\": %.1f}\n", (long long)k, ms, 1.0 * k * k * k / ms / 1e9);
    for (int x = 0; x < 2; ++x) {
      CK(cudaMemcpy(M, U, sizeof(double) * k * k, cudaMemcpyDeviceToDevice));
      CK(cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, CUDA_R_64F, M, k,
                                     CUDA_R_64F, S, CUDA_R_64F, &dws, &hws));
      CK(cudaMalloc(&dw, dws));
      hw.resize(hws + 16);
      tstart();
      CK(cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, CUDA_R_64F, M, k, CUDA_R_64F, S,
                          CUDA_R_64F, dw, dws, hw.data(), hws, info));
      ms = tstop();
      printf("{\"k\": %lld, \"op\": \"syevd_k\", \"ms\": %.1f}\n", (long long)k, ms);
      cudaFree(dw);
    }
    // geqrf of a 2k x k stacked matrix (QR-based QDWH step)
    double* B;
    CK(cudaMalloc(&B, sizeof(double) * 2 * k * k));
    gen<<<4096, 256>>>(B, 2 * k, k, 11u);
    CK(cusolverDnXgeqrf_bufferSize(h, prm, 2 * k, k, CUDA_R_64F, B, 2 * k, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws));
    CK(cudaMalloc(&dw, dws));
    hw.resize(hws + 16);
    tstart();
    CK(cusolverDnXgeqrf(h, prm, 2 * k, k, CUDA_R_64F, B, 2 * k, CUDA_R_64F, tau, CUDA_R_64F, dw, dws, hw.data(), hws, info));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"geqrf_2kxk\", \"ms\": %.1f}\n", (long long)k, ms);
    cudaFree(dw);
    int lw = 0;
    CK(cusolverDnDorgqr_bufferSize(h, 2 * k, k, k, B, 2 * k, tau, &lw));
    CK(cudaMalloc(&dw, sizeof(double) * lw));
    tstart();
    CK(cusolverDnDorgqr(h, 2 * k, k, k, B, 2 * k, tau, (double*)dw, lw, info));
    ms = tstop();
    printf("{\"k\": %lld, \"op\": \"orgqr_2kxk\", \"ms\": %.1f}\n", (long long)k, ms);
    cudaFree(dw);
    cudaFree(B);
  }
  return 0;
}
