// QR options in front of the polar SVD for the c5 sketch shape (s = 2e4, k = 1e4,
// columns scaled 1 -> 1e-5): (a) geqrf + gesvdp(R) [the library's route],
// (b) gesvdp on the s x k sketch directly, (c) CholeskyQR2 (two rounds of
// syrk + potrf + trsm; R = R2 R1) + gesvdp(R).  Time and sigma agreement with (a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench5.cu -lcusolver -lcublas -o svd_bench5
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
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < s * k; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = idx / s;
    unsigned long long h = (unsigned long long)idx * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    double u = ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    A[idx] = (u - 0.5) * pow(10.0, -5.0 * (double)j / (double)(k - 1));
  }
}
__global__ void upper(const double* A, int64_t lda, int64_t k, double* R) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < k * k; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % k, j = idx / k;
    R[idx] = i <= j ? A[j * lda + i] : 0.0;
  }
}

int main(int argc, char** argv) {
  const int64_t k = argc > 1 ? atoll(argv[1]) : 10000, s = 2 * k;
  cusolverDnHandle_t h; cublasHandle_t cb; cusolverDnParams_t prm;
  CK(cusolverDnCreate(&h)); CK(cublasCreate(&cb)); CK(cusolverDnCreateParams(&prm));
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  double *A0, *A, *tau, *R, *R2, *S, *U, *V, *Gm; int* info;
  CK(cudaMalloc(&A0, 8 * s * k)); CK(cudaMalloc(&A, 8 * s * k)); CK(cudaMalloc(&tau, 8 * k));
  CK(cudaMalloc(&R, 8 * k * k)); CK(cudaMalloc(&R2, 8 * k * k)); CK(cudaMalloc(&S, 8 * k));
  CK(cudaMalloc(&U, 8 * s * k)); CK(cudaMalloc(&V, 8 * k * k)); CK(cudaMalloc(&Gm, 8 * k * k)); CK(cudaMalloc(&info, 16));
  gen<<<4096, 256>>>(A0, s, k, 3u);
  size_t dws = 0, hws = 0, d2 = 0, h2 = 0, d3 = 0, h3 = 0, d4 = 0, h4 = 0;
  CK(cusolverDnXgeqrf_bufferSize(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws));
  CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, R, k, CUDA_R_64F, S, CUDA_R_64F, U, k, CUDA_R_64F, V, k, CUDA_R_64F, &d2, &h2));
  CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, s, k, CUDA_R_64F, A, s, CUDA_R_64F, S, CUDA_R_64F, U, s, CUDA_R_64F, V, k, CUDA_R_64F, &d3, &h3));
  CK(cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_UPPER, k, CUDA_R_64F, Gm, k, CUDA_R_64F, &d4, &h4));
  size_t dw = std::max({dws, d2, d3, d4}), hw = std::max({hws, h2, h3, h4});
  void* work; CK(cudaMalloc(&work, dw)); std::vector<char> hwork(hw + 16);
  std::vector<double> sa(k), sb(k);
  const double one = 1.0, zero = 0.0;
  auto svdR = [&]() { double herr; CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, R, k, CUDA_R_64F, S, CUDA_R_64F, U, k, CUDA_R_64F, V, k, CUDA_R_64F, work, dw, hwork.data(), hw, info, &herr)); };
  for (int rep = 0; rep < 2; ++rep) {
    // (a)
    CK(cudaMemcpy(A, A0, 8 * s * k, cudaMemcpyDeviceToDevice));
    tstart();
    CK(cusolverDnXgeqrf(h, prm, s, k, CUDA_R_64F, A, s, CUDA_R_64F, tau, CUDA_R_64F, work, dw, hwork.data(), hw, info));
    upper<<<4096, 256>>>(A, s, k, R);
    float ta_qr = tstop(); tstart(); svdR(); float ta_svd = tstop();
    CK(cudaMemcpy(sa.data(), S, 8 * k, cudaMemcpyDeviceToHost));
    printf("{\"k\": %lld, \"route\": \"geqrf+gesvdp(R)\", \"qr_ms\": %.1f, \"svd_ms\": %.1f}\n", (long long)k, ta_qr, ta_svd);
    // (b)
    CK(cudaMemcpy(A, A0, 8 * s * k, cudaMemcpyDeviceToDevice));
    tstart(); { double herr; CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, s, k, CUDA_R_64F, A, s, CUDA_R_64F, S, CUDA_R_64F, U, s, CUDA_R_64F, V, k, CUDA_R_64F, work, dw, hwork.data(), hw, info, &herr)); }
    float tb = tstop();
    CK(cudaMemcpy(sb.data(), S, 8 * k, cudaMemcpyDeviceToHost));
    double eb = 0; for (int64_t i = 0; i < k; ++i) eb = std::max(eb, fabs(sb[i] - sa[i]) / sa[i]);
    printf("{\"k\": %lld, \"route\": \"gesvdp(sketch)\", \"ms\": %.1f, \"sigma_maxrel_vs_a\": %.3e}\n", (long long)k, tb, eb);
    // (c) CholeskyQR2: G = A^T A, R1 = chol(G), Q = A R1^-1, G = Q^T Q, R2 = chol, R = R2 R1
    CK(cudaMemcpy(A, A0, 8 * s * k, cudaMemcpyDeviceToDevice));
    tstart();
    for (int round = 0; round < 2; ++round) {
      CK(cublasDsyrk(cb, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, k, s, &one, A, s, &zero, Gm, k));
      CK(cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_UPPER, k, CUDA_R_64F, Gm, k, CUDA_R_64F, work, dw, hwork.data(), hw, info));
      upper<<<4096, 256>>>(Gm, k, k, round == 0 ? R2 : Gm);
      CK(cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, s, k, &one, round == 0 ? R2 : Gm, k, A, s));
    }
    // R = Gm(R2 of round 2) * R2(R1): triangular product into R
    CK(cudaMemcpy(R, R2, 8 * k * k, cudaMemcpyDeviceToDevice));
    CK(cublasDtrmm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, k, k, &one, Gm, k, R2, k, R, k));
    float tc_qr = tstop();
    int hi = 0; CK(cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost));
    tstart(); svdR(); float tc_svd = tstop();
    CK(cudaMemcpy(sb.data(), S, 8 * k, cudaMemcpyDeviceToHost));
    double ec = 0; for (int64_t i = 0; i < k; ++i) ec = std::max(ec, fabs(sb[i] - sa[i]) / sa[i]);
    printf("{\"k\": %lld, \"route\": \"cholqr2+gesvdp(R)\", \"qr_ms\": %.1f, \"svd_ms\": %.1f, \"potrf_info\": %d, \"sigma_maxrel_vs_a\": %.3e}\n",
           (long long)k, tc_qr, tc_svd, hi, ec);
    fflush(stdout);
  }
  return 0;
}
