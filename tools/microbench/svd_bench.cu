// cuSOLVER SVD options for the s x k sketch (outside the LSRN hot path):
// time + accuracy of (QR ->) gesvd / gesvdj / Xgesvdp on a k x k triangular R.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench.cu -lcusolver -lcublas -o svd_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cublas_v2.h>

#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s line %d code %d\"}\n", #x, __LINE__, (int)e); exit(1);} } while (0)

int main(int argc, char** argv) {
  int s = argc > 1 ? atoi(argv[1]) : 4000, k = argc > 2 ? atoi(argv[2]) : 2000;
  int rank = argc > 3 ? atoi(argv[3]) : k;
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cublasHandle_t cb; CK(cublasCreate(&cb));
  // A = random s x k with singular values 1 .. 1e-4 on `rank`, 0 after (column-major)
  std::vector<double> hA((size_t)s * k);
  srand(1);
  for (auto& v : hA) v = (rand() / (double)RAND_MAX - 0.5);
  double *A, *W, *tau, *R, *S, *VT, *U, *work; int* info;
  CK(cudaMalloc(&A, sizeof(double) * s * k)); CK(cudaMalloc(&W, sizeof(double) * s * k));
  CK(cudaMalloc(&tau, sizeof(double) * k)); CK(cudaMalloc(&R, sizeof(double) * k * k));
  CK(cudaMalloc(&S, sizeof(double) * k)); CK(cudaMalloc(&VT, sizeof(double) * k * k));
  CK(cudaMalloc(&U, sizeof(double) * k * k)); CK(cudaMalloc(&info, 16));
  CK(cudaMemcpy(A, hA.data(), sizeof(double) * s * k, cudaMemcpyHostToDevice));
  // impose spectrum: A <- A * diag(scale) (cheap, ill-conditioned; rank-deficient tail zeroed)
  for (int j = 0; j < k; ++j) {
    double sc = j < rank ? pow(10.0, -4.0 * j / (double)std::max(rank - 1, 1)) : 0.0;
    CK(cublasDscal(cb, s, &sc, A + (size_t)j * s, 1));
  }
  int l1, l2, l3 = 0; size_t dl = 0, hl = 0;
  CK(cusolverDnDgeqrf_bufferSize(h, s, k, A, s, &l1));
  CK(cusolverDnDgesvd_bufferSize(h, k, k, &l2));
  gesvdjInfo_t jp; CK(cusolverDnCreateGesvdjInfo(&jp));
  CK(cusolverDnXgesvdjSetTolerance(jp, 1e-15));
  CK(cusolverDnXgesvdjSetMaxSweeps(jp, 30));
  CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, R, k, S, U, k, VT, k, &l3, jp));
  CK(cusolverDnXgesvdp_bufferSize(h, nullptr, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, R, k, CUDA_R_64F, S,
                                  CUDA_R_64F, U, k, CUDA_R_64F, VT, k, CUDA_R_64F, &dl, &hl));
  size_t lw = std::max({(size_t)l1, (size_t)l2, (size_t)l3, dl / 8 + 1});
  CK(cudaMalloc(&work, sizeof(double) * lw));
  std::vector<char> hwork(hl + 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto qr = [&]() {
    CK(cudaMemcpy(W, A, sizeof(double) * s * k, cudaMemcpyDeviceToDevice));
    CK(cusolverDnDgeqrf(h, s, k, W, s, tau, work, (int)lw, info));
    CK(cudaMemset(R, 0, sizeof(double) * k * k));
    CK(cudaMemcpy2D(R, k * sizeof(double), W, s * sizeof(double), k * sizeof(double), k, cudaMemcpyDeviceToDevice));
    // zero strictly-lower part: copy upper triangle only via host-free trick: use cublas? (do it on host for bench)
    std::vector<double> hr((size_t)k * k);
    CK(cudaMemcpy(hr.data(), R, sizeof(double) * k * k, cudaMemcpyDeviceToHost));
    for (int j = 0; j < k; ++j) for (int i = j + 1; i < k; ++i) hr[(size_t)j * k + i] = 0;
    CK(cudaMemcpy(R, hr.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice));
  };
  std::vector<double> ref(k), got(k);
  auto run = [&](const char* name, int which) {
    qr();
    cudaDeviceSynchronize();
    float msq = 0;
    {
      cudaEventRecord(e0);
      CK(cusolverDnDgeqrf(h, s, k, W, s, tau, work, (int)lw, info));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&msq, e0, e1);
      qr();
    }
    cudaEventRecord(e0);
    double resid = 0; int hinfo = 0;
    if (which == 0) CK(cusolverDnDgesvd(h, 'N', 'A', k, k, R, k, S, nullptr, 1, VT, k, work, (int)lw, nullptr, info));
    if (which == 1) CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, R, k, S, U, k, VT, k, work, (int)lw, info, jp));
    if (which == 2) CK(cusolverDnXgesvdp(h, nullptr, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, R, k, CUDA_R_64F, S,
                                         CUDA_R_64F, U, k, CUDA_R_64F, VT, k, CUDA_R_64F, work, dl, hwork.data(), hl, info, &resid));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(got.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
    if (which == 0) ref = got;
    double maxrel = 0; int r = 0;
    for (int i = 0; i < k; ++i) {
      if (ref[i] > 1e-12 * ref[0]) { maxrel = std::max(maxrel, fabs(got[i] - ref[i]) / ref[i]); }
      if (got[i] > std::max(s, k) * 2.22e-16 * got[0]) ++r;
    }
    printf("{\"svd\": \"%s\", \"s\": %d, \"k\": %d, \"qr_ms\": %.2f, \"svd_ms\": %.2f, \"info\": %d, \"rank\": %d, \"sigma_maxrel_vs_gesvd\": %.3e, \"resid\": %.3e}\n",
           name, s, k, msq, ms, hinfo, r, maxrel, resid);
  };
  run("gesvd", 0);
  run("gesvdj", 1);
  run("gesvdp", 2);
  run("gesvd", 0);
  return 0;
}
