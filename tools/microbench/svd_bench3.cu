// SVD options for a large k x k R (c4: k = 2e4), where the Jordan-Wielandt
// eigenproblem (2k = 4e4) exceeds cuSOLVER's symmetric-eigensolver limit
// (n <= 32768, profiles/r01_syevdx_limit.jsonl).  Outside the hot path (Alg. 1
// step 4).  Options, each with time, sigma error vs gesvd and the
// V-subspace distance to gesvd's V:
//   gesvd(N, A) on R                        (the current fallback)
//   gesvdj(tol 1e-14, 15 sweeps) on R
//   "preconditioned Jacobi": syevd(R^T R) -> V0, B = R V0, gesvdj(B) with few
//   sweeps -> V = V0 Vb (the one-sided Jacobi on B restores full accuracy;
//   timing study only, SURVEY H6 forbids using the Gram eigenvectors directly)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench3.cu -lcusolver -lcublas -o svd_bench3
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

int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 20000;
  const int s = 2 * k;
  cusolverDnHandle_t h; cublasHandle_t cb;
  CK(cusolverDnCreate(&h)); CK(cublasCreate(&cb));
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  // R: QR of an s x k Gaussian matrix with columns scaled 1 -> 1e-4 (full rank)
  double *A, *tau, *R0, *Rw, *S, *U, *V, *V0, *refV, *M, *work;
  int* info;
  CK(cudaMalloc(&A, sizeof(double) * (size_t)s * k));
  CK(cudaMalloc(&tau, sizeof(double) * k));
  {
    std::vector<double> col(s);
    srand(3);
    for (int j = 0; j < k; ++j) {
      const double sc = pow(10.0, -4.0 * j / (double)(k - 1));
      for (int i = 0; i < s; ++i) col[i] = sc * (rand() / (double)RAND_MAX - 0.5);
      CK(cudaMemcpy(A + (size_t)j * s, col.data(), sizeof(double) * s, cudaMemcpyHostToDevice));
    }
  }
  CK(cudaMalloc(&R0, sizeof(double) * (size_t)k * k)); CK(cudaMalloc(&Rw, sizeof(double) * (size_t)k * k));
  CK(cudaMalloc(&S, sizeof(double) * k)); CK(cudaMalloc(&U, sizeof(double) * (size_t)k * k));
  CK(cudaMalloc(&V, sizeof(double) * (size_t)k * k)); CK(cudaMalloc(&V0, sizeof(double) * (size_t)k * k));
  CK(cudaMalloc(&refV, sizeof(double) * (size_t)k * k)); CK(cudaMalloc(&M, sizeof(double) * (size_t)k * k));
  CK(cudaMalloc(&info, 16));
  int l1 = 0, l2 = 0, l3 = 0, l4 = 0;
  CK(cusolverDnDgeqrf_bufferSize(h, s, k, A, s, &l1));
  CK(cusolverDnDgesvd_bufferSize(h, k, k, &l2));
  gesvdjInfo_t jp; CK(cusolverDnCreateGesvdjInfo(&jp));
  CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, Rw, k, S, U, k, V, k, &l3, jp));
  CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, Rw, k, S, &l4));
  const size_t lw = std::max({(size_t)l1, (size_t)l2, (size_t)l3, (size_t)l4});
  CK(cudaMalloc(&work, sizeof(double) * lw));
  tstart();
  CK(cusolverDnDgeqrf(h, s, k, A, s, tau, work, (int)lw, info));
  printf("{\"k\": %d, \"geqrf_ms\": %.1f}\n", k, tstop()); fflush(stdout);
  // R0 = upper triangle of the factored A (column-major, k x k)
  CK(cudaMemset(R0, 0, sizeof(double) * (size_t)k * k));
  for (int j = 0; j < k; ++j) CK(cudaMemcpy(R0 + (size_t)j * k, A + (size_t)j * s, sizeof(double) * (j + 1), cudaMemcpyDeviceToDevice));
  cudaFree(A);
  const double one = 1, zero = 0;
  std::vector<double> refS(k), sig(k);
  auto subspace = [&](const double* Vc) {   // sqrt(k - ||refV^T Vc||_F^2)
    CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, k, &one, refV, k, Vc, k, &zero, M, k));
    double nrm; CK(cublasDnrm2(cb, k * k, M, 1, &nrm));
    return sqrt(fabs(k - nrm * nrm));
  };
  auto sigerr = [&]() {
    double m = 0; for (int i = 0; i < k; ++i) m = std::max(m, fabs(sig[i] - refS[i]) / refS[i]); return m;
  };
  // 1. gesvd N,A (reference)
  CK(cudaMemcpy(Rw, R0, sizeof(double) * (size_t)k * k, cudaMemcpyDeviceToDevice));
  tstart();
  CK(cusolverDnDgesvd(h, 'N', 'A', k, k, Rw, k, S, nullptr, 1, U, k, work, (int)lw, nullptr, info));
  float ms = tstop();
  CK(cudaMemcpy(refS.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
  CK(cublasDgeam(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, &one, U, k, &zero, U, k, refV, k));
  printf("{\"svd\": \"gesvd_NA\", \"ms\": %.1f}\n", ms); fflush(stdout);
  // 2. gesvdj on R
  CK(cusolverDnXgesvdjSetTolerance(jp, 1e-14)); CK(cusolverDnXgesvdjSetMaxSweeps(jp, 15));
  CK(cudaMemcpy(Rw, R0, sizeof(double) * (size_t)k * k, cudaMemcpyDeviceToDevice));
  tstart();
  CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, Rw, k, S, U, k, V, k, work, (int)lw, info, jp));
  ms = tstop();
  int sweeps = 0; double resid = 0;
  cusolverDnXgesvdjGetSweeps(h, jp, &sweeps); cusolverDnXgesvdjGetResidual(h, jp, &resid);
  CK(cudaMemcpy(sig.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
  printf("{\"svd\": \"gesvdj_R\", \"ms\": %.1f, \"sweeps\": %d, \"sigma_maxrel\": %.3e, \"subspace\": %.3e}\n", ms, sweeps,
         sigerr(), subspace(V)); fflush(stdout);
  // 3. preconditioned Jacobi: syevd(R^T R) -> V0, B = R V0, gesvdj(B) -> V = V0 Vb
  tstart();
  CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, k, &one, R0, k, R0, k, &zero, V0, k));
  CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, V0, k, S, work, (int)lw, info));
  const float ms_eig = tstop();
  for (int sw : {2, 4}) {
    tstart();
    CK(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, &one, R0, k, V0, k, &zero, Rw, k));   // B = R V0
    CK(cusolverDnXgesvdjSetTolerance(jp, 1e-14)); CK(cusolverDnXgesvdjSetMaxSweeps(jp, sw));
    CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, Rw, k, S, U, k, M, k, work, (int)lw, info, jp));
    CK(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, &one, V0, k, M, k, &zero, V, k));      // V = V0 Vb
    const float ms_j = tstop();
    cusolverDnXgesvdjGetSweeps(h, jp, &sweeps); cusolverDnXgesvdjGetResidual(h, jp, &resid);
    CK(cudaMemcpy(sig.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
    printf("{\"svd\": \"gram_then_gesvdj\", \"max_sweeps\": %d, \"eig_ms\": %.1f, \"jacobi_ms\": %.1f, \"sweeps\": %d, "
           "\"sigma_maxrel\": %.3e, \"subspace\": %.3e}\n", sw, ms_eig, ms_j, sweeps, sigerr(), subspace(V));
    fflush(stdout);
  }
  return 0;
}
