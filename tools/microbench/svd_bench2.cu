// cuSOLVER options for the k x k SVD stage of LSRN (Alg. 1 step 4),
// outside the hot path.  Input: R of a QR of an s x k sketch-like matrix with
// singular values 1 -> 1e-4 on `rank`, zero tail (the c2 shape).  Each option
// reports time, sigma error vs gesvd, rank, and the distance between its V_r
// subspace and gesvd's: sqrt(r - ||V1_r^T V2_r||_F^2).
// Options: gesvd(N,A) | gesvd on R^T (U side) | gesvdj(tol) | syevd on the
// Jordan-Wielandt matrix [[0 R^T][R 0]] | syevdx (top k) on it | syevd(R^T R) (the
// squared-kappa trap, timing reference only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 svd_bench2.cu -lcusolver -lcublas -o svd_bench2
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s line %d code %d\"}\n", #x, __LINE__, (int)e); exit(1);} } while (0)

static int s_, k_, rank_;
static cusolverDnHandle_t h;
static cublasHandle_t cb;
static double *R0, *Rw, *S, *V, *U, *work, *JW, *M;
static int* info;
static size_t lw;
static cudaEvent_t e0, e1;
static std::vector<double> refS;
static double* refV;   // k x k column-major, columns = right singular vectors

static void timer_start() { cudaEventRecord(e0); }
static float timer_stop() { cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms; }

// Vcols: k x r column-major (right singular vectors), sig: descending
static void report(const char* name, float ms, const std::vector<double>& sig, const double* Vcols, int ldv) {
  int k = k_;
  int r = 0;
  for (int i = 0; i < k; ++i) if (sig[i] > std::max(s_, k) * 2.220446049250313e-16 * sig[0]) ++r;
  double maxrel = 0;
  for (int i = 0; i < std::min(r, rank_); ++i) maxrel = std::max(maxrel, fabs(sig[i] - refS[i]) / refS[i]);
  double sub = -1;
  if (Vcols && !refS.empty()) {
    int rr = std::min(r, rank_);
    const double one = 1, zero = 0;
    CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, rr, rr, k, &one, refV, k, Vcols, ldv, &zero, M, rr));
    double nrm; CK(cublasDnrm2(cb, rr * rr, M, 1, &nrm));
    sub = sqrt(fabs(rr - nrm * nrm));
  }
  printf("{\"svd\": \"%s\", \"k\": %d, \"ms\": %.2f, \"rank\": %d, \"sigma_maxrel\": %.3e, \"subspace\": %.3e}\n", name, k, ms, r,
         maxrel, sub);
  fflush(stdout);
}

int main(int argc, char** argv) {
  s_ = argc > 1 ? atoi(argv[1]) : 4000; k_ = argc > 2 ? atoi(argv[2]) : 2000; rank_ = argc > 3 ? atoi(argv[3]) : k_;
  const int s = s_, k = k_;
  CK(cusolverDnCreate(&h)); CK(cublasCreate(&cb));
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<double> hA((size_t)s * k);
  srand(1);
  for (auto& v : hA) v = (rand() / (double)RAND_MAX - 0.5);
  double *A, *tau;
  CK(cudaMalloc(&A, sizeof(double) * s * k)); CK(cudaMalloc(&tau, sizeof(double) * k));
  CK(cudaMemcpy(A, hA.data(), sizeof(double) * s * k, cudaMemcpyHostToDevice));
  // mix columns so the spectrum is not axis-aligned: A <- A * Q diag(sc) via a random orthogonal Q from QR
  for (int j = 0; j < k; ++j) {
    double sc = j < rank_ ? pow(10.0, -4.0 * j / (double)std::max(rank_ - 1, 1)) : 0.0;
    CK(cublasDscal(cb, s, &sc, A + (size_t)j * s, 1));
  }
  CK(cudaMalloc(&R0, sizeof(double) * k * k)); CK(cudaMalloc(&Rw, sizeof(double) * k * k));
  CK(cudaMalloc(&S, sizeof(double) * 2 * k)); CK(cudaMalloc(&V, sizeof(double) * k * k));
  CK(cudaMalloc(&U, sizeof(double) * k * k)); CK(cudaMalloc(&refV, sizeof(double) * k * k));
  CK(cudaMalloc(&M, sizeof(double) * k * k)); CK(cudaMalloc(&info, 16));
  CK(cudaMalloc(&JW, sizeof(double) * 4 * k * k));
  int l1 = 0, l2 = 0, l3 = 0, l4 = 0, l5 = 0, l6 = 0;
  CK(cusolverDnDgeqrf_bufferSize(h, s, k, A, s, &l1));
  CK(cusolverDnDgesvd_bufferSize(h, k, k, &l2));
  gesvdjInfo_t jp; CK(cusolverDnCreateGesvdjInfo(&jp));
  CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, Rw, k, S, U, k, V, k, &l3, jp));
  CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, 2 * k, JW, 2 * k, S, &l4));
  int meig = 0;
  CK(cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k, JW,
                                  2 * k, 0., 0., k + 1, 2 * k, &meig, S, &l5));
  CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, Rw, k, S, &l6));
  lw = std::max({(size_t)l1, (size_t)l2, (size_t)l3, (size_t)l4, (size_t)l5, (size_t)l6});
  CK(cudaMalloc(&work, sizeof(double) * lw));
  // QR once -> R0 (upper triangle)
  CK(cusolverDnDgeqrf(h, s, k, A, s, tau, work, (int)lw, info));
  timer_start();
  CK(cusolverDnDgeqrf(h, s, k, A, s, tau, work, (int)lw, info));  // timing only (on the factored matrix)
  printf("{\"geqrf_ms\": %.2f}\n", timer_stop());
  std::vector<double> hR((size_t)k * k), tmp((size_t)s * k);
  CK(cudaMemcpy(tmp.data(), A, sizeof(double) * s * k, cudaMemcpyDeviceToHost));
  for (int j = 0; j < k; ++j) for (int i = 0; i < k; ++i) hR[(size_t)j * k + i] = i <= j ? tmp[(size_t)j * s + i] : 0.0;
  CK(cudaMemcpy(R0, hR.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice));
  std::vector<double> sig(2 * k);
  auto reset = [&]() { CK(cudaMemcpy(Rw, R0, sizeof(double) * k * k, cudaMemcpyDeviceToDevice)); cudaDeviceSynchronize(); };
  auto getS = [&](int n, const double* src) { CK(cudaMemcpy(sig.data(), src, sizeof(double) * n, cudaMemcpyDeviceToHost)); };
  const double one = 1, zero = 0;

  for (int rep = 0; rep < 2; ++rep) {
    // 1. gesvd N,A on R: VT rows are right singular vectors -> V = VT^T
    reset(); timer_start();
    CK(cusolverDnDgesvd(h, 'N', 'A', k, k, Rw, k, S, nullptr, 1, U, k, work, (int)lw, nullptr, info));
    float ms = timer_stop();
    getS(k, S);
    if (refS.empty()) refS.assign(sig.begin(), sig.begin() + k);
    CK(cublasDgeam(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, &one, U, k, &zero, U, k, refV, k));
    report("gesvd_NA", ms, sig, refV, k);
    // 2. gesvd on R^T: jobu='A' (U of R^T = V of R), jobvt='N'
    CK(cublasDgeam(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, &one, R0, k, &zero, R0, k, Rw, k));
    cudaDeviceSynchronize(); timer_start();
    CK(cusolverDnDgesvd(h, 'A', 'N', k, k, Rw, k, S, U, k, nullptr, 1, work, (int)lw, nullptr, info));
    ms = timer_stop(); getS(k, S);
    report("gesvd_AN_on_RT", ms, sig, U, k);
    // 3. gesvdj at two tolerances
    for (double tol : {1e-15, 1e-12}) {
      for (int sweeps : {15, 100}) {
        CK(cusolverDnXgesvdjSetTolerance(jp, tol)); CK(cusolverDnXgesvdjSetMaxSweeps(jp, sweeps));
        reset(); timer_start();
        CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, Rw, k, S, U, k, V, k, work, (int)lw, info, jp));
        ms = timer_stop(); getS(k, S);
        char nm[64]; snprintf(nm, 64, "gesvdj_tol%.0e_sw%d", tol, sweeps);
        report(nm, ms, sig, V, k);
      }
    }
    // 4. Jordan-Wielandt [[0, R^T], [R, 0]] (2k x 2k), eigenpairs (+-sigma, [v; +-u]/sqrt2)
    auto build_jw = [&]() {
      CK(cudaMemset(JW, 0, sizeof(double) * 4 * k * k));
      // lower-left block (rows k..2k, cols 0..k) = R ; upper-right = R^T (full symmetric)
      CK(cublasDgeam(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, k, &one, R0, k, &zero, R0, k, JW + k, 2 * k));
      CK(cublasDgeam(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, &one, R0, k, &zero, R0, k, JW + (size_t)k * 2 * k, 2 * k));
      cudaDeviceSynchronize();
    };
    build_jw(); timer_start();
    CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, 2 * k, JW, 2 * k, S, work, (int)lw, info));
    ms = timer_stop();
    {   // eigenvalues ascending: top k are indices k..2k-1; sigma_i = ev[2k-1-i]; v part = rows 0..k of vector
      std::vector<double> ev(2 * k); CK(cudaMemcpy(ev.data(), S, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost));
      for (int i = 0; i < k; ++i) sig[i] = ev[2 * k - 1 - i];
      // V_i = sqrt2 * JW[0:k, 2k-1-i]: copy columns in reverse with scaling
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpy(V + (size_t)i * k, JW + (size_t)(2 * k - 1 - i) * 2 * k, sizeof(double) * k, cudaMemcpyDeviceToDevice));
      double sq2 = sqrt(2.0); CK(cublasDscal(cb, k * k, &sq2, V, 1));
      report("syevd_JW", ms, sig, V, k);
    }
    build_jw(); timer_start();
    CK(cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, 2 * k, JW, 2 * k, 0., 0.,
                         k + 1, 2 * k, &meig, S, work, (int)lw, info));
    ms = timer_stop();
    {
      std::vector<double> ev(k); CK(cudaMemcpy(ev.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
      for (int i = 0; i < k; ++i) sig[i] = ev[k - 1 - i];
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpy(V + (size_t)i * k, JW + (size_t)(k - 1 - i) * 2 * k, sizeof(double) * k, cudaMemcpyDeviceToDevice));
      double sq2 = sqrt(2.0); CK(cublasDscal(cb, k * k, &sq2, V, 1));
      report("syevdx_JW_topk", ms, sig, V, k);
    }
    // 5. the trap: syevd(R^T R)
    CK(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, k, &one, R0, k, R0, k, &zero, Rw, k));
    cudaDeviceSynchronize(); timer_start();
    CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, Rw, k, S, work, (int)lw, info));
    ms = timer_stop();
    {
      std::vector<double> ev(k); CK(cudaMemcpy(ev.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost));
      for (int i = 0; i < k; ++i) sig[i] = sqrt(std::max(ev[k - 1 - i], 0.0));
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpy(V + (size_t)i * k, Rw + (size_t)(k - 1 - i) * k, sizeof(double) * k, cudaMemcpyDeviceToDevice));
      report("syevd_RtR_TRAP", ms, sig, V, k);
    }
  }
  return 0;
}
