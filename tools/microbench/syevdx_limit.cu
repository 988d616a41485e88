// Which sizes does cuSOLVER's (64-bit API) syevdx / syevd / gesvd accept?  (bufferSize queries only)
#include <cstdio>
#include <cusolverDn.h>
int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cusolverDnParams_t p; cusolverDnCreateParams(&p);
  for (long n : {8192L, 16384L, 20000L, 32768L, 32769L, 40000L, 46340L}) {
    size_t d = 0, hb = 0; int64_t meig = 0; double vl = 0, vu = 0;
    int s1 = (int)cusolverDnXsyevdx_bufferSize(h, p, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER,
                                             n, CUDA_R_64F, nullptr, n, &vl, &vu, n / 2 + 1, n, &meig, CUDA_R_64F, nullptr,
                                             CUDA_R_64F, &d, &hb);
    size_t d2 = 0, h2 = 0;
    int s2 = (int)cusolverDnXsyevd_bufferSize(h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, nullptr,
                                            n, CUDA_R_64F, nullptr, CUDA_R_64F, &d2, &h2);
    size_t d3 = 0, h3 = 0;
    int s3 = (int)cusolverDnXgesvd_bufferSize(h, p, 'N', 'A', n / 2, n / 2, CUDA_R_64F, nullptr, n / 2, CUDA_R_64F, nullptr,
                                            CUDA_R_64F, nullptr, 1, CUDA_R_64F, nullptr, n / 2, CUDA_R_64F, &d3, &h3);
    printf("{\"n\": %ld, \"syevdx\": [%d, %.3g], \"syevd\": [%d, %.3g], \"gesvd_half\": [%d, %.3g]}\n", n, s1, (double)d, s2,
           (double)d2, s3, (double)d3);
  }
  return 0;
}
