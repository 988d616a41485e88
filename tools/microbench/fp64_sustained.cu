// Sustained FP64 tensor (DMMA.8x8x4) throughput on B200: the same kernel as
// fp64_peak.cu's dmma test, launched back to back for ~12 s so that the clocks
// settle under the power cap (the bench's c5 sketch runs 14 s).  One JSON line per
// second of launches + a summary.  The caller samples nvidia-smi clocks alongside.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_sustained fp64_sustained.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters, double a0, double b0) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 12.0;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  const int warps = 8, blocks = nsm * 2, threads = 32 * warps, iters = 200000;
  const double flops_per_launch = (double)blocks * warps * iters * 8 * 512;
  cudaEvent_t e0, e1, t0;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&t0);
  k_dmma<<<blocks, threads>>>(out, iters / 10, 1.0, 1.0);
  cudaDeviceSynchronize();
  cudaEventRecord(t0);
  double total_ms = 0, total_flops = 0;
  int n = 0;
  while (total_ms < seconds * 1e3) {
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters, 1.0, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    total_ms += ms;
    total_flops += flops_per_launch;
    ++n;
    printf("{\"launch\": %d, \"ms\": %.2f, \"tflops\": %.3f}\n", n, ms, flops_per_launch / ms / 1e9);
    fflush(stdout);
  }
  float wall;
  cudaEventElapsedTime(&wall, t0, e1);
  printf("{\"test\": \"dmma_sustained\", \"launches\": %d, \"seconds\": %.2f, \"tflops_avg\": %.3f, \"tflops_wall\": %.3f}\n", n,
         total_ms / 1e3, total_flops / total_ms / 1e9, total_flops / wall / 1e9);
  return 0;
}
