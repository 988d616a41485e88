// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64),
// DFMA, DMMA+DFMA mixed (do they share the FP64 datapath?), and the cost of a
// fp64 Philox4x32-10 + Box-Muller normal. Prints one JSON line per test.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double a0, double b0) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NCH>
__global__ void k_dfma(double* out, int iters, double a0, double b0) {
  double c[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i] = i * 1e-3;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// per iteration: NACC DMMA + NCH DFMA (per thread)
template <int NACC, int NCH>
__global__ void k_mixed(double* out, int iters, double a0, double b0) {
  double acc[NACC][2];
  double c[NCH];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i] = i * 1e-3;
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u; k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void k_bm(double* out, int iters, uint64_t seed) {
  uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 o = philox(make_uint4(it, j, 0, 0), key);
    uint64_t w0 = o.x | ((uint64_t)o.y << 32), w1 = o.z | ((uint64_t)o.w << 32);
    double u1 = ((w0 >> 11) + 1) * 0x1.0p-53, u2 = (w1 >> 11) * 0x1.0p-53;
    double rho = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    s += rho * cs + rho * sn;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_philox_only(double* out, int iters, uint64_t seed) {
  uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t s = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 o = philox(make_uint4(it, j, 0, 0), key);
    s += o.x ^ o.y ^ o.z ^ o.w;
  }
  if (s == 123456u) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();  // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out; CK(cudaMalloc(&out, 64));
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    int blocks = nsm * 2, threads = 32 * warps;
    float ms = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 1.0, 1.0); });
    double flops = (double)blocks * warps * iters * 8 * 512;
    printf("{\"test\": \"dmma_m8n8k4\", \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", warps, blocks, ms, flops / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    int blocks = nsm * 2, threads = 32 * warps;
    float ms = timeit([&] { k_dfma<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    double flops = (double)blocks * threads * iters * 8 * 2;
    printf("{\"test\": \"dfma\", \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", warps, blocks, ms, flops / ms / 1e9);
  }
  {
    // mixed: per iteration 8 DMMA (8*512 flops/warp) + 16 DFMA/thread (16*2*32 = 1024 flops/warp)
    int warps = 8, blocks = nsm * 2, threads = 32 * warps;
    float ms = timeit([&] { k_mixed<8, 16><<<blocks, threads>>>(out, iters, 1.0, 1.0); });
    float ms_d = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 1.0, 1.0); });
    float ms_f = timeit([&] { k_dfma<16><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    printf("{\"test\": \"mixed_8dmma_16dfma\", \"ms_mixed\": %.3f, \"ms_dmma_alone\": %.3f, \"ms_dfma_alone\": %.3f, \"verdict\": \"%s\"}\n",
           ms, ms_d, ms_f, (ms > 0.85 * (ms_d + ms_f)) ? "shared_pipe" : "overlap");
  }
  {
    int blocks = nsm * 8, threads = 256, it2 = 2000;
    float ms = timeit([&] { k_bm<<<blocks, threads>>>(out, it2, 5981); });
    double normals = 2.0 * blocks * threads * it2;
    printf("{\"test\": \"philox_boxmuller_fp64\", \"ms\": %.3f, \"gnormals_per_s\": %.3f}\n", ms, normals / ms / 1e6);
    float ms2 = timeit([&] { k_philox_only<<<blocks, threads>>>(out, it2, 5981); });
    printf("{\"test\": \"philox_only\", \"ms\": %.3f, \"gcalls_per_s\": %.3f}\n", ms2, (double)blocks * threads * it2 / ms2 / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
