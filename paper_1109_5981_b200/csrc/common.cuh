// Shared device helpers for the LSRN sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define LSRN_DEV __device__ __forceinline__

namespace lsrn {

constexpr int kNumSMs = 148;  // B200; the host queries the real count

LSRN_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order warp sum of p[0..n) read through L2 (__ldcg: written by other CTAs
// of the same grid): lane l adds p[l], p[l+32], ... in order, then a butterfly.
// Deterministic for a given n; every lane returns the total.  Call with the full warp.
LSRN_DEV double warp_sum_l2(const double* p, int64_t n) {
  double v = 0.0;
  for (int64_t i = threadIdx.x & 31; i < n; i += 32) v += __ldcg(p + i);
  return warp_sum(v);
}

// cp.async 16 B global -> shared with zero fill of the bytes past src_bytes.
LSRN_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// cp.async 8 B (ca path, 8-byte granularity) with zero fill.
LSRN_DEV void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// cp.async 4 B (ca path).
LSRN_DEV void cp_async4(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
LSRN_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
LSRN_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Streaming 16-byte load that does not allocate in L1 (A is read once per pass).
LSRN_DEV double2 ldg_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
LSRN_DEV double ldg_stream1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor core (DMMA.8x8x4 on sm_100a).
// Fragments: lane l holds A[l/4][l%4], B[l%4][l/4], D[l/4][2(l%4) + {0,1}].
LSRN_DEV void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// ---- mbarrier + 1-D TMA bulk copy (sm_90+ PTX) -------------------------------
LSRN_DEV unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

LSRN_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
LSRN_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

LSRN_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

LSRN_DEV void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

LSRN_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Prefetch `bytes` (multiple of 16) at src into L2 (no completion to wait for).
LSRN_DEV void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// An L2 cache policy "evict last" for the whole access (createpolicy), and a 1-D bulk
// copy global -> shared that carries it: for data several CTAs re-read through L2.
LSRN_DEV uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
LSRN_DEV void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// L2 prefetch of [begin, end) rounded out to 16-byte boundaries (empty ranges ignored).
LSRN_DEV void prefetch_l2_range(const void* begin, const void* end) {
  const uintptr_t b = reinterpret_cast<uintptr_t>(begin) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(end) + 15) & ~uintptr_t(15);
  if (e > b) bulk_prefetch_l2(reinterpret_cast<const void*>(b), static_cast<unsigned>(e - b));
}

// 1-D bulk copy global -> this CTA's shared memory, completion on `bar` (bytes % 16 == 0).
LSRN_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace lsrn
