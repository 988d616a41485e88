// K4 (CSR sketch) and the CSR long pass (K6-CSR) for sparse A in the tall form:
// X = A (m >= n) as CSR, or X = A^T (m < n) as CSR of A^T, i.e. A in CSC.
//
// The paper notes that LSRN "automatically speeds up when A is sparse" because
// it only touches A through products (Abstract; §4.1) and
// ran a sparse, "far from optimized" threaded matvec (§6.5).
//
// Sketch Ã = G A for CSR A (Alg. 1 step 3) with G never stored.  The
// cost is set by regenerating G, not by HBM: each G[i, j] is a
// Philox call + half a Box-Muller pair (~40 FP64 ops), and a nonzero of row j
// is used once per sketch row.  The shard is therefore split by column density:
//   * heavy columns (density >= 1/32, at most 64 of them) are gathered into a
//     dense cnt x ND block D and sketched row-stationary (csr_sketch_heavy):
//     thread = sketch row i, G[i, j] generated ONCE per (i, j) and reused by all
//     ND heavy columns of row j;
//   * the remaining nonzeros are sketched column-stationary from a CSC copy
//     (csr_sketch_light): thread = sketch row i, one G[i, j] per nonzero.
// The two lanes of a Box-Muller pair (rows 2q, 2q+1, C9) take two
// columns at a time: each evaluates one full pair (Philox + Box-Muller) for its
// own column and one shuffle swaps the halves (gaussian_lane2).
//
// The CSC copy is built deterministically (per-chunk counts, exclusive scans,
// in-order fill), so the sketch and the iterations are bitwise reproducible.
//
// Iteration (CSR long pass): u_j <- c1 u_j + c2 (A_j . t) from the CSR rows
// (csr_rowdot, which also accumulates the heavy columns of w = A^T u per block),
// then the light columns of w gathered column by column from the CSC copy
// (csr_colgather); out = [w ; ||u||^2] like colreduce_kernel.
#include <algorithm>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "philox_bm.cuh"

namespace lsrn {

namespace {
constexpr int THR = 256;

LSRN_DEV double block_sum(double v, double* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;   // valid in thread 0
}

// Two columns at once: G[i, ja] and G[i, jb] for the calling lane's sketch row i.
// Lane 2q evaluates the whole pair (G[2q, ja], G[2q+1, ja]), lane 2q+1 the pair
// (G[2q, jb], G[2q+1, jb]); one shuffle hands each lane the value it lacks.  Per
// normal this is half a Philox call and half a Box-Muller pair with every lane
// busy -- gaussian_lane (both lanes of a pair run the same Philox call) spends
// twice the integer work (the first version did that: the c4 sketch took 13.9 s,
// Philox-bound in the light part).
LSRN_DEV void gaussian_lane2(uint2 key, uint64_t q, uint64_t ja, uint64_t jb, bool odd, const double* T,
                             double& za, double& zb) {
  double z0, z1;
  box_muller_tab(philox_counter(key, q, odd ? jb : ja), T, z0, z1);
  // even lane owns row 2q: keeps z0(ja), needs z0(jb) from the odd lane;
  // odd lane owns row 2q+1: keeps z1(jb), needs z1(ja) from the even lane
  const double recv = __shfl_xor_sync(0xffffffffu, odd ? z0 : z1, 1);
  za = odd ? recv : z0;
  zb = odd ? z1 : recv;
}
}  // namespace

// ------------------------------------------------------------ CSC construction
// cntc[chunk][c] = number of nonzeros of column c in rows [chunk*CH, (chunk+1)*CH).
// Also validates the canonical-CSR contract (lsrn.h): column indices in [0, k)
// (bad |= 1) and strictly increasing within each row (bad |= 2) -- the CSC
// fill and the heavy-column accumulation rely on distinct columns per row.
__global__ void csr_chunk_count_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                       int64_t rows, int64_t k, int64_t CH, int* __restrict__ cntc,
                                       int* __restrict__ bad) {
  extern __shared__ int hist[];
  const int64_t chunk = blockIdx.x;
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  const int64_t r0 = chunk * CH, r1 = min(rows, r0 + CH);
  const int64_t base = rowptr[0];
  const int64_t e0 = rowptr[r0] - base, e1 = rowptr[r1] - base;
  int flag = 0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {     // row structure
    const int64_t a0 = rowptr[r] - base, a1 = rowptr[r + 1] - base;
    if (a1 < a0) flag |= 4;
    for (int64_t e = a0 + 1; e < a1; ++e)
      if (colind[e] <= colind[e - 1]) flag |= 2;
  }
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int c = colind[e];
    if (c < 0 || c >= k) {
      flag |= 1;
      continue;
    }
    atomicAdd(&hist[c], 1);   // integer: exact
  }
  if (flag) atomicOr(bad, flag);
  __syncthreads();
  int* out = cntc + chunk * k;
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) out[c] = hist[c];
}

// per column: total[c] = sum_chunk cntc; offs[chunk][c] = exclusive prefix over chunks (relative)
__global__ void csr_chunk_scan_kernel(const int* __restrict__ cntc, int64_t nchunks, int64_t k,
                                      int64_t* __restrict__ offs, int64_t* __restrict__ total) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < k; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t run = 0;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      offs[ch * k + c] = run;
      run += cntc[ch * k + c];
    }
    total[c] = run;
  }
}

// colptr = exclusive scan of the light-column totals (heavy columns hold no CSC
// entries: their values live in D).  Single CTA, sequential tiles of THR.
__global__ void csr_colptr_kernel(const int64_t* __restrict__ total, const int* __restrict__ colmap, int64_t k,
                                  int64_t* __restrict__ colptr) {
  __shared__ int64_t sh[THR];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < k; t0 += THR) {
    const int64_t c = t0 + threadIdx.x;
    const int64_t v = (c < k && colmap[c] < 0) ? total[c] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < THR; off <<= 1) {      // Hillis-Steele inclusive scan
      const int64_t add = (threadIdx.x >= off) ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += add;
      __syncthreads();
    }
    if (c < k) colptr[c] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == THR - 1) carry += sh[THR - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) colptr[k] = carry;
}

// Light entries per row chunk (for the light CSR's chunk offsets).
__global__ void csr_chunk_light_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                       int64_t rows, int64_t CH, const int* __restrict__ colmap,
                                       int64_t* __restrict__ lchunk_cnt) {
  __shared__ int64_t sh[THR / 32];
  const int64_t chunk = blockIdx.x;
  const int64_t base = rowptr[0];
  const int64_t r0 = chunk * CH, r1 = min(rows, r0 + CH);
  const int64_t e0 = rowptr[r0] - base, e1 = rowptr[r1] - base;
  int64_t n = 0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) n += colmap[colind[e]] < 0 ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < THR / 32; ++w) t += sh[w];
    lchunk_cnt[chunk] = t;
  }
}

// out[i] = sum_{i' < i} in[i'] for i <= n (out[n] = total).  Single CTA, tiles of THR.
__global__ void excl_scan_kernel(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  __shared__ int64_t sh[THR];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < n; t0 += THR) {
    const int64_t i = t0 + threadIdx.x;
    const int64_t v = i < n ? in[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < THR; off <<= 1) {      // Hillis-Steele inclusive scan
      const int64_t add = (threadIdx.x >= off) ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < n) out[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == THR - 1) carry += sh[THR - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// In-order fill of the CSC copy of the light columns (rowidx = local row, cval),
// of the heavy block D (rows x ld_d, zero-filled beforehand) and of the light CSR
// (lrowptr / lcol / lval: each row's light entries in their CSR order).  One CTA
// per chunk, one warp walking the chunk's rows in order (distinct columns within
// a row -> no conflicts; light positions within a row by ballot).
__global__ void csr_fill_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                const double* __restrict__ val, int64_t rows, int64_t k, int64_t CH,
                                const int64_t* __restrict__ offs, const int64_t* __restrict__ colptr,
                                const int* __restrict__ colmap, int32_t* __restrict__ rowidx,
                                double* __restrict__ cval, double* __restrict__ D, int64_t ld_d,
                                const int64_t* __restrict__ lchunk_off, int64_t* __restrict__ lrowptr,
                                int32_t* __restrict__ lcol, double* __restrict__ lval) {
  extern __shared__ int64_t cur[];
  const int64_t chunk = blockIdx.x;
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) cur[c] = colptr[c] + offs[chunk * k + c];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int64_t base = rowptr[0];
  const int64_t r1 = min(rows, (chunk + 1) * CH);
  int64_t lrun = lchunk_off[chunk];
  for (int64_t r = chunk * CH; r < r1; ++r) {
    const int64_t e0 = rowptr[r] - base, e1 = rowptr[r + 1] - base;
    if (lane == 0) lrowptr[r] = lrun;
    for (int64_t eb = e0; eb < e1; eb += 32) {
      const int64_t e = eb + lane;
      const bool ok = e < e1;
      const int c = ok ? colind[e] : 0;
      const double a = ok ? val[e] : 0.0;
      const int h = ok ? colmap[c] : 0;
      const unsigned lm = __ballot_sync(0xffffffffu, ok && h < 0);
      if (ok) {
        if (h >= 0) {
          D[r * ld_d + h] = a;
        } else {
          const int64_t pos = cur[c]++;
          rowidx[pos] = (int32_t)r;
          cval[pos] = a;
          const int64_t lp = lrun + __popc(lm & ((1u << lane) - 1u));
          lcol[lp] = c;
          lval[lp] = a;
        }
      }
      lrun += __popc(lm);
    }
    __syncwarp();
  }
  if (lane == 0 && r1 == rows) lrowptr[rows] = lrun;
}

// ------------------------------------------------------------ K4 sketch kernels
// Heavy part: part[split][i][h] = sum_{j in split} G[i, lo + j] D[j][h].
template <int ND>
__global__ void __launch_bounds__(THR)
csr_sketch_heavy_kernel(const double* __restrict__ D, int ldd, int nd, int64_t rows, int64_t lo, int64_t s,
                        uint64_t seed, int64_t rows_per_split, double* __restrict__ part) {
  constexpr int JT = 32;                       // D rows staged per step
  __shared__ __align__(16) double Ds[JT][ND];
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  const uint2 key = philox_key(seed);
  const int64_t i = (int64_t)blockIdx.x * THR + threadIdx.x;
  const bool odd = (threadIdx.x & 1) != 0;
  const uint64_t q = (uint64_t)(i >> 1);
  const int64_t j0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t j1 = min(rows, j0 + rows_per_split);
  double acc[ND];
#pragma unroll
  for (int h = 0; h < ND; ++h) acc[h] = 0.0;
  for (int64_t jb = j0; jb < j1; jb += JT) {
    const int nj = (int)min((int64_t)JT, j1 - jb);
    __syncthreads();
    for (int e = threadIdx.x; e < JT * ND; e += THR) {
      const int r = e / ND, h = e % ND;
      Ds[r][h] = (r < nj && h < nd) ? D[(jb + r) * ldd + h] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < nj; r += 2) {            // rows r, r+1 (Ds row nj is zero when nj is odd)
      double za, zb;
      gaussian_lane2(key, q, (uint64_t)(lo + jb + r), (uint64_t)(lo + jb + r + 1), odd, bmT, za, zb);
#pragma unroll
      for (int h = 0; h < ND; h += 2) {
        const double2 d = *reinterpret_cast<const double2*>(&Ds[r][h]);
        const double2 e = *reinterpret_cast<const double2*>(&Ds[r + 1][h]);
        acc[h] = fma(zb, e.x, fma(za, d.x, acc[h]));
        acc[h + 1] = fma(zb, e.y, fma(za, d.y, acc[h + 1]));
      }
    }
  }
  if (i < s) {
    double* o = part + ((int64_t)blockIdx.y * s + i) * ND;
#pragma unroll
    for (int h = 0; h < ND; ++h) o[h] = acc[h];
  }
}

// Light part: At[i][c] = sum_{(j, a) in CSC column c} G[i, lo + j] a for light columns.
// G[:, j] is regenerated for every light nonzero (s normals each).  A row-stationary
// alternative (CTA = IT sketch rows x all k columns in shared memory, every normal
// generated once, the light CSR streamed and bucketed by owner warp) was measured
// on t4 (k = 1024): 0.93 s (2.19 s without bucketing) against 0.66 s for this
// kernel -- the per-row-block synchronisation and the serial shared-memory updates
// cost more than the 21x redundant Box-Muller work saves.
__global__ void __launch_bounds__(THR)
csr_sketch_light_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                        const double* __restrict__ cval, const int* __restrict__ colmap, int64_t k, int64_t lo,
                        int64_t s, uint64_t seed, int cols_per_cta, double* __restrict__ At) {
  constexpr int NT = 256;                      // nonzeros staged per step
  __shared__ int32_t js[NT];
  __shared__ double as[NT];
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  __syncthreads();
  const uint2 key = philox_key(seed);
  const int64_t i = (int64_t)blockIdx.x * THR + threadIdx.x;
  const bool odd = (threadIdx.x & 1) != 0;
  const uint64_t q = (uint64_t)(i >> 1);
  const int64_t cb = (int64_t)blockIdx.y * cols_per_cta;
  for (int64_t c = cb; c < min(k, cb + cols_per_cta); ++c) {
    if (colmap[c] >= 0) continue;              // heavy column: written by the heavy finish
    const int64_t e0 = colptr[c], e1 = colptr[c + 1];
    double acc = 0.0;
    for (int64_t eb = e0; eb < e1; eb += NT) {
      const int ne = (int)min((int64_t)NT, e1 - eb);
      __syncthreads();
      if (threadIdx.x < ne) {
        js[threadIdx.x] = rowidx[eb + threadIdx.x];
        as[threadIdx.x] = cval[eb + threadIdx.x];
      }
      __syncthreads();
      for (int e = 0; e < ne; e += 2) {           // nonzeros e, e+1 (a = 0 past the end)
        const bool two = e + 1 < ne;
        double za, zb;
        gaussian_lane2(key, q, (uint64_t)(lo + js[e]), (uint64_t)(lo + js[two ? e + 1 : e]), odd, bmT, za, zb);
        acc = fma(za, as[e], acc);
        if (two) acc = fma(zb, as[e + 1], acc);
      }
    }
    if (i < s) At[i * k + c] = acc;
  }
}

// Generate-once light sketch (csr_sketch_slab_kernel).  The per-nonzero kernel
// above regenerates G[:, j] for every light nonzero of row j (21x the s L normals
// on t4).  Here a CTA owns IB = 32 sketch rows (lane = sketch row) and a tile of
// CW = 512 columns (warp w: columns w*32 .. w*32+31, one register accumulator per
// column per lane), and walks a range of CJ = 256-row chunks of the long index:
//   phase G: all threads generate the chunk's G tile Gs[jj][ii] (CJ x IB, 64 KB of
//            shared memory) -- each G[i, j] ONCE per column tile;
//   phase S: warp w, for each of its 32 columns c, runs over the column's CSC
//            entries that fall in the chunk (a contiguous sub-range of the CSC
//            column: cp[J][c] .. cp[J+1][c]) and accumulates acc[c] += Gs[jj][lane] a.
// Normals generated = s L x (number of column tiles), independent of nnz; the
// FMA side costs one shared load per (sketch row, nonzero).  Partial results of
// the long-index splits go to part[split][c][i] and are summed in fixed order
// (csr_slab_finish_kernel): deterministic, no atomics.
namespace slab {
constexpr int IB = 32;                // sketch rows per CTA (= lanes)
constexpr int NW = 16;                // warps per CTA
constexpr int THREADS = NW * 32;
constexpr int CPW = 32;               // columns per warp (register accumulators)
constexpr int CW = NW * CPW;          // 512 columns per CTA tile
constexpr int CJ = 256;               // long-index rows per chunk
constexpr int SW = 256;               // staged entries per warp and chunk (16 B each)
// shared memory: Gs[CJ][IB] | Box-Muller table | entries [NW][SW] (double2) |
//                column bases [NW][32] (int64) | column offsets [NW][33] (int)
constexpr size_t OFF_TAB = (size_t)CJ * IB * 8;
constexpr size_t OFF_ENT = (OFF_TAB + (size_t)bm::TAB_SIZE * 8 + 15) / 16 * 16;
constexpr size_t OFF_BASE = OFF_ENT + (size_t)NW * SW * 16;
constexpr size_t OFF_SOFF = OFF_BASE + (size_t)NW * 32 * 8;
constexpr size_t SMEM = OFF_SOFF + (size_t)NW * 33 * 4;
}  // namespace slab

__global__ void __launch_bounds__(slab::THREADS, 1)
csr_sketch_slab_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                       const double* __restrict__ cval, const int* __restrict__ colmap,
                       const int32_t* __restrict__ cp, int64_t k, int64_t rows, int64_t lo, int64_t s,
                       uint64_t seed, int64_t chunks_per_split, int64_t nchunks, double* __restrict__ part) {
  using namespace slab;
  extern __shared__ __align__(16) double smem[];
  char* sm = reinterpret_cast<char*>(smem);
  double* Gs = smem;                          // [CJ][IB]
  double* bmT = reinterpret_cast<double*>(sm + OFF_TAB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* ent = reinterpret_cast<double2*>(sm + OFF_ENT) + (size_t)warp * SW;
  int64_t* sbase = reinterpret_cast<int64_t*>(sm + OFF_BASE) + (size_t)warp * 32;
  int32_t* soff = reinterpret_cast<int32_t*>(sm + OFF_SOFF) + (size_t)warp * 33;
  bm_load_table(bmT);
  const uint2 key = philox_key(seed);
  const int64_t I = blockIdx.x;
  const int64_t c0 = (int64_t)blockIdx.y * CW + (int64_t)warp * CPW;
  const int64_t myc = c0 + lane;              // this lane's column, for the pointer loads
  const bool col_ok = myc < k && colmap[myc] < 0;
  const int64_t mybase = col_ok ? colptr[myc] : 0;
  double acc[CPW];
#pragma unroll
  for (int t = 0; t < CPW; ++t) acc[t] = 0.0;
  const int64_t J0 = (int64_t)blockIdx.z * chunks_per_split;
  const int64_t J1 = min(nchunks, J0 + chunks_per_split);
  for (int64_t J = J0; J < J1; ++J) {
    const int64_t jrow0 = J * CJ;
    const int32_t jr0 = (int32_t)jrow0;
    // Stage this warp's entries of the chunk first (one round of independent loads for
    // all 32 columns, overlapping other warps' work, instead of a dependent round trip
    // per column): lane t's column occupies ent[soff[t] .. soff[t+1]) as {value,
    // Gs row offset} pairs.  More than SW entries: direct loads below.
    int32_t e0 = 0, e1 = 0;
    if (col_ok) {
      e0 = __ldg(cp + J * k + myc);
      e1 = __ldg(cp + (J + 1) * k + myc);
    }
    int32_t incl = e1 - e0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const bool staged = total <= SW;
    if (staged) {
      soff[lane + 1] = incl;
      if (lane == 0) soff[0] = 0;
      sbase[lane] = mybase + e0;
      __syncwarp();
#pragma unroll 1
      for (int32_t f = lane; f < total; f += 32) {
        int lo_t = 0, hi_t = 31;                  // column t with soff[t] <= f < soff[t + 1]
#pragma unroll
        for (int it = 0; it < 5; ++it) {
          const int mid = (lo_t + hi_t + 1) >> 1;
          if (soff[mid] <= f) lo_t = mid; else hi_t = mid - 1;
        }
        const int64_t g = sbase[lo_t] + (f - soff[lo_t]);
        ent[f] = make_double2(__ldg(cval + g), __longlong_as_double((long long)(__ldg(rowidx + g) - jr0)));
      }
    }
    __syncthreads();                          // previous chunk's phase S done with Gs (and the table loaded)
#pragma unroll 2
    for (int p = threadIdx.x; p < CJ * (IB / 2); p += THREADS) {
      const int jj = p / (IB / 2), pp = p % (IB / 2);
      const int64_t j = jrow0 + jj;
      double z0 = 0.0, z1 = 0.0;
      if (j < rows) gaussian_pair(key, (uint64_t)(I * (IB / 2) + pp), (uint64_t)(lo + j), bmT, z0, z1);
      *reinterpret_cast<double2*>(&Gs[jj * IB + 2 * pp]) = make_double2(z0, z1);
    }
    __syncthreads();
    if (staged) {
#pragma unroll
      for (int t = 0; t < CPW; ++t) {
        const int q1 = soff[t + 1];
        double a = acc[t];
        int q = soff[t];
        // two entries per trip (loads of both issued before the dependent FMAs; the
        // accumulation order is unchanged)
#pragma unroll 1
        for (; q + 1 < q1; q += 2) {
          const double2 ev0 = ent[q], ev1 = ent[q + 1];   // broadcast
          const double g0 = Gs[(int)__double_as_longlong(ev0.y) * IB + lane];
          const double g1 = Gs[(int)__double_as_longlong(ev1.y) * IB + lane];
          a = fma(g0, ev0.x, a);
          a = fma(g1, ev1.x, a);
        }
        if (q < q1) {
          const double2 ev = ent[q];
          a = fma(Gs[(int)__double_as_longlong(ev.y) * IB + lane], ev.x, a);
        }
        acc[t] = a;
      }
      __syncwarp();                            // ent / soff restaged by the next chunk
    } else {
#pragma unroll
      for (int t = 0; t < CPW; ++t) {
        const int64_t base = __shfl_sync(0xffffffffu, mybase, t);
        const int32_t f0 = __shfl_sync(0xffffffffu, e0, t), f1 = __shfl_sync(0xffffffffu, e1, t);
        double a = acc[t];
#pragma unroll 1
        for (int32_t e = f0; e < f1; ++e)
          a = fma(Gs[(__ldg(rowidx + base + e) - jr0) * IB + lane], __ldg(cval + base + e), a);
        acc[t] = a;
      }
    }
  }
  const int64_t i = I * IB + lane;
  if (i < s) {
#pragma unroll
    for (int t = 0; t < CPW; ++t) {
      const int64_t c = c0 + t;
      if (c < k) part[((int64_t)blockIdx.z * k + c) * s + i] = acc[t];
    }
  }
}

// ---------------------------------------------------------------------------
// Stored-G CSR sketch (csr_sketch = 2, the default when the slab does not pay: c4).
// The per-nonzero kernel above evaluates G[:, j] once per light nonzero of row j
// (c4: 20 x s L = 1.6e12 normals, 7.3 s).  Here the rows of the shard are taken in
// chunks whose G block (s x rows, <= 8 GB) is generated ONCE (csr_gen_g_kernel,
// G[j][i] with i contiguous), and the heavy and light kernels read it instead of
// regenerating it: the heavy part streams it row by row, the light part gathers
// G[j, i-block] per nonzero (2 KB coalesced per 256 sketch rows) and accumulates
// into the transposed partial Pt[c][i] (coalesced read-modify-write, one per chunk;
// fixed chunk order: deterministic).  Memory for FLOPs: ~8 B of G traffic per
// (nonzero, sketch row) instead of a Box-Muller pair per two.
__global__ void __launch_bounds__(256)
csr_gen_g_kernel(double* __restrict__ G, int64_t s2, int64_t rows, int64_t jbase, uint64_t seed) {
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  __syncthreads();
  const uint2 key = philox_key(seed);
  // rows over CTAs, pairs of a row over threads: no 64-bit division per pair (the
  // flat index p -> (p / hp, p % hp) per pair: 162 -> 139 us per t4 launch,
  // profiles/r02_gen2d_launches_t4.txt)
  const int64_t hp = s2 / 2;
  for (int64_t jl = blockIdx.x; jl < rows; jl += gridDim.x) {
    double* Gr = G + jl * s2;
    const uint64_t j = (uint64_t)(jbase + jl);
    for (int64_t q = threadIdx.x; q < hp; q += blockDim.x) {
      double z0, z1;
      gaussian_pair(key, (uint64_t)q, j, bmT, z0, z1);
      *reinterpret_cast<double2*>(Gr + 2 * q) = make_double2(z0, z1);
    }
  }
}

// Heavy part from stored G: part[split][i][h] (+)= sum_{j in split} G[j][i] D[j][h].
// The JT rows' G values are loaded before their FMAs (JT loads in flight per thread:
// one at a time left the kernel latency-bound at 0.33 TB/s, 2 s on c4).
template <int ND>
__global__ void __launch_bounds__(THR)
csr_sketch_heavy_g_kernel(const double* __restrict__ D, int ldd, int nd, int64_t rows, const double* __restrict__ G,
                          int64_t s2, int64_t s, int64_t rows_per_split, double* __restrict__ part, int accumulate) {
  constexpr int JT = 16;
  __shared__ __align__(16) double Ds[JT][ND];
  const int64_t i = (int64_t)blockIdx.x * THR + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t j1 = min(rows, j0 + rows_per_split);
  double acc[ND];
#pragma unroll
  for (int h = 0; h < ND; ++h) acc[h] = 0.0;
  for (int64_t jb = j0; jb < j1; jb += JT) {
    const int nj = (int)min((int64_t)JT, j1 - jb);
    __syncthreads();
    for (int e = threadIdx.x; e < JT * ND; e += THR) {
      const int r = e / ND, h = e % ND;
      Ds[r][h] = (r < nj && h < nd) ? D[(jb + r) * ldd + h] : 0.0;
    }
    __syncthreads();
    if (i < s) {
      double z[JT];
#pragma unroll
      for (int r = 0; r < JT; ++r) z[r] = r < nj ? G[(jb + r) * s2 + i] : 0.0;
#pragma unroll
      for (int r = 0; r < JT; ++r)          // Ds rows past nj are zero
#pragma unroll
        for (int h = 0; h < ND; h += 2) {
          const double2 d = *reinterpret_cast<const double2*>(&Ds[r][h]);
          acc[h] = fma(z[r], d.x, acc[h]);
          acc[h + 1] = fma(z[r], d.y, acc[h + 1]);
        }
    }
  }
  if (i < s) {
    double* o = part + ((int64_t)blockIdx.y * s + i) * ND;
#pragma unroll
    for (int h = 0; h < ND; ++h) o[h] = accumulate ? o[h] + acc[h] : acc[h];
  }
}

// Heavy part from stored G on the FP64 tensor cores: part[split] (s x ND) (+)= G^T D over
// the split's rows, a GEMM with M = s, N = ND, K = rows.  CTA = 64 sketch rows x ND, 4
// warps of 16 x ND (DMMA.8x8x4 fragments), K in steps of 16 rows with both operand
// tiles (G rows are contiguous in i, D rows in h) double-buffered by cp.async.
constexpr int HM_M = 64, HM_K = 16, HM_THREADS = 128;
template <int ND>
__global__ void __launch_bounds__(HM_THREADS)
csr_sketch_heavy_mma_kernel(const double* __restrict__ D, int ldd, int nd, int64_t rows, const double* __restrict__ G,
                            int64_t s2, int64_t s, int64_t rows_per_split, double* __restrict__ part, int accumulate) {
  constexpr int LDG = HM_M + 4, LDD = ND + 4, NJ = ND / 8;
  __shared__ __align__(16) double Gs[2][HM_K][LDG];
  __shared__ __align__(16) double Ds[2][HM_K][LDD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * HM_M;
  const int64_t j0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t j1 = min(rows, j0 + rows_per_split);
  const int nk = j1 > j0 ? (int)((j1 - j0 + HM_K - 1) / HM_K) : 0;
  const int64_t mvalid = min((int64_t)HM_M, s - i0);           // sketch rows of this tile
  auto issue = [&](int kb, int b) {
    const int64_t jb = j0 + (int64_t)kb * HM_K;
    // G: HM_K rows x HM_M doubles (16-byte pieces; rows / sketch rows past the end read nothing, zero-filled)
    for (int e = tid; e < HM_K * HM_M / 2; e += HM_THREADS) {
      const int kk = e / (HM_M / 2), m2 = 2 * (e % (HM_M / 2));
      const bool ok = jb + kk < j1 && m2 < mvalid;
      const int nb = ok ? (m2 + 1 < mvalid ? 16 : 8) : 0;
      cp_async16(&Gs[b][kk][m2], ok ? G + (jb + kk) * s2 + i0 + m2 : G, nb);
    }
    for (int e = tid; e < HM_K * ND / 2; e += HM_THREADS) {
      const int kk = e / (ND / 2), h2 = 2 * (e % (ND / 2));
      const bool ok = jb + kk < j1 && h2 < nd;
      const int nb = ok ? (h2 + 1 < nd ? 16 : 8) : 0;
      cp_async16(&Ds[b][kk][h2], ok ? D + (jb + kk) * ldd + h2 : D, nb);
    }
  };
  double acc[2][NJ][2];
#pragma unroll
  for (int fi = 0; fi < 2; ++fi)
#pragma unroll
    for (int fj = 0; fj < NJ; ++fj) acc[fi][fj][0] = acc[fi][fj][1] = 0.0;
  if (nk > 0) issue(0, 0);
  cp_async_commit();
  for (int kb = 0; kb < nk; ++kb) {
    const int b = kb & 1;
    if (kb + 1 < nk) issue(kb + 1, b ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < HM_K / 4; ++ks) {
      const int k = ks * 4 + (lane & 3);
      double a[2], bf[NJ];
#pragma unroll
      for (int fi = 0; fi < 2; ++fi) a[fi] = Gs[b][k][warp * 16 + fi * 8 + (lane >> 2)];
#pragma unroll
      for (int fj = 0; fj < NJ; ++fj) bf[fj] = Ds[b][k][fj * 8 + (lane >> 2)];
#pragma unroll
      for (int fi = 0; fi < 2; ++fi)
#pragma unroll
        for (int fj = 0; fj < NJ; ++fj) dmma884(acc[fi][fj], a[fi], bf[fj]);
    }
    __syncthreads();                      // buffer b is refilled two steps later
  }
#pragma unroll
  for (int fi = 0; fi < 2; ++fi) {
    const int64_t i = i0 + warp * 16 + fi * 8 + (lane >> 2);
    if (i >= s) continue;
    double* o = part + ((int64_t)blockIdx.y * s + i) * ND;
#pragma unroll
    for (int fj = 0; fj < NJ; ++fj) {
      const int h = fj * 8 + 2 * (lane & 3);
      o[h] = accumulate ? o[h] + acc[fi][fj][0] : acc[fi][fj][0];
      o[h + 1] = accumulate ? o[h + 1] + acc[fi][fj][1] : acc[fi][fj][1];
    }
  }
}

// Light part from stored G, chunk J (rows [row0, row0 + rows) of the shard):
// Pt[c][i] (+)= sum over the light entries (j, a) of column c in the chunk of a G[j - row0][i].
template <int UNR>
__global__ void __launch_bounds__(THR)
csr_sketch_light_g_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                          const double* __restrict__ cval, const int* __restrict__ colmap,
                          const int32_t* __restrict__ cp, int64_t J, int64_t k, int64_t s, int64_t s2,
                          const double* __restrict__ G, int64_t row0, int cols_per_cta, double* __restrict__ Pt,
                          int accumulate) {
  constexpr int NT = 256;
  __shared__ int32_t js[NT];
  __shared__ double as[NT];
  // column groups fastest: the CTAs resident together share one sketch-row block, so
  // its slice of the chunk's G rows (2 KB each) stays in L2 for the ~20 nonzeros of a row
  const int64_t i = (int64_t)blockIdx.y * THR + threadIdx.x;
  const int64_t cb = (int64_t)blockIdx.x * cols_per_cta;
  for (int64_t c = cb; c < min(k, cb + cols_per_cta); ++c) {
    if (colmap[c] >= 0) continue;
    const int64_t e0 = colptr[c] + cp[J * k + c], e1 = colptr[c] + cp[(J + 1) * k + c];
    double acc = 0.0;
    for (int64_t eb = e0; eb < e1; eb += NT) {
      const int ne = (int)min((int64_t)NT, e1 - eb);
      __syncthreads();
      if (threadIdx.x < ne) {
        js[threadIdx.x] = (int32_t)(rowidx[eb + threadIdx.x] - row0);
        as[threadIdx.x] = cval[eb + threadIdx.x];
      }
      __syncthreads();
      if (i < s) {
        int e = 0;
        for (; e + UNR <= ne; e += UNR) {      // UNR gathers in flight
          double g[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) g[u] = G[(int64_t)js[e + u] * s2 + i];
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = fma(g[u], as[e + u], acc);
        }
        for (; e < ne; ++e) acc = fma(G[(int64_t)js[e] * s2 + i], as[e], acc);
      }
    }
    if (i < s) Pt[c * s + i] = accumulate ? Pt[c * s + i] + acc : acc;
  }
}

// cp[J][c] = number of CSC entries of light column c with row < J * CJ, J = 0..nchunks
// (warp per column; rows within a CSC column are ascending).  Heavy columns: 0.
__global__ void csr_chunkptr_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                                    const int* __restrict__ colmap, int64_t k, int64_t nchunks, int64_t chunk_rows,
                                    int32_t* __restrict__ cp) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= k) return;
  const int64_t e0 = colmap[c] < 0 ? colptr[c] : 0, e1 = colmap[c] < 0 ? colptr[c + 1] : 0;
  const int64_t n = e1 - e0;
  for (int64_t t = lane; t <= n; t += 32) {
    // chunks J in (chunk(t - 1), chunk(t)] start at entry t (chunk(-1) = -1, chunk(n) = nchunks)
    const int64_t hi = t < n ? rowidx[e0 + t] / chunk_rows : nchunks;
    const int64_t lo_ = t > 0 ? rowidx[e0 + t - 1] / chunk_rows : -1;
    for (int64_t J = lo_ + 1; J <= hi; ++J) cp[J * k + c] = (int32_t)t;
  }
}

// At[i][c] = sum_split part[split][c][i] for the light columns (fixed split order);
// 32 x 32 tiles through shared memory so that both sides are coalesced.
__global__ void csr_slab_finish_kernel(const double* __restrict__ part, int nsplit, int64_t s, int64_t k,
                                       const int* __restrict__ colmap, double* __restrict__ At) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t c = c0 + r, i = i0 + threadIdx.x;
    double v = 0.0;
    if (c < k && i < s)
      for (int sp = 0; sp < nsplit; ++sp) v += part[((int64_t)sp * k + c) * s + i];
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, c = c0 + threadIdx.x;
    if (i < s && c < k && colmap[c] < 0) At[i * k + c] = tile[threadIdx.x][r];
  }
}

// At[i][H[h]] = sum_split part[split][i][h]   (fixed split order)
__global__ void csr_heavy_finish_kernel(const double* __restrict__ part, int nsplit, int64_t s, int nd, int ND,
                                        const int* __restrict__ heavy_cols, int64_t k, double* __restrict__ At) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * nd; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nd;
    const int h = (int)(e % nd);
    double v = 0.0;
    for (int p = 0; p < nsplit; ++p) v += part[((int64_t)p * s + i) * ND + h];
    At[i * k + heavy_cols[h]] = v;
  }
}

// At[i][c] += si G[i, L + c]  (tall Tikhonov block, §5)
__global__ void sketch_add_gblock_kernel(double* __restrict__ At, int64_t s, int64_t k, int64_t L, double si,
                                         uint64_t seed) {
  __shared__ double bmT[bm::TAB_SIZE];
  bm_load_table(bmT);
  __syncthreads();
  const uint2 key = philox_key(seed);
  const int64_t npair = (s + 1) / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npair * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qq = e / k, c = e % k;
    double z0, z1;
    gaussian_pair(key, (uint64_t)qq, (uint64_t)(L + c), bmT, z0, z1);
    At[(2 * qq) * k + c] += si * z0;
    if (2 * qq + 1 < s) At[(2 * qq + 1) * k + c] += si * z1;
  }
}

// ------------------------------------------------------------ iteration kernels
// u_j <- c1 u_j + c2 (A_j . t) (warp per row, contiguous row blocks per warp);
// heavy columns h: wpart[block][h] = sum_j a_jh u_j (per-warp shared-memory
// accumulators; the heavy columns of one row are distinct, so no two lanes hit
// the same slot); npart[block] = partial ||u||^2.
template <int ND>
__global__ void __launch_bounds__(THR)
csr_rowdot_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                  const double* __restrict__ val, int64_t rows, const double* __restrict__ t,
                  const int* __restrict__ colmap, const double* __restrict__ coef, double sx, double* __restrict__ u,
                  double* __restrict__ acc, double* __restrict__ npart, double* __restrict__ wpart,
                  const int* __restrict__ done) {
  __shared__ double sh[THR / 32];
  __shared__ double wd[THR / 32][ND > 0 ? ND : 1];
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THR) >> 5;
  if (ND > 0)
    for (int h = lane; h < ND; h += 32) wd[wib][h] = 0.0;
  __syncwarp();
  const double c1 = coef[0], c2 = coef[1] * sx;
  const double ca = (acc != nullptr) ? coef[2] : 0.0;
  const int64_t base = rowptr[0];
  double nrm = 0.0;
  const int64_t per = (rows + nwarps - 1) / nwarps;
  const int64_t r0 = warp * per, r1 = min(rows, r0 + per);
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t e0 = rowptr[r] - base, e1 = rowptr[r + 1] - base;
    double d = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32) d = fma(val[e], __ldg(t + colind[e]), d);
    d = warp_sum(d);
    const double uo = __shfl_sync(0xffffffffu, lane == 0 ? u[r] : 0.0, 0);
    const double un = fma(c1, uo, c2 * d);
    if (lane == 0) {
      u[r] = un;
      if (acc != nullptr) acc[r] = fma(ca, un, acc[r]);   // CS, Alg. 2 form: x += alpha v on the long side
    }
    nrm = fma(un, un, nrm);
    if (ND > 0) {
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int h = colmap[colind[e]];
        if (h >= 0) wd[wib][h] = fma(val[e], un, wd[wib][h]);
      }
      __syncwarp();
    }
  }
  if (lane != 0) nrm = 0.0;
  const double b = block_sum(nrm, sh);     // contains __syncthreads: wd complete
  if (threadIdx.x == 0) npart[blockIdx.x] = b;
  if (ND > 0) {
    for (int h = threadIdx.x; h < ND; h += THR) {
      double v = 0.0;
      for (int w = 0; w < THR / 32; ++w) v += wd[w][h];
      wpart[(int64_t)blockIdx.x * ND + h] = sx * v;
    }
  }
}

// Long pass in the heavy-dense + light-CSR form (k > csr_rowdot_all_max_k()):
//   u_j <- c1 u_j + c2 (D_j . t_heavy + sum_light a t_c),  w_heavy += D_j u_j,
// npart[block] = partial ||u||^2, wpart[block][h] = sx sum_j D_jh u_j (fixed-order
// block reduction).  Lane l owns heavy columns l and l + 32 (t and the w
// accumulators in registers, no column map, no shared-memory atomics), the D row
// is one coalesced load, the ~20 light entries of a row one gather; two rows per
// step keep independent loads in flight.  The light w comes from the CSC gather.
template <int HPL>
__global__ void __launch_bounds__(THR)
csr_rowdot_hl_kernel(const double* __restrict__ D, int ldd, int ND, int nd, const int* __restrict__ heavy_cols,
                     const int64_t* __restrict__ lrowptr, const int32_t* __restrict__ lcol,
                     const double* __restrict__ lval, int64_t rows, const double* __restrict__ t,
                     const double* __restrict__ coef, double sx, double* __restrict__ u, double* __restrict__ acc,
                     double* __restrict__ npart, double* __restrict__ wpart, const int* __restrict__ done) {
  __shared__ double sh[THR / 32];
  __shared__ double wsh[THR / 32][HPL * 32];
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THR) >> 5;
  const double c1 = coef[0], c2 = coef[1] * sx;
  const double ca = (acc != nullptr) ? coef[2] : 0.0;
  double th[HPL], wh[HPL];
#pragma unroll
  for (int q = 0; q < HPL; ++q) {
    const int h = lane + 32 * q;
    th[q] = h < nd ? __ldg(t + heavy_cols[h]) : 0.0;
    wh[q] = 0.0;
  }
  double nrm = 0.0;
  const int64_t per = (rows + nwarps - 1) / nwarps;
  const int64_t r0 = warp * per, r1 = min(rows, r0 + per);
  const int64_t lbase = lrowptr[0];
  for (int64_t r = r0; r < r1; r += 2) {
    const bool has2 = r + 1 < r1;
    double da[HPL], db[HPL];
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
      const int h = lane + 32 * q;
      da[q] = h < nd ? ldg_stream1(D + r * ldd + h) : 0.0;
      db[q] = (h < nd && has2) ? ldg_stream1(D + (r + 1) * ldd + h) : 0.0;
    }
    const int64_t ea0 = lrowptr[r] - lbase, ea1 = lrowptr[r + 1] - lbase;
    const int64_t eb1 = has2 ? lrowptr[r + 2] - lbase : ea1;
    double sa = 0.0, sb = 0.0;
    for (int64_t e = ea0 + lane; e < ea1; e += 32) sa = fma(ldg_stream1(lval + e), __ldg(t + lcol[e]), sa);
    for (int64_t e = ea1 + lane; e < eb1; e += 32) sb = fma(ldg_stream1(lval + e), __ldg(t + lcol[e]), sb);
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
      sa = fma(da[q], th[q], sa);
      sb = fma(db[q], th[q], sb);
    }
    const double uoa = lane == 0 ? u[r] : 0.0;
    const double uob = (lane == 0 && has2) ? u[r + 1] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const double una = fma(c1, __shfl_sync(0xffffffffu, uoa, 0), c2 * sa);
    const double unb = has2 ? fma(c1, __shfl_sync(0xffffffffu, uob, 0), c2 * sb) : 0.0;
    if (lane == 0) {
      u[r] = una;
      if (acc != nullptr) acc[r] = fma(ca, una, acc[r]);
      nrm = fma(una, una, nrm);
      if (has2) {
        u[r + 1] = unb;
        if (acc != nullptr) acc[r + 1] = fma(ca, unb, acc[r + 1]);
        nrm = fma(unb, unb, nrm);
      }
    }
#pragma unroll
    for (int q = 0; q < HPL; ++q) wh[q] = fma(db[q], unb, fma(da[q], una, wh[q]));
  }
#pragma unroll
  for (int q = 0; q < HPL; ++q) wsh[wib][lane + 32 * q] = wh[q];
  if (lane != 0) nrm = 0.0;
  const double b = block_sum(nrm, sh);     // contains __syncthreads: wsh complete
  if (threadIdx.x == 0) npart[blockIdx.x] = b;
  for (int h = threadIdx.x; h < nd; h += THR) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < THR / 32; ++w) v += wsh[w][h];
    wpart[(int64_t)blockIdx.x * ND + h] = sx * v;
  }
}

// The same pass with eight rows per warp step and every load of the step issued
// up front: one coalesced load of the eight row pointers and u values, the D rows
// (lane l: heavy columns l, l + 32), and the batch's light entries as one
// contiguous stream (each lane adds its products to the row they fall in).  The
// eight row dots come out of one butterfly transpose-reduction (lane l ends with
// row (l >> 2) & 7).  Deterministic: fixed lane order and reduction tree.
template <int HPL>
__global__ void __launch_bounds__(THR)
csr_rowdot_hl8_kernel(const double* __restrict__ D, int ldd, int ND, int nd, const int* __restrict__ heavy_cols,
                      const int64_t* __restrict__ lrowptr, const int32_t* __restrict__ lcol,
                      const double* __restrict__ lval, int64_t rows, const double* __restrict__ t,
                      const double* __restrict__ coef, double sx, double* __restrict__ u, double* __restrict__ acc,
                      double* __restrict__ npart, double* __restrict__ wpart, const int* __restrict__ done) {
  constexpr int RB = 8;
  __shared__ double sh[THR / 32];
  __shared__ double wsh[THR / 32][HPL * 32];
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THR) >> 5;
  const double c1 = coef[0], c2 = coef[1] * sx;
  const double ca = (acc != nullptr) ? coef[2] : 0.0;
  double th[HPL], wh[HPL];
#pragma unroll
  for (int q = 0; q < HPL; ++q) {
    const int h = lane + 32 * q;
    th[q] = h < nd ? __ldg(t + heavy_cols[h]) : 0.0;
    wh[q] = 0.0;
  }
  double nrm = 0.0;
  int64_t per = (rows + nwarps - 1) / nwarps;
  per = (per + RB - 1) / RB * RB;
  const int64_t r0 = min(rows, warp * per), r1 = min(rows, r0 + per);
  const int64_t lbase = lrowptr[0];
  const int myrow = (lane >> 2) & 7;
  for (int64_t rb = r0; rb < r1; rb += RB) {
    const int nb = (int)min((int64_t)RB, r1 - rb);
    const int64_t lpl = lane <= nb ? lrowptr[rb + lane] - lbase : 0;
    const double uo = lane < nb ? u[rb + lane] : 0.0;
    double dv[RB][HPL];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int q = 0; q < HPL; ++q) {
        const int h = lane + 32 * q;
        dv[i][q] = (i < nb && h < nd) ? ldg_stream1(D + (rb + i) * ldd + h) : 0.0;
      }
    const int64_t e0 = __shfl_sync(0xffffffffu, lpl, 0);
    const int64_t e1 = __shfl_sync(0xffffffffu, lpl, nb);
    int off[RB];                                 // row starts relative to e0 (rows 1..7)
#pragma unroll
    for (int i = 1; i < RB; ++i) off[i] = (int)(__shfl_sync(0xffffffffu, lpl, i < nb ? i : nb) - e0);
    double ac[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) ac[i] = 0.0;
#pragma unroll 2
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const double prod = ldg_stream1(lval + e) * __ldg(t + lcol[e]);
      const int rel = (int)(e - e0);
      int ri = 0;
#pragma unroll
      for (int i = 1; i < RB; ++i) ri += rel >= off[i] ? 1 : 0;
#pragma unroll
      for (int i = 0; i < RB; ++i) ac[i] += ri == i ? prod : 0.0;
    }
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int q = 0; q < HPL; ++q) ac[i] = fma(dv[i][q], th[q], ac[i]);
    // butterfly transpose-reduction of ac[0..7] over the 32 lanes
    const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0, b2 = (lane & 4) != 0;
    double a4[4], a2[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double keep = b4 ? ac[i + 4] : ac[i], send = b4 ? ac[i] : ac[i + 4];
      a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double keep = b3 ? a4[i + 2] : a4[i], send = b3 ? a4[i] : a4[i + 2];
      a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double v;
    {
      const double keep = b2 ? a2[1] : a2[0], send = b2 ? a2[0] : a2[1];
      v = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    const double uor = __shfl_sync(0xffffffffu, uo, myrow);
    const double un = fma(c1, uor, c2 * v);               // row myrow (valid if myrow < nb)
    if ((lane & 3) == 0 && myrow < nb) {
      u[rb + myrow] = un;
      if (acc != nullptr) acc[rb + myrow] = fma(ca, un, acc[rb + myrow]);
      nrm = fma(un, un, nrm);
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const double uni = __shfl_sync(0xffffffffu, un, 4 * i);
      if (i < nb)
#pragma unroll
        for (int q = 0; q < HPL; ++q) wh[q] = fma(dv[i][q], uni, wh[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < HPL; ++q) wsh[wib][lane + 32 * q] = wh[q];
  // ||u||^2: fixed-order sum of the eight row-holder lanes of each warp
  double nw = 0.0;
#pragma unroll
  for (int i = 0; i < RB; ++i) nw += __shfl_sync(0xffffffffu, nrm, 4 * i);
  if (lane != 0) nw = 0.0;
  const double b = block_sum(nw, sh);      // contains __syncthreads: wsh complete
  if (threadIdx.x == 0) npart[blockIdx.x] = b;
  for (int h = threadIdx.x; h < nd; h += THR) {
    double w = 0.0;
#pragma unroll
    for (int ww = 0; ww < THR / 32; ++ww) w += wsh[ww][h];
    wpart[(int64_t)blockIdx.x * ND + h] = sx * w;
  }
}

// Single-pass CSR long pass for short rows of w (k <= csr_rowdot_all_max_k()):
// the same u update as csr_rowdot_kernel, and w = sx X^T u accumulated for ALL
// columns in per-warp shared-memory copies (the columns of one row are distinct,
// so lanes never collide), reduced over the block's warps in fixed order into
// wpart[block][k]; colreduce_kernel then sums the blocks and adds the norm.  X is
// read once per pass and no CSC gather is needed (the paper's t4 shape has
// k = 1024 columns of 82 000 nonzeros each: a warp-per-column gather had only
// 1024 warps of work and ran at 0.97 TB/s).
__global__ void __launch_bounds__(THR)
csr_rowdot_all_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                      const double* __restrict__ val, int64_t rows, int64_t k, const double* __restrict__ t,
                      const double* __restrict__ coef, double sx, double* __restrict__ u, double* __restrict__ acc,
                      double* __restrict__ npart, double* __restrict__ wpart, const int* __restrict__ done) {
  extern __shared__ double wsh[];            // [THR / 32][k]
  __shared__ double sh[THR / 32];
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* wd = wsh + (int64_t)wib * k;
  for (int64_t c = lane; c < k; c += 32) wd[c] = 0.0;
  __syncwarp();
  const int64_t warp = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THR) >> 5;
  const double c1 = coef[0], c2 = coef[1] * sx;
  const double ca = (acc != nullptr) ? coef[2] : 0.0;
  const int64_t base = rowptr[0];
  double nrm = 0.0;
  const int64_t per = (rows + nwarps - 1) / nwarps;
  const int64_t r0 = warp * per, r1 = min(rows, r0 + per);
  // Chunks of 32 rows: the row pointers, old u and acc of the chunk arrive in one
  // coalesced load each (lane l <-> row rc + l), and the new u / acc leave the same
  // way.  Inside a chunk two rows per step, software-pipelined: the colind / val
  // loads of the next pair are issued before the current pair is reduced, so their
  // DRAM latency overlaps the current pair's t-gathers, shuffles and shared-memory
  // updates (t4: 1.0 -> 0.70 ms per pass; the first version waited on rowptr ->
  // colind -> t per pair; four rows per step with the same pipelining: 1.37 ms; an
  // L2 prefetch of the next chunk's entries: 1.01 ms).  Rows of <= 32 entries keep (c, a) in registers for the w update;
  // longer rows loop.  Also rejected (round 2, t4): staging each warp's next 32-row chunk in
  // shared memory with cp.async (8 KB in flight per warp, but 8 warps per SM: 0.84-1.30 ms)
  // and lane-per-row dots without the shuffle tree (half the instructions, 0.88 ms): both
  // leave the per-row w scatter (shared-memory read-modify-write chain, one row at a time)
  // as the critical path, which the two-row pipelining here overlaps with the next loads.
  for (int64_t rc = r0; rc < r1; rc += 32) {
    const int nr = (int)min((int64_t)32, r1 - rc);
    const int64_t rp = lane < nr ? rowptr[rc + lane] - base : 0;
    const int64_t rpend = rowptr[rc + nr] - base;

    const double uold = lane < nr ? u[rc + lane] : 0.0;
    const double aold = (acc != nullptr && lane < nr) ? acc[rc + lane] : 0.0;
    double unew = 0.0;
    auto rptr = [&](int i) -> int64_t {        // row pointer of chunk row i (i <= nr)
      const int64_t v = __shfl_sync(0xffffffffu, rp, i & 31);
      return i < nr ? v : rpend;
    };
    // prefetched first 32 entries of rows (i, i+1)
    int nca = 0, ncb = 0;
    double naa = 0.0, nab = 0.0;
    auto prefetch = [&](int i) {
      const int64_t e0 = rptr(i), e1 = rptr(i + 1), e2 = (i + 1 < nr) ? rptr(i + 2) : e1;
      nca = ncb = 0;
      naa = nab = 0.0;
      if (e0 + lane < e1) {
        nca = colind[e0 + lane];
        naa = ldg_stream1(val + e0 + lane);
      }
      if (e1 + lane < e2) {
        ncb = colind[e1 + lane];
        nab = ldg_stream1(val + e1 + lane);
      }
    };
    prefetch(0);
    for (int i = 0; i < nr; i += 2) {
      const bool has2 = i + 1 < nr;
      const int64_t ea0 = rptr(i), ea1 = rptr(i + 1);
      const int64_t eb1 = has2 ? rptr(i + 2) : ea1;
      const int ca_ = nca, cb_ = ncb;
      const double aa = naa, ab = nab;
      if (i + 2 < nr) prefetch(i + 2);          // next pair's loads in flight during this pair
      double da = (ea0 + lane < ea1) ? aa * __ldg(t + ca_) : 0.0;
      double db = (ea1 + lane < eb1) ? ab * __ldg(t + cb_) : 0.0;
      for (int64_t e = ea0 + 32 + lane; e < ea1; e += 32) da = fma(val[e], __ldg(t + colind[e]), da);
      for (int64_t e = ea1 + 32 + lane; e < eb1; e += 32) db = fma(val[e], __ldg(t + colind[e]), db);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        da += __shfl_xor_sync(0xffffffffu, da, o);
        db += __shfl_xor_sync(0xffffffffu, db, o);
      }
      const double una = fma(c1, __shfl_sync(0xffffffffu, uold, i), c2 * da);
      const double unb = fma(c1, __shfl_sync(0xffffffffu, uold, (i + 1) & 31), c2 * db);
      if (lane == i) unew = una;
      if (has2 && lane == i + 1) unew = unb;
      if (ea0 + lane < ea1) wd[ca_] = fma(aa, una, wd[ca_]);
      for (int64_t e = ea0 + 32 + lane; e < ea1; e += 32) wd[colind[e]] = fma(val[e], una, wd[colind[e]]);
      __syncwarp();                           // row b may share columns with row a
      if (has2) {
        if (ea1 + lane < eb1) wd[cb_] = fma(ab, unb, wd[cb_]);
        for (int64_t e = ea1 + 32 + lane; e < eb1; e += 32) wd[colind[e]] = fma(val[e], unb, wd[colind[e]]);
      }
      __syncwarp();
    }
    if (lane < nr) {
      u[rc + lane] = unew;
      if (acc != nullptr) acc[rc + lane] = fma(ca, unew, aold);
      nrm = fma(unew, unew, nrm);
    }
  }
  const double b = block_sum(nrm, sh);     // contains __syncthreads: every warp's wd complete
  if (threadIdx.x == 0) npart[blockIdx.x] = b;
  for (int64_t c = threadIdx.x; c < k; c += THR) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < THR / 32; ++w) v += wsh[(int64_t)w * k + c];
    wpart[(int64_t)blockIdx.x * k + c] = sx * v;
  }
}

// Dots of G rows, one value per lane on entry (lane's share of row j in d[j]),
// reduced by a transposing butterfly: at offset 16 a lane keeps one half of its G
// values and sends the other half, at 8 a quarter, ... (G - 1 + 5 - log2 G
// shuffles instead of 5 G).  On exit d[0] of lane l is the sum of row l >> (5 - log2 G).
template <int G>
LSRN_DEV double transpose_reduce(double (&d)[G], int lane) {
  int off = 16;
#pragma unroll
  for (int n = G; n > 1; n >>= 1, off >>= 1) {
    const int half = n >> 1;
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? d[i] : d[i + half];
      const double keep = hi ? d[i + half] : d[i];
      d[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (; off > 0; off >>= 1) d[0] += __shfl_xor_sync(0xffffffffu, d[0], off);
  return d[0];
}

// The single-pass long pass of csr_rowdot_all_kernel with a deeper load pipeline.
// That kernel keeps one pair of rows (~0.5 KB on t4) in flight per warp, so 24 warps
// per SM hold ~12 KB and the pass is DRAM-latency bound (1.57 TB/s on t4).  Here a
// warp walks its rows in chunks of G * NB rows, each chunk in NB groups of G rows;
// the first 32 entries of every row of a group (colind, val) are loaded into a ring
// of NB register buffers NB - 1 groups ahead of the group being reduced, the row
// pointers / u / acc of a chunk two chunks ahead.  A group is reduced in one
// transposing butterfly (transpose_reduce), then its rows update the warp's shared
// copy of w one row at a time in row order (rows may share columns), exactly as in
// csr_rowdot_all_kernel.  Deterministic (fixed lane order, reduction tree and row
// order); rows longer than 32 entries take the remainder from global memory.
template <int G, int NB, int MINB, bool TS>
__global__ void __launch_bounds__(THR, MINB)
csr_rowdot_all_pipe_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                           const double* __restrict__ val, int64_t rows, int64_t k, const double* __restrict__ t,
                           const double* __restrict__ coef, double sx, double* __restrict__ u,
                           double* __restrict__ acc, double* __restrict__ npart, double* __restrict__ wpart,
                           const int* __restrict__ done) {
  constexpr int CHUNK = G * NB;
  static_assert(CHUNK <= 32 && (G & (G - 1)) == 0 && G <= 32, "chunk of at most 32 rows, G a power of two");
  constexpr int SH = (G == 1) ? 5 : (G == 2) ? 4 : (G == 4) ? 3 : (G == 8) ? 2 : (G == 16) ? 1 : 0;
  extern __shared__ double wsh[];            // [THR / 32][k] (+ t[k] when TS)
  __shared__ double sh[THR / 32];
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* wd = wsh + (int64_t)wib * k;
  for (int64_t c = lane; c < k; c += 32) wd[c] = 0.0;
  // TS: t gathered from shared memory.  A row's ~21 random t[c] hit ~18 distinct 128-byte
  // lines, i.e. ~18 L1 wavefronts per gather, against ~3-4 bank-conflict wavefronts from
  // shared memory; the L1 / shared-memory data path is the pass's bottleneck on t4.
  const double* tg = t;
  if (TS) {
    double* ts = wsh + (int64_t)(THR / 32) * k;
    for (int64_t c = threadIdx.x; c < k; c += THR) ts[c] = t[c];
    __syncthreads();
    tg = ts;
  } else {
    __syncwarp();
  }
  const int64_t warp = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THR) >> 5;
  const double c1 = coef[0], c2 = coef[1] * sx;
  const bool has_acc = acc != nullptr;
  const double ca = has_acc ? coef[2] : 0.0;
  const int64_t base = rowptr[0];
  const int64_t per = (rows + nwarps - 1) / nwarps;
  const int64_t r0 = min(rows, warp * per), r1 = min(rows, r0 + per);
  const int64_t nchunks = (r1 - r0 + CHUNK - 1) / CHUNK;

  // chunk descriptor: cb = the chunk's first entry (relative to the shard); lane l holds
  // rp = the row pointer of row min(l, nr) of the chunk minus cb (a chunk has at most
  // CHUNK k entries since the columns of a row are distinct), end = the pointer past the
  // chunk's last row; uo / ao = old u / acc of row l
  struct Chunk {
    int64_t cb;
    int rp, end;
    double uo, ao;
  };
  auto load_chunk = [&](int64_t ci, Chunk& C) {
    C.cb = 0;
    C.rp = 0;
    C.end = 0;
    C.uo = 0.0;
    C.ao = 0.0;
    if (ci < nchunks) {
      const int64_t rc = r0 + ci * CHUNK;
      const int nr = (int)min((int64_t)CHUNK, r1 - rc);
      const int64_t p = rowptr[rc + min(lane, nr)] - base;
      const int64_t pe = rowptr[rc + nr] - base;
      C.cb = __shfl_sync(0xffffffffu, p, 0);
      C.rp = (int)(p - C.cb);
      C.end = (int)(pe - C.cb);
      if (lane < nr) {
        C.uo = u[rc + lane];
        if (has_acc) C.ao = acc[rc + lane];
      }
    }
  };
  auto rptr = [&](const Chunk& C, int i) -> int {   // i in [0, CHUNK]
    const int v = __shfl_sync(0xffffffffu, C.rp, i & 31);
    return i < CHUNK ? v : C.end;
  };
  struct Buf {
    int c[G];          // column, -1 where the lane holds no entry of row j
    double a[G];
  };
  auto load_group = [&](const Chunk& C, int q, Buf& B) {
    const int32_t* ci_ = colind + C.cb;
    const double* va_ = val + C.cb;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int e0 = rptr(C, q * G + j), e1 = rptr(C, q * G + j + 1);
      B.c[j] = -1;
      B.a[j] = 0.0;
      if (e0 + lane < e1) {
        B.c[j] = ci_[e0 + lane];
        B.a[j] = ldg_stream1(va_ + e0 + lane);
      }
    }
  };
  double nrm = 0.0;
  auto reduce_group = [&](const Chunk& C, int64_t ci, int q, const Buf& B, bool lng) {
    double d[G];
#pragma unroll
    for (int j = 0; j < G; ++j) d[j] = (B.c[j] >= 0) ? B.a[j] * tg[B.c[j]] : 0.0;
    if (lng) {                                                 // rows of more than 32 entries
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int64_t e0 = C.cb + rptr(C, q * G + j), e1 = C.cb + rptr(C, q * G + j + 1);
        for (int64_t e = e0 + 32 + lane; e < e1; e += 32) d[j] = fma(val[e], tg[colind[e]], d[j]);
      }
    }
    const double dot = transpose_reduce<G>(d, lane);
    const int R = lane >> SH;                                  // this lane's row of the group
    const int rin = q * G + R;                                 // row within the chunk
    const int64_t row = r0 + ci * CHUNK + rin;
    const double un = fma(c1, __shfl_sync(0xffffffffu, C.uo, rin), c2 * dot);
    const double ao = __shfl_sync(0xffffffffu, C.ao, rin);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const double uj = __shfl_sync(0xffffffffu, un, j << SH);
      if (B.c[j] >= 0) wd[B.c[j]] = fma(B.a[j], uj, wd[B.c[j]]);
      if (lng) {
        const int64_t e0 = C.cb + rptr(C, q * G + j), e1 = C.cb + rptr(C, q * G + j + 1);
        for (int64_t e = e0 + 32 + lane; e < e1; e += 32) wd[colind[e]] = fma(val[e], uj, wd[colind[e]]);
      }
      __syncwarp();                                            // the next row may share columns
    }
    if ((lane & ((1 << SH) - 1)) == 0 && row < r1) {
      u[row] = un;
      if (has_acc) acc[row] = fma(ca, un, ao);
      nrm = fma(un, un, nrm);
    }
  };

  Chunk C0, C1, C2;
  Buf B[NB];
  load_chunk(0, C0);
  load_chunk(1, C1);
#pragma unroll
  for (int q = 0; q < NB - 1; ++q) load_group(C0, q, B[q]);
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    load_chunk(ci + 2, C2);
    // rows of more than 32 entries in this chunk (warp-uniform)
    const int nxt = rptr(C0, min(lane + 1, CHUNK));            // every lane shuffles
    const bool lng = __any_sync(0xffffffffu, lane < CHUNK && nxt - C0.rp > 32);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      // group q + NB - 1 of this chunk, or group q - 1 of the next, into the buffer freed last
      if (q == 0)
        load_group(C0, NB - 1, B[NB - 1]);
      else
        load_group(C1, q - 1, B[q - 1]);
      reduce_group(C0, ci, q, B[q], lng);
    }
    C0 = C1;
    C1 = C2;
  }
  const double b = block_sum(nrm, sh);     // contains __syncthreads: every warp's wd complete
  if (threadIdx.x == 0) npart[blockIdx.x] = b;
  for (int64_t c = threadIdx.x; c < k; c += THR) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < THR / 32; ++w) v += wsh[(int64_t)w * k + c];
    wpart[(int64_t)blockIdx.x * k + c] = sx * v;
  }
}

// w_c = sum_{(j,a) in col c} a u_j (light columns: warp per column, lanes stride
// the CSC column; heavy columns: the row pass's block partials);
// Tikhonov block and ||u||^2 as in colreduce_kernel: out = [w ; ||u||^2 + ||zI||^2].
__global__ void __launch_bounds__(THR)
csr_colgather_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                     const double* __restrict__ cval, int64_t k, double sx, const double* __restrict__ u,
                     const int* __restrict__ colmap, const double* __restrict__ wpart, int ND,
                     const double* __restrict__ npart, int nparts, double* __restrict__ zI,
                     const double* __restrict__ t, const double* __restrict__ coef, double sI,
                     double* __restrict__ out, double* __restrict__ blockpart, unsigned* __restrict__ counter,
                     const int* __restrict__ done) {
  __shared__ double sh[THR / 32];
  __shared__ bool last;
  if (done != nullptr && *done != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * THR + threadIdx.x) >> 5;
  double nI = 0.0;
  if (c < k) {
    double w = 0.0;
    const int h = colmap[c];
    if (h >= 0) {          // heavy: fixed-order sum of the row-pass block partials
      for (int g = lane; g < nparts; g += 32) w += wpart[(int64_t)g * ND + h];
    } else {
      // (four entries per lane in flight ran slower: 278 vs 200 us on the c4-shaped pass)
      for (int64_t e = colptr[c] + lane; e < colptr[c + 1]; e += 32) w = fma(cval[e], u[rowidx[e]], w);
      w *= sx;
    }
    w = warp_sum(w);
    if (zI != nullptr) {
      const double zn = fma(coef[0], zI[c], coef[1] * (sI * t[c]));
      if (lane == 0) zI[c] = zn;
      w = fma(sI, zn, w);
      nI = (lane == 0) ? zn * zn : 0.0;
    }
    if (lane == 0) out[c] = w;
  }
  const double b = block_sum(nI, sh);
  if (threadIdx.x == 0) {
    blockpart[blockIdx.x] = b;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    const double n = warp_sum_l2(npart, nparts) + warp_sum_l2(blockpart, gridDim.x);
    if (threadIdx.x == 0) {
      out[k] = n;
      *counter = 0u;
    }
  }
}

// ------------------------------------------------------------ host side
int64_t csr_chunk_rows() { return 8192; }
int64_t csr_nchunks(int64_t rows) { return rows > 0 ? (rows + csr_chunk_rows() - 1) / csr_chunk_rows() : 0; }
int csr_rowdot_blocks(int nsm) { return nsm * 8; }
// heavy-dense + light-CSR pass: one wave of resident CTAs (<= csr_rowdot_blocks)
int csr_rowdot_hl_blocks(int nsm, int ND) {
  int per_sm = 0;
  cudaError_t e = ND > 32 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_rowdot_hl8_kernel<2>, THR, 0)
                          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_rowdot_hl8_kernel<1>, THR, 0);
  if (e != cudaSuccess || per_sm < 1) per_sm = 2;
  return nsm * std::min(per_sm, 8);
}
int64_t csr_rowdot_all_max_k() { return 2048; }      // 8 warps x k doubles of shared memory (128 KB)
// Variants of the single pass (option csr_all): 0 csr_rowdot_all_kernel (round 1, one
// pair of rows in flight per warp); 6 the pipelined kernel, (G, NB) = (8, 2), t read
// through L1; 10 (default) the same with t in shared memory.  The other pipelines
// measured on t4 -- (8,4) (4,4) (4,8) (4,2) (2,4), with and without TS, 0.52-0.91 ms
// against 0.42 ms -- were removed (profiles/r02_csr_all_t4*.jsonl).
namespace {
int all_minb(int v) { return (v == 6 || v == 10) ? 2 : 4; }
bool all_ts(int v) { return v == 10; }     // t staged in shared memory
const void* all_kernel(int v) {
  switch (v) {
    case 6: return (const void*)csr_rowdot_all_pipe_kernel<8, 2, 2, false>;
    case 10: return (const void*)csr_rowdot_all_pipe_kernel<8, 2, 2, true>;
    default: return (const void*)csr_rowdot_all_kernel;
  }
}
}  // namespace
int csr_rowdot_all_default_variant() { return 10; }
// CTAs of 8 warps, as many per SM as the per-warp w copies (8 k doubles) and the
// variant's registers allow
int csr_rowdot_all_blocks(int nsm, int64_t k, int variant) {
  const int64_t per_cta = 8 * k * (THR / 32 + (all_ts(variant) ? 1 : 0));
  int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (220 * 1024) / per_cta));
  per_sm = std::min<int64_t>(per_sm, all_minb(variant));
  return (int)(nsm * per_sm);
}
int csr_rowdot_all_blocks_max(int nsm, int64_t k) {
  int b = 0;
  for (int v : {0, 6, 10}) b = std::max(b, csr_rowdot_all_blocks(nsm, k, v));
  return b;
}

cudaError_t launch_csr_rowdot_all(const CsrRowdotArgs& a, int64_t k, int variant, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)(THR / 32 + (all_ts(variant) ? 1 : 0)) * (size_t)k;
  const void* fn = all_kernel(variant);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&a.rowptr, (void*)&a.colind, (void*)&a.val, (void*)&a.rows, (void*)&k, (void*)&a.t,
                  (void*)&a.coef, (void*)&a.sx, (void*)&a.u, (void*)&a.acc, (void*)&a.npart, (void*)&a.wpart,
                  (void*)&a.done};
  e = cudaLaunchKernel(fn, dim3((unsigned)a.nblocks), dim3(THR), args, smem, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
int csr_colgather_blocks(int64_t k) { return (int)((k * 32 + THR - 1) / THR); }
size_t csr_max_k() { return 24 * 1024; }     // CSC cursors (int64) of a chunk live in shared memory

static unsigned grid_cap(int64_t n, int threads, int64_t cap) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

cudaError_t launch_csr_build(const CsrBuildArgs& a, cudaStream_t st) {
  const int64_t nch = csr_nchunks(a.rows);
  const int64_t CH = csr_chunk_rows();
  cudaError_t e0 = cudaMemsetAsync(a.bad, 0, sizeof(int), st);
  if (e0 != cudaSuccess) return e0;
  if (nch > 0) {
    const size_t sh1 = sizeof(int) * (size_t)a.k;
    cudaError_t e = cudaFuncSetAttribute(csr_chunk_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh1);
    if (e != cudaSuccess) return e;
    csr_chunk_count_kernel<<<(unsigned)nch, 512, sh1, st>>>(a.rowptr, a.colind, a.rows, a.k, CH, a.cntc, a.bad);
  }
  csr_chunk_scan_kernel<<<grid_cap(a.k, 256, 4096), 256, 0, st>>>(a.cntc, nch, a.k, a.offs, a.total);
  return cudaGetLastError();
}

cudaError_t launch_csr_fill(const CsrBuildArgs& a, cudaStream_t st) {
  const int64_t nch = csr_nchunks(a.rows);
  csr_colptr_kernel<<<1, THR, 0, st>>>(a.total, a.colmap, a.k, a.colptr);
  if (nch > 0)
    csr_chunk_light_kernel<<<(unsigned)nch, THR, 0, st>>>(a.rowptr, a.colind, a.rows, csr_chunk_rows(), a.colmap,
                                                           a.lchunk_cnt);
  excl_scan_kernel<<<1, THR, 0, st>>>(a.lchunk_cnt, nch, a.lchunk_off);
  if (a.rows == 0) {
    cudaError_t e = cudaMemsetAsync(a.lrowptr, 0, sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
  }
  if (a.D != nullptr && a.rows > 0) {
    cudaError_t e = cudaMemsetAsync(a.D, 0, sizeof(double) * (size_t)a.rows * a.ld_d, st);
    if (e != cudaSuccess) return e;
  }
  if (nch > 0) {
    const size_t sh = sizeof(int64_t) * (size_t)a.k;
    cudaError_t e = cudaFuncSetAttribute(csr_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    if (e != cudaSuccess) return e;
    csr_fill_kernel<<<(unsigned)nch, 256, sh, st>>>(a.rowptr, a.colind, a.val, a.rows, a.k, csr_chunk_rows(), a.offs,
                                                    a.colptr, a.colmap, a.rowidx, a.cval, a.D, a.ld_d, a.lchunk_off,
                                                    a.lrowptr, a.lcol, a.lval);
  }
  return cudaGetLastError();
}

template <int ND>
static void heavy_t(const CsrSketchArgs& a, dim3 grid, cudaStream_t st) {
  csr_sketch_heavy_kernel<ND><<<grid, THR, 0, st>>>(a.D, a.ldd, a.nd, a.rows, a.lo, a.s, a.seed, a.rows_per_split,
                                                    a.part);
}

cudaError_t launch_csr_sketch(const CsrSketchArgs& a, cudaStream_t st, int nsm) {
  const unsigned row_blocks = (unsigned)((a.s + THR - 1) / THR);
  if (a.nd > 0) {
    dim3 grid(row_blocks, (unsigned)a.nsplit);
    switch (a.ND) {
      case 16: heavy_t<16>(a, grid, st); break;
      case 32: heavy_t<32>(a, grid, st); break;
      default: heavy_t<64>(a, grid, st); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    csr_heavy_finish_kernel<<<grid_cap(a.s * a.nd, 256, (int64_t)nsm * 16), 256, 0, st>>>(
        a.part, a.nsplit, a.s, a.nd, a.ND, a.heavy_cols, a.k, a.At);
  }
  if (a.skip_light) return cudaSuccess;        // light part by the generate-once slab kernel
  const int cpc = 4;
  dim3 g2(row_blocks, (unsigned)((a.k + cpc - 1) / cpc));
  csr_sketch_light_kernel<<<g2, THR, 0, st>>>(a.colptr, a.rowidx, a.cval, a.colmap, a.k, a.lo, a.s, a.seed, cpc,
                                              a.At);
  return cudaGetLastError();
}

int64_t csr_slab_chunk_rows() { return slab::CJ; }
int64_t csr_slab_tile_cols() { return slab::CW; }
int64_t csr_slab_row_blocks(int64_t s) { return (s + slab::IB - 1) / slab::IB; }

cudaError_t launch_csr_chunkptr(const int64_t* colptr, const int32_t* rowidx, const int* colmap, int64_t k,
                                int64_t nchunks, int32_t* cp, cudaStream_t st, int64_t chunk_rows) {
  if (k <= 0) return cudaSuccess;
  if (chunk_rows <= 0) chunk_rows = slab::CJ;
  csr_chunkptr_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, st>>>(colptr, rowidx, colmap, k, nchunks,
                                                                       chunk_rows, cp);
  return cudaGetLastError();
}

template <int ND>
static void heavy_g_t(const CsrSketchGArgs& a, const double* G, int64_t rows, int64_t rps, int nsplit, int acc,
                      cudaStream_t st) {
  if (ovr().csr_heavy_fma == 1) {          // the FP64-FMA kernel (reference for the DMMA one)
    dim3 grid((unsigned)((a.s + THR - 1) / THR), (unsigned)nsplit);
    csr_sketch_heavy_g_kernel<ND><<<grid, THR, 0, st>>>(a.D + 0, a.ldd, a.nd, rows, G, a.s2, a.s, rps, a.part, acc);
    return;
  }
  dim3 grid((unsigned)((a.s + HM_M - 1) / HM_M), (unsigned)nsplit);
  csr_sketch_heavy_mma_kernel<ND><<<grid, HM_THREADS, 0, st>>>(a.D, a.ldd, a.nd, rows, G, a.s2, a.s, rps, a.part, acc);
}

int64_t csr_g_s2(int64_t s) { return (s + 1) / 2 * 2; }

cudaError_t launch_csr_sketch_g(const CsrSketchGArgs& a, cudaStream_t st, int nsm) {
  const int64_t nch = (a.rows + a.g_rows - 1) / a.g_rows;
  const unsigned row_blocks = (unsigned)((a.s + THR - 1) / THR);
  cudaError_t e = launch_csr_chunkptr(a.colptr, a.rowidx, a.colmap, a.k, nch, a.cp, st, a.g_rows);
  if (e != cudaSuccess) return e;
  for (int64_t J = 0; J < nch; ++J) {
    const int64_t r0 = J * a.g_rows, nr = std::min(a.g_rows, a.rows - r0);
    csr_gen_g_kernel<<<grid_cap(nr, 1, (int64_t)nsm * 16), 256, 0, st>>>(a.G, a.s2, nr, a.lo + r0, a.seed);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (a.nd > 0) {
      const int64_t rps = (nr + a.nsplit - 1) / a.nsplit;
      const double* D = a.D + r0 * a.ldd;
      CsrSketchGArgs b = a;
      b.D = D;
      switch (a.ND) {
        case 16: heavy_g_t<16>(b, a.G, nr, rps, a.nsplit, J > 0, st); break;
        case 32: heavy_g_t<32>(b, a.G, nr, rps, a.nsplit, J > 0, st); break;
        default: heavy_g_t<64>(b, a.G, nr, rps, a.nsplit, J > 0, st); break;
      }
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // columns per CTA and gathers in flight per thread (csr_light: 10 * cpc + unroll).
    // Round 1 used 16 columns and 4 gathers: t4's grid of 64 x 8 CTAs held 27 warps per SM
    // and the gathers were latency-bound (ncu: 22 cycles per issued instruction, L2 41 %
    // busy).  One column per CTA for k <= 2048 (t4: 8192 CTAs), four above (c4), eight
    // gathers in flight: t4 207 -> 147 ms, c4 1.98 -> 1.82 s (profiles/r02_csr_light*.jsonl).
    const int cpc = ovr().csr_light > 0 ? ovr().csr_light / 10 : (a.k <= 2048 ? 1 : 4);
    const int unr = ovr().csr_light > 0 ? ovr().csr_light % 10 : 8;
    dim3 g2((unsigned)((a.k + cpc - 1) / cpc), row_blocks);
    if (unr == 8)
      csr_sketch_light_g_kernel<8><<<g2, THR, 0, st>>>(a.colptr, a.rowidx, a.cval, a.colmap, a.cp, J, a.k, a.s, a.s2,
                                                       a.G, r0, cpc, a.Pt, J > 0);
    else if (unr == 2)
      csr_sketch_light_g_kernel<2><<<g2, THR, 0, st>>>(a.colptr, a.rowidx, a.cval, a.colmap, a.cp, J, a.k, a.s, a.s2,
                                                       a.G, r0, cpc, a.Pt, J > 0);
    else
      csr_sketch_light_g_kernel<4><<<g2, THR, 0, st>>>(a.colptr, a.rowidx, a.cval, a.colmap, a.cp, J, a.k, a.s, a.s2,
                                                       a.G, r0, cpc, a.Pt, J > 0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (a.nd > 0) {
    csr_heavy_finish_kernel<<<grid_cap(a.s * a.nd, 256, (int64_t)nsm * 16), 256, 0, st>>>(
        a.part, a.nsplit, a.s, a.nd, a.ND, a.heavy_cols, a.k, a.At);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  dim3 g3((unsigned)((a.s + 31) / 32), (unsigned)((a.k + 31) / 32));
  csr_slab_finish_kernel<<<g3, dim3(32, 8), 0, st>>>(a.Pt, 1, a.s, a.k, a.colmap, a.At);
  return cudaGetLastError();
}

cudaError_t launch_csr_sketch_slab(const CsrSlabArgs& a, cudaStream_t st) {
  using namespace slab;
  cudaError_t e = cudaFuncSetAttribute(csr_sketch_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (e != cudaSuccess) return e;
  const int64_t cps = (a.nchunks + a.nsplit - 1) / a.nsplit;
  dim3 grid((unsigned)csr_slab_row_blocks(a.s), (unsigned)((a.k + CW - 1) / CW), (unsigned)a.nsplit);
  csr_sketch_slab_kernel<<<grid, THREADS, SMEM, st>>>(a.colptr, a.rowidx, a.cval, a.colmap, a.cp, a.k, a.rows, a.lo,
                                                      a.s, a.seed, cps, a.nchunks, a.part);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2((unsigned)((a.s + 31) / 32), (unsigned)((a.k + 31) / 32));
  csr_slab_finish_kernel<<<g2, dim3(32, 8), 0, st>>>(a.part, a.nsplit, a.s, a.k, a.colmap, a.At);
  return cudaGetLastError();
}

cudaError_t launch_sketch_add_gblock(double* At, int64_t s, int64_t k, int64_t L, double si, uint64_t seed,
                                     cudaStream_t st, int nsm) {
  sketch_add_gblock_kernel<<<grid_cap(((s + 1) / 2) * k, 256, (int64_t)nsm * 16), 256, 0, st>>>(At, s, k, L, si,
                                                                                              seed);
  return cudaGetLastError();
}

cudaError_t launch_csr_rowdot(const CsrRowdotArgs& a, cudaStream_t st) {
  const unsigned nb = (unsigned)a.nblocks;
#define LSRN_ROWDOT(ND_) csr_rowdot_kernel<ND_><<<nb, THR, 0, st>>>(a.rowptr, a.colind, a.val, a.rows, a.t, \
      a.colmap, a.coef, a.sx, a.u, a.acc, a.npart, a.wpart, a.done)
  switch (a.ND) {
    case 0: LSRN_ROWDOT(0); break;
    case 16: LSRN_ROWDOT(16); break;
    case 32: LSRN_ROWDOT(32); break;
    default: LSRN_ROWDOT(64); break;
  }
#undef LSRN_ROWDOT
  return cudaGetLastError();
}

cudaError_t launch_csr_rowdot_hl(const CsrRowdotArgs& a, cudaStream_t st) {
  const unsigned nb = (unsigned)a.nblocks;
  const int ND = a.ND > 0 ? a.ND : 32;
  const bool v8 = ovr().csr_rowdot != 2;   // override csr_rowdot = 2: two rows per step
  if (v8) {
    if (ND > 32)
      csr_rowdot_hl8_kernel<2><<<nb, THR, 0, st>>>(a.D, a.ldd, ND, a.nd, a.heavy_cols, a.lrowptr, a.lcol, a.lval, a.rows,
                                                   a.t, a.coef, a.sx, a.u, a.acc, a.npart, a.wpart, a.done);
    else
      csr_rowdot_hl8_kernel<1><<<nb, THR, 0, st>>>(a.D, a.ldd, ND, a.nd, a.heavy_cols, a.lrowptr, a.lcol, a.lval, a.rows,
                                                   a.t, a.coef, a.sx, a.u, a.acc, a.npart, a.wpart, a.done);
    return cudaGetLastError();
  }
  if (ND > 32)
    csr_rowdot_hl_kernel<2><<<nb, THR, 0, st>>>(a.D, a.ldd, ND, a.nd, a.heavy_cols, a.lrowptr, a.lcol, a.lval, a.rows, a.t,
                                                a.coef, a.sx, a.u, a.acc, a.npart, a.wpart, a.done);
  else
    csr_rowdot_hl_kernel<1><<<nb, THR, 0, st>>>(a.D, a.ldd, ND, a.nd, a.heavy_cols, a.lrowptr, a.lcol, a.lval, a.rows, a.t,
                                                a.coef, a.sx, a.u, a.acc, a.npart, a.wpart, a.done);
  return cudaGetLastError();
}

cudaError_t launch_csr_colgather(const CsrGatherArgs& a, cudaStream_t st) {
  csr_colgather_kernel<<<(unsigned)csr_colgather_blocks(a.k), THR, 0, st>>>(
      a.colptr, a.rowidx, a.cval, a.k, a.sx, a.u, a.colmap, a.wpart, a.ND, a.npart, a.nparts, a.zI, a.t, a.coef, a.sI,
      a.out, a.blockpart,
      a.counter, a.done);
  return cudaGetLastError();
}

}  // namespace lsrn
