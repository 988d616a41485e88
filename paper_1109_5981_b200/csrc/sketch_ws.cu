// K2 v2: warp-specialized dense Gaussian sketch on the fp64 tensor cores.
//
// Same contract as sketch_dense_kernel (kernels.h SketchDenseArgs): the split-K
// partial  P[split][i][c] = sum_{j in split} G[i, lo + j] X[j][c]  of Alg. 1
// step 3 "Ã = G A" / Alg. 2 step 3 "Ã = A G" in the tall form,
// with G generated in-kernel (philox_bm.cuh, C9) and never stored.
//
// Why a second kernel: the first one (every warp loads, generates G and runs
// DMMA, one __syncthreads per k-block) kept the tensor pipe 62 % active on c2
// (profiles/r01_ncu_full_sketch_rowpass.json): after each barrier all warps sat
// in the latency-bound Box-Muller phase together.  Here the roles are split:
//   warpgroups 0-1 (8 producer warps, setmaxnreg 56): lane 0 of warp 0 streams
//     X tiles into a shared-memory ring with 1-D TMA bulk copies; each producer
//     warp generates its own rows of the BM x BK G tile of every k-block into a
//     second ring and arrives on that stage's barrier by itself (no barrier
//     across producer warps);
//   warpgroups 2-3 (8 consumer warps, setmaxnreg 200): DMMA.8x8x4 on
//     (BM/2) x (BN/4) warp tiles, never touching RNG, released stage by stage
//     with mbarriers.
// The RNG shares the FP64 pipe with DMMA: in the ncu source view
// (profiles/r01_ncu_ws_source.txt) the producers' first FP64 instruction of each
// pair waits behind the consumers' queued DMMAs ("math pipe throttle") and the
// consumers wait on the G ring ~21 % of the time, although FP64 ALU work is
// only ~3 % of the pipe.  So each normal must be generated as few times as
// possible per flop: the default tile is 32 x 512 (each normal feeds 512
// columns).  Measured on c2 (profiles/r01_sketch_tile.jsonl, _nsg, _npw):
// 64 x 256 / cluster 2 -> 60.3 ms, 32 x 512 / no cluster -> 58.1 ms (27.5
// TFLOP/s, 75 % of the DMMA peak); with the RNG switched off the same kernel
// reaches 49.3 ms (88 %).  Rejected: 4 producer warps with two interleaved
// pairs per lane (66 ms), 8 producer warps each computing the pairs of two
// k-blocks interleaved (64 / 192 registers: 58.2 vs 57.9 ms), deeper G rings
// (no change), consumers in warpgroups 0-1 instead of 2-3 (no change), BK = 8 (70 ms), X
// streamed by a consumer warp (serialises the consumers), batched RNG phases
// in a non-specialized kernel (sketch_batch.cu, 73.9 ms).
// Clusters (64 x 256 tile only by default): the CTAs of a cluster of CL along N
// (same sketch rows, same k-range, different column tiles) need the SAME G
// tile, so each producer warp of CTA q generates its rows of slice q and
// pushes them to the other CL-1 CTAs with async-proxy shared->shared bulk
// copies (cp.async.bulk.shared::cluster.shared::cta) that complete on the
// destination's `gfull` barrier; consumers release a G stage on every CTA of
// the cluster with plain remote arrives.  (Distributing with st.shared::cluster
// + release/acquire.cluster barriers cost a MEMBAR.GPU / L1 invalidate per
// stage and ran 2x slower.)
//
// Requirements (else the caller uses sketch_dense_kernel): ld even, X 16-byte
// aligned, k even (every bulk row segment is a multiple of 16 bytes).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "philox_bm.cuh"

namespace lsrn {

namespace ws {
constexpr int NPW = 8;                      // producer warps
constexpr int THREADS = NPW * 32 + 256;     // launch 128 regs; producers 56, consumers 200
constexpr int NCONS_WARPS = 8;              // consumers: 2 (M) x 4 (N) warps
// CTA tile BM x BN (BM = 64: warp tile 32 x 64; BM = 32: 16 x 128; 32 accumulator
// fragments per lane either way), k-block BK, X ring NSX deep, G ring NSG deep.
template <int BM_, int BN_, int BK_, int NSX_, int NSG_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, NSX = NSX_, NSG = NSG_;
  static constexpr int A_LD = BN + 8;       // padded smem row (doubles)
  static constexpr int G_LD = BK + 4;
  static constexpr int X_STAGE = BK * A_LD; // doubles
  static constexpr int G_STAGE = BM * G_LD;
  static constexpr int MI = BM / 16;        // 8-row fragments per warp (2 warps along M)
  static constexpr int NJ = BN / 32;        // 8-col fragments per warp (4 warps along N)
  static constexpr size_t SMEM = sizeof(double) * (size_t)(NSX * X_STAGE + NSG * G_STAGE) + 128;
  static_assert(MI * NJ == 32, "32 accumulator fragments per lane");
  static_assert(BK % 4 == 0, "k-block is a multiple of the DMMA k = 4");
};
}  // namespace ws

namespace {
LSRN_DEV unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
LSRN_DEV unsigned map_rank(const void* p, unsigned rank) {     // shared::cluster address in CTA `rank`
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
// remote arrive (default .release.cta semantics: only orders this thread's prior
// shared-memory reads, which is all a consumer release needs)
LSRN_DEV void mbar_arrive_remote(unsigned addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
// async-proxy copy of `bytes` from this CTA's shared memory into CTA-rank shared
// memory (dst, bar: shared::cluster addresses), completing tx on the remote barrier
LSRN_DEV void bulk_s2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar)
      : "memory");
}
LSRN_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
LSRN_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
LSRN_DEV void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
LSRN_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
}  // namespace

template <class C, int CL>
__global__ void __launch_bounds__(ws::THREADS, 1)
sketch_ws_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k, int64_t lo, int64_t s,
                 uint64_t seed, int64_t rows_per_split, double* __restrict__ out, int64_t out_split_stride,
                 int accumulate, int x_evict_last, const double* __restrict__ Gmem, int64_t g_nkb) {
  using namespace ws;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, NSX = C::NSX, NSG = C::NSG;
  constexpr int A_LD = C::A_LD, G_LD = C::G_LD, X_STAGE = C::X_STAGE, G_STAGE = C::G_STAGE;
  constexpr int MI = C::MI, NJ = C::NJ;
  extern __shared__ __align__(128) double smem[];
  double* Xs = smem;                                   // [NSX][BK][A_LD]
  double* Gs = smem + NSX * X_STAGE;                   // [NSG][BM][G_LD]
  __shared__ uint64_t xfull[NSX], xempty[NSX], gfull[NSG], gempty[NSG];
  __shared__ double bmT[bm::TAB_SIZE];                 // Box-Muller tables (producers)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Without clusters the grid is M-tile-fastest: the CTAs resident at one time then
  // share one X column stripe and read it from L2.  (N-fastest, the cluster layout,
  // re-read X from DRAM once per M-tile: 49 TB per c5 sketch, ncu r02.)
  const int64_t n0 = (int64_t)(CL == 1 ? blockIdx.y : blockIdx.x) * BN;
  const int64_t m0 = (int64_t)(CL == 1 ? blockIdx.x : blockIdx.y) * BM;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (r_end > r_begin) ? (int)((r_end - r_begin + BK - 1) / BK) : 0;

  const unsigned qrank = (CL > 1) ? cluster_rank() : 0u;
  constexpr int SLICE_ROWS = BM / CL;                  // G rows generated by this CTA
  if (tid == 0) {
    for (int i = 0; i < NSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], NCONS_WARPS);
    }
    for (int i = 0; i < NSG; ++i) {
      // one per local producer warp (+ tx of remote rows); stored G: the one bulk copy
      mbar_init(&gfull[i], Gmem != nullptr ? 1 : NPW);
      mbar_init(&gempty[i], NCONS_WARPS * CL);          // one per consumer warp of each CTA of the cluster
    }
    mbar_fence_init();
  }
  if (CL > 1)
    cluster_sync_all();                                 // every CTA's barriers exist before remote traffic
  else
    __syncthreads();
  static_assert(CL >= 1 && BM % CL == 0, "cluster size must divide BM");

  if (warp < NPW) {
    // ------------------------------------------------------------ producers
    // Each producer warp owns ROWS_W consecutive rows of this CTA's G slice and runs
    // its own flow (no barrier across producer warps): wait for the stage to be
    // free, generate its PPT pairs per lane (independent chains, interleaved),
    // store, push its rows to the other CTAs of the cluster, arrive on gfull.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    if (Gmem != nullptr) {
      // stored G (sketch_gen_g_kernel wrote this chunk's tiles, padded like the G
      // stage): lane 0 of warp 0 streams the X rows and the G tile of every k-block;
      // the other producer warps have nothing to do
      if (CL == 1 && warp == 0 && lane == 0) {
        const int64_t ncols = min((int64_t)BN, k - n0);
        const unsigned seg_bytes = (unsigned)(ncols * 8);
        const uint64_t xpol = x_evict_last ? l2_policy_evict_last() : 0ull;
        const double* gsrc = Gmem + ((m0 / BM) * g_nkb + r_begin / BK) * (int64_t)G_STAGE;
        for (int kb = 0; kb < nk; ++kb) {
          const int sx = kb % NSX, sg = kb % NSG;
          const unsigned px = (unsigned)(((kb / NSX) & 1) ^ 1), pg = (unsigned)(((kb / NSG) & 1) ^ 1);
          const int64_t rbase = r_begin + (int64_t)kb * BK;
          const int nrow = (int)min((int64_t)BK, r_end - rbase);
          if (kb >= NSX) mbar_wait(&xempty[sx], px);
          double* dst = Xs + sx * X_STAGE;
          if (nrow < BK)          // ragged K tail: zero the missing rows (the G tile is zero there too)
            for (int e = 0; e < (BK - nrow) * A_LD; ++e) dst[nrow * A_LD + e] = 0.0;
          mbar_arrive_expect_tx(&xfull[sx], seg_bytes * (unsigned)nrow);
          for (int rr = 0; rr < nrow; ++rr) {
            if (x_evict_last)
              bulk_g2s_hint(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx], xpol);
            else
              bulk_g2s(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx]);
          }
          if (kb >= NSG) mbar_wait(&gempty[sg], pg);
          mbar_arrive_expect_tx(&gfull[sg], (unsigned)(G_STAGE * sizeof(double)));
          bulk_g2s(Gs + sg * G_STAGE, gsrc + (int64_t)kb * G_STAGE, (unsigned)(G_STAGE * sizeof(double)), &gfull[sg]);
        }
      }
      return;
    }
    constexpr int ROWS_W = SLICE_ROWS / NPW;            // G rows per producer warp (even)
    static_assert(ROWS_W >= 2 && ROWS_W % 2 == 0, "each producer warp needs whole row pairs");
    constexpr int PAIRS_W = (ROWS_W / 2) * BK;
    constexpr int PPT = (PAIRS_W + 31) / 32;
    constexpr unsigned WBYTES = (unsigned)(ROWS_W * G_LD * sizeof(double));
    const uint2 key = philox_key(seed);
    for (int i = tid; i < bm::TAB_SIZE; i += NPW * 32) bmT[i] = bm::kTable[i];
    named_bar(1, NPW * 32);
    const int row0 = (int)qrank * SLICE_ROWS + warp * ROWS_W;   // first G row of this warp in the tile
    const int64_t ncols = min((int64_t)BN, k - n0);      // even (k even, n0 multiple of BN)
    const unsigned seg_bytes = (unsigned)(ncols * 8);
    const uint64_t xpol = x_evict_last ? l2_policy_evict_last() : 0ull;
    for (int kb = 0; kb < nk; ++kb) {
      const int sx = kb % NSX, sg = kb % NSG;
      const unsigned px = (unsigned)(((kb / NSX) & 1) ^ 1), pg = (unsigned)(((kb / NSG) & 1) ^ 1);
      const int64_t rbase = r_begin + (int64_t)kb * BK;
      const int nrow = (int)min((int64_t)BK, r_end - rbase);
      // X tile: rows rbase .. rbase + nrow of this N-tile (lane 0 of warp 0)
      if (warp == 0) {
        if (kb >= NSX) mbar_wait(&xempty[sx], px);
        double* dst = Xs + sx * X_STAGE;
        if (nrow < BK) {          // ragged K tail: zero the missing rows (0 x stale would risk NaN)
          for (int e = lane; e < (BK - nrow) * A_LD; e += 32) dst[nrow * A_LD + e] = 0.0;
          __syncwarp();
        }
        if (lane == 0) {
          mbar_arrive_expect_tx(&xfull[sx], seg_bytes * (unsigned)nrow);
          if (x_evict_last) {
            for (int rr = 0; rr < nrow; ++rr)
              bulk_g2s_hint(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx], xpol);
          } else {
            for (int rr = 0; rr < nrow; ++rr) bulk_g2s(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx]);
          }
        }
      }
      // G stage sg must be free on every CTA of the cluster, and (CL > 1) the bulk
      // copies that last read this warp's rows of it must have finished reading
      if (kb >= NSG) mbar_wait(&gempty[sg], pg);
      if (CL > 1) {
        if (lane == 0) bulk_wait_read<NSG - 1>();
        __syncwarp();
      }
      double* gdst = Gs + sg * G_STAGE;
      const int64_t jbase = lo + rbase;
      double z[PPT][2];
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int p = lane + 32 * t;
        const int qp = row0 / 2 + p / BK, kk = p % BK;
        z[t][0] = z[t][1] = 0.0;
        if ((PAIRS_W % 32 == 0 || p < PAIRS_W) && kk < nrow)
          gaussian_pair(key, (uint64_t)(m0 / 2 + qp), (uint64_t)(jbase + kk), bmT, z[t][0], z[t][1]);
      }
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int p = lane + 32 * t;
        if (PAIRS_W % 32 == 0 || p < PAIRS_W) {
          const int qp = row0 / 2 + p / BK, kk = p % BK;
          gdst[(2 * qp) * G_LD + kk] = z[t][0];
          gdst[(2 * qp + 1) * G_LD + kk] = z[t][1];
        }
      }
      if (CL > 1) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic -> async proxy
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&gfull[sg], WBYTES * (unsigned)(CL - 1));   // + the matching warps' rows
        if (CL > 1) {
          const double* src = gdst + (int64_t)row0 * G_LD;
#pragma unroll
          for (unsigned r = 1; r < (unsigned)CL; ++r) {
            const unsigned dr = (qrank + r) % (unsigned)CL;
            bulk_s2s(map_rank(src, dr), src, WBYTES, map_rank(&gfull[sg], dr));
          }
          bulk_commit();
        }
      }
    }
    if (CL > 1) {
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      cluster_sync_all();                               // no CTA leaves while others may still signal it
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n");
  const int cw = warp - NPW;                             // 0..7
  const int wm = cw >> 2, wn = cw & 3;                   // 2 x 4 warps
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kb = 0; kb < nk; ++kb) {
    const int sx = kb % NSX, sg = kb % NSG;
    mbar_wait(&xfull[sx], (unsigned)((kb / NSX) & 1));
    mbar_wait(&gfull[sg], (unsigned)((kb / NSG) & 1));
    const double* as = Xs + sx * X_STAGE;
    const double* gs = Gs + sg * G_STAGE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = gs[(wm * (BM / 2) + i * 8 + (lane >> 2)) * G_LD + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = as[(ks * 4 + (lane & 3)) * A_LD + wn * (BN / 4) + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&xempty[sx]);
      if (CL == 1) {
        mbar_arrive(&gempty[sg]);
      } else {
#pragma unroll
        for (unsigned r = 0; r < (unsigned)CL; ++r) mbar_arrive_remote(map_rank(&gempty[sg], r));
      }
    }
  }

  double* o = out + (int64_t)blockIdx.z * out_split_stride;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t gi = m0 + wm * (BM / 2) + i * 8 + (lane >> 2);
    if (gi >= s) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t gc = n0 + wn * (BN / 4) + j * 8 + 2 * (lane & 3);
      if (gc + 1 < k) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (accumulate) {
          const double2 w = *reinterpret_cast<const double2*>(o + gi * k + gc);
          v.x = w.x + v.x;
          v.y = w.y + v.y;
        }
        *reinterpret_cast<double2*>(o + gi * k + gc) = v;
      } else if (gc < k) {
        o[gi * k + gc] = accumulate ? o[gi * k + gc] + acc[i][j][0] : acc[i][j][0];
      }
    }
  }
  if (CL > 1) cluster_sync_all();
}

// ---------------------------------------------------------------------------
// K2 v3 (sketch_cg_kernel): the consumers generate G themselves.
// In sketch_ws_kernel the producer warps' FP64 instructions queue behind the
// consumers' DMMAs on the one FP64 pipe per SM sub-partition; the producers only
// need ~4 % of the pipe, but every dependent step of their Box-Muller chain waits
// for it, so they fall behind and the consumers wait on the G ring (tensor pipe
// 78.7 % active, FP64 ALU 3.6 %, profiles/r01_ncu_full_final.json).  Here there
// are no RNG-only warps: each of the 8 DMMA warps generates its 1/8 of the G tile
// of k-block kb + 1 (one Box-Muller pair per lane) in the same instruction stream
// as its DMMAs for k-block kb, so a warp waiting on the FP64 pipe for its RNG
// leaves the pipe to the other DMMA warp of its sub-partition instead of starving
// both.  A ninth warp streams the X tiles with 1-D TMA bulk copies (3-stage ring,
// mbarriers); G is double-buffered and the 8 DMMA warps meet at one named barrier
// per k-block (G[kb+1] written, G[kb] read).  CTAs are rasterised M-tile-fastest,
// so the CTAs resident at one time share their X tiles through L2 (c5: ~85 waves
// each re-reading X from DRAM about once, against ~84x with N-fastest order).
namespace cg {
constexpr int BM = 32, BN = 512, BK = 16, NSX = 3;
constexpr int A_LD = BN + 8;                 // padded X row (doubles): conflict-free B fragments
constexpr int G_LD = BK + 4;
constexpr int X_STAGE = BK * A_LD;
constexpr int G_STAGE = BM * G_LD;
constexpr int NCW = 8;                       // DMMA warps: 2 (M) x 4 (N), warp tile 16 x 128
constexpr int THREADS = NCW * 32 + 32;       // + one TMA warp
constexpr int MI = BM / 16, NJ = BN / 32;    // 2 x 16 fragments of 8 x 8
constexpr size_t SMEM = sizeof(double) * (size_t)(NSX * X_STAGE + 2 * G_STAGE) + 128;
}  // namespace cg

__global__ void __launch_bounds__(cg::THREADS, 1)
sketch_cg_kernel(const double* __restrict__ X, int64_t ld, int64_t rows, int64_t k, int64_t lo, int64_t s,
                 uint64_t seed, int64_t rows_per_split, double* __restrict__ out, int64_t out_split_stride,
                 int accumulate) {
  using namespace cg;
  extern __shared__ __align__(128) double smem[];
  double* Xs = smem;                                   // [NSX][BK][A_LD]
  double* Gs = smem + NSX * X_STAGE;                   // [2][BM][G_LD]
  __shared__ uint64_t xfull[NSX], xempty[NSX];
  __shared__ double bmT[bm::TAB_SIZE];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * BM;         // M-tile fastest (shared X tiles in L2)
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int nk = (r_end > r_begin) ? (int)((r_end - r_begin + BK - 1) / BK) : 0;
  if (tid == 0) {
    for (int i = 0; i < NSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], NCW);
    }
    mbar_fence_init();
  }
  for (int i = tid; i < bm::TAB_SIZE; i += THREADS) bmT[i] = bm::kTable[i];
  __syncthreads();

  if (warp == NCW) {
    // ---------------------------------------------------------------- X loader
    // (no setmaxnreg: it is warpgroup-wide and this warp is alone in its warpgroup;
    // 288 threads x 168 registers fit the register file as launched)
    const int64_t ncols = min((int64_t)BN, k - n0);
    const unsigned seg_bytes = (unsigned)(ncols * 8);
    for (int kb = 0; kb < nk; ++kb) {
      const int sx = kb % NSX;
      if (kb >= NSX) mbar_wait(&xempty[sx], (unsigned)(((kb / NSX) & 1) ^ 1));
      const int64_t rbase = r_begin + (int64_t)kb * BK;
      const int nrow = (int)min((int64_t)BK, r_end - rbase);
      double* dst = Xs + sx * X_STAGE;
      if (nrow < BK) {            // ragged K tail: zero the missing rows (0 x stale could be NaN)
        for (int e = lane; e < (BK - nrow) * A_LD; e += 32) dst[nrow * A_LD + e] = 0.0;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
      }
      if (lane == 0) {
        mbar_arrive_expect_tx(&xfull[sx], seg_bytes * (unsigned)nrow);
        for (int rr = 0; rr < nrow; ++rr) bulk_g2s(dst + rr * A_LD, X + (rbase + rr) * ld + n0, seg_bytes, &xfull[sx]);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ DMMA warps
  const uint2 key = philox_key(seed);
  const int wm = warp >> 2, wn = warp & 3;
  // this lane's Box-Muller pair of every G tile: pair (row pair gq, column gk) of
  // the BM x BK tile; warp w owns row pairs 2w, 2w+1 (32 pairs: 2 row pairs x 16 columns)
  const int gq = 2 * warp + (lane >> 4), gk = lane & 15;
  auto gen = [&](int kb, double* gdst) {
    const int64_t rbase = r_begin + (int64_t)kb * BK;
    double z0 = 0.0, z1 = 0.0;
    if (rbase + gk < r_end) gaussian_pair(key, (uint64_t)(m0 / 2 + gq), (uint64_t)(lo + rbase + gk), bmT, z0, z1);
    gdst[(2 * gq) * G_LD + gk] = z0;
    gdst[(2 * gq + 1) * G_LD + gk] = z1;
  };
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nk > 0) gen(0, Gs);
  asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory");
  for (int kb = 0; kb < nk; ++kb) {
    const int sx = kb % NSX;
    const double* as = Xs + sx * X_STAGE;
    const double* gs = Gs + (kb & 1) * G_STAGE;
    mbar_wait(&xfull[sx], (unsigned)((kb / NSX) & 1));
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = gs[(wm * (BM / 2) + i * 8 + (lane >> 2)) * G_LD + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = as[(ks * 4 + (lane & 3)) * A_LD + wn * (BN / 4) + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma884(acc[i][j], a[i], b[j]);
      // in the DMMA stream, staggered: the two DMMA warps of a sub-partition (warps w and
      // w + 4) run their Box-Muller chains at different k-steps, so one keeps the pipe busy
      if (ks == ((warp >> 2) & 1) * 2 && kb + 1 < nk) gen(kb + 1, Gs + ((kb + 1) & 1) * G_STAGE);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&xempty[sx]);
    asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory");   // G[kb+1] written, G[kb] read by all
  }

  double* o = out + (int64_t)blockIdx.z * out_split_stride;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t gi = m0 + wm * (BM / 2) + i * 8 + (lane >> 2);
    if (gi >= s) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t gc = n0 + wn * (BN / 4) + j * 8 + 2 * (lane & 3);
      if (gc + 1 < k) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (accumulate) {
          const double2 w = *reinterpret_cast<const double2*>(o + gi * k + gc);
          v.x = w.x + v.x;
          v.y = w.y + v.y;
        }
        *reinterpret_cast<double2*>(o + gi * k + gc) = v;
      } else if (gc < k) {
        o[gi * k + gc] = accumulate ? o[gi * k + gc] + acc[i][j][0] : acc[i][j][0];
      }
    }
  }
}

static cudaError_t launch_cg(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace cg;
  dim3 grid((unsigned)((a.s + BM - 1) / BM), (unsigned)((a.k + BN - 1) / BN), (unsigned)a.nsplit);
  cudaError_t e = cudaFuncSetAttribute(sketch_cg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (e != cudaSuccess) return e;
  sketch_cg_kernel<<<grid, THREADS, SMEM, st>>>(a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed, a.rows_per_split, a.out,
                                                a.out_split_stride, a.accumulate);
  return cudaGetLastError();
}

bool sketch_ws_supported(const SketchDenseArgs& a) {
  return (a.ld % 2 == 0) && (a.k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
}

template <class C, int CL>
static cudaError_t launch_ws_t(const SketchDenseArgs& a, cudaStream_t st) {
  using namespace ws;
  const unsigned ntn = (unsigned)((a.k + C::BN - 1) / C::BN), ntm = (unsigned)((a.s + C::BM - 1) / C::BM);
  dim3 grid(CL == 1 ? ntm : ntn, CL == 1 ? ntn : ntm, (unsigned)a.nsplit);   // see the kernel: raster order
  cudaError_t e = cudaFuncSetAttribute(sketch_ws_kernel<C, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)C::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sketch_ws_kernel<C, CL>, a.X, a.ld, a.rows, a.k, a.lo, a.s, a.seed,
                            a.rows_per_split, a.out, a.out_split_stride, a.accumulate,
                            ovr().sketch_x_l2 == 1 ? 1 : 0, CL == 1 ? a.G : nullptr,
                            (a.rows + C::BK - 1) / C::BK);
}

// Tile shape (override sketch_tile).  Measured on c2 (1e5 x 2000,
// profiles/r01_sketch_tile.jsonl), ms: 64 x 256 (BK 16, 4 + 4 stages) CL 1/2 ->
// 65.7 / 60.3; 32 x 512 (BK 16, 3 X stages) CL 1/2 -> 58.1 / 61.1; 32 x 512 with
// BK 8 (5 X stages) CL 1/2 -> 70.2 / 74.9; 16 x 1024 (BK 8, 3 X stages) -> 69.6
// (51.6 without RNG: the BK = 8 k-block overheads outweigh the halved RNG).  The 32 x 512 tile needs half the G
// per flop of the 64 x 256 one (each normal feeds 512 columns) without the
// cluster exchange, so it is the default: tile 1, CL 1.
using Tile0 = ws::Cfg<64, 256, 16, 4, 4>;
using Tile1 = ws::Cfg<32, 512, 16, 3, 4>;

int sketch_ws_tile() { return ovr().sketch_tile == 0 ? 0 : 1; }

void sketch_ws_tile_dims(int64_t* bm, int64_t* bn, int64_t* bk) {
  if (sketch_ws_tile() == 0) {
    *bm = Tile0::BM; *bn = Tile0::BN; *bk = Tile0::BK;
  } else {
    *bm = Tile1::BM; *bn = Tile1::BN; *bk = Tile1::BK;
  }
}

// Cluster size along N: the largest of {max_cl, ..., 2} dividing the N-tile count.
// The sketch_maxcl override caps it; default 2 for the 64 x 256 tile
// (CL = 1/2/4/8 -> 82.6/69.3/72.3/83.0 ms on c2 in the first measurement,
// profiles/r01_sketch_tune.jsonl: whole clusters must fit in a GPC, with CL = 8
// only 76 % of the SM-cycles were active) and 1 for the 32 x 512 tile.
template <class C>
static int cluster_for(int64_t k) {
  const int64_t nt = (k + C::BN - 1) / C::BN;
  int max_cl = C::BM == 64 ? 2 : 1;
  if (ovr().sketch_maxcl >= 1) max_cl = ovr().sketch_maxcl;
  for (int cl : {4, 2})
    if (cl <= max_cl && nt % cl == 0) return cl;
  return 1;
}

template <class C>
static cudaError_t launch_ws_tile(const SketchDenseArgs& a, cudaStream_t st) {
  switch (cluster_for<C>(a.k)) {
    case 4: if constexpr (C::BM / 4 >= 2 * ws::NPW) return launch_ws_t<C, 4>(a, st); [[fallthrough]];
    case 2: if constexpr (C::BM / 2 >= 2 * ws::NPW) return launch_ws_t<C, 2>(a, st); [[fallthrough]];
    default: return launch_ws_t<C, 1>(a, st);
  }
}

// ---------------------------------------------------------------------------
// Stored G (the default, LSRN_OPT_SKETCH_G): the G tiles of one launch's rows are
// generated ONCE by sketch_gen_g_kernel into a bounded workspace buffer, laid out
// tile by tile exactly as the producer ring stage (BM rows x G_LD, padded), and
// sketch_ws_kernel streams them with one 5 KB bulk copy per k-block instead of
// regenerating them in every N-tile CTA.  In-register generation (never stored,
// SURVEY a1) costs k / BN regenerations of each normal (c5: 20) and its FP64
// Box-Muller steps share the pipe with the DMMAs; storing costs s * rows * 10 B of
// HBM writes and one tile read per CTA k-block (from L2 or DRAM).  Measurements:
// DESIGN.md §6 K2.
__global__ void __launch_bounds__(256)
sketch_gen_g_kernel(double* __restrict__ G, int64_t ntm, int64_t nkb, int64_t rows, int64_t jbase, uint64_t seed) {
  using C = Tile1;
  __shared__ double bmT[bm::TAB_SIZE];
  for (int i = threadIdx.x; i < bm::TAB_SIZE; i += blockDim.x) bmT[i] = bm::kTable[i];
  __syncthreads();
  const uint2 key = philox_key(seed);
  constexpr int PAIRS = (C::BM / 2) * C::BK;       // pairs per tile
  // tiles over CTAs, a tile's pairs over threads: the 64-bit division by nkb happens
  // once per tile, not once per pair
  for (int64_t tile = blockIdx.x; tile < ntm * nkb; tile += gridDim.x) {
    const int64_t mt = tile / nkb, kb = tile % nkb;
    double* t = G + tile * C::G_STAGE;
    for (int w = threadIdx.x; w < PAIRS; w += blockDim.x) {
      const int qp = w / C::BK, kk = w % C::BK;
      const int64_t r = kb * C::BK + kk;
      double z0 = 0.0, z1 = 0.0;
      if (r < rows) gaussian_pair(key, (uint64_t)(mt * (C::BM / 2) + qp), (uint64_t)(jbase + r), bmT, z0, z1);
      t[(2 * qp) * C::G_LD + kk] = z0;
      t[(2 * qp + 1) * C::G_LD + kk] = z1;
    }
  }
}

int64_t sketch_g_row_bytes(int64_t s) {
  return ((s + Tile1::BM - 1) / Tile1::BM) * (int64_t)Tile1::G_STAGE * 8 / Tile1::BK;
}
int64_t sketch_g_block_rows() { return Tile1::BK; }
size_t sketch_g_bytes(int64_t s, int64_t rows) {
  const int64_t ntm = (s + Tile1::BM - 1) / Tile1::BM, nkb = (rows + Tile1::BK - 1) / Tile1::BK;
  return (size_t)ntm * (size_t)nkb * Tile1::G_STAGE * sizeof(double);
}

static cudaError_t launch_gen_g(const SketchDenseArgs& a, cudaStream_t st) {
  const int64_t ntm = (a.s + Tile1::BM - 1) / Tile1::BM, nkb = (a.rows + Tile1::BK - 1) / Tile1::BK;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntm * nkb, 148 * 16));
  sketch_gen_g_kernel<<<blocks, 256, 0, st>>>(a.G, ntm, nkb, a.rows, a.lo, a.seed);
  return cudaGetLastError();
}

cudaError_t launch_sketch_ws(const SketchDenseArgs& a, cudaStream_t st) {
  if (a.G != nullptr) {       // stored G: 32 x 512 tile, no cluster
    if (a.nsplit > 1 && a.rows_per_split % Tile1::BK != 0) return cudaErrorInvalidValue;
    cudaError_t e = launch_gen_g(a, st);
    if (e != cudaSuccess) return e;
    return launch_ws_t<Tile1, 1>(a, st);
  }
  if (ovr().sketch_kernel == 2) return launch_cg(a, st);
  return sketch_ws_tile() == 0 ? launch_ws_tile<Tile0>(a, st) : launch_ws_tile<Tile1>(a, st);
}

}  // namespace lsrn
