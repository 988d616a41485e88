// Host-side launch interface of the LSRN kernels (internal; not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace lsrn {

// ---- kernel-plan overrides (lsrn_ctx_set_option; testing / tuning aids)
// Each field < 0 (or 0 where noted) leaves the planner's shape-based choice.
// Every value selects among kernels that compute the same result; none changes
// the arithmetic.  The context's overrides are installed for the duration of an
// API call (OverrideScope) and read by the host-side planners through ovr().
struct Overrides {
  int sketch_kernel = -1;     // 0 warp-specialized DMMA (sketch_ws.cu), 1 non-specialized (sketch_dense.cu),
                              // 2 DMMA warps generating G themselves (sketch_cg_kernel)
  int sketch_tile = -1;       // 0: 64 x 256 tile, 1: 32 x 512 tile
  int sketch_maxcl = -1;      // cap on the G-sharing cluster size along N
  int sketch_nsplit = -1;     // split-K factor (>= 1)
  int sketch_x_l2 = -1;       // 1: X tiles loaded with an L2 evict_last policy
  int sketch_chunks = -1;     // device-resident A: row chunks launched one after the other (0/1 = one launch)
  int sketch_g = -1;          // dense sketch G: -1 stored per launch (8 GB budget), 0 in-register (never
                              // stored), N > 0 stored with an N-MB budget
  int rowpass_keep = -1;      // 0/1: re-read / register-kept row tile
  int rowpass_occ = -1;       // 1/2 CTAs per SM
  int rowpass_wide1 = -1;     // 0 disables the single 512-thread CTA plan for 8192 < k <= 10240
  int rowpass_wide2 = -1;     // 0 disables the 2 x 512-thread cluster plan for 16384 < k <= 20480
  int rowpass_asyncx = -1;    // 0: cluster barrier per tile instead of the st.async exchange
  int rowpass_nt = -1;        // 256 / 512 threads for cluster plans
  int rowpass_tr = -1;        // wide rows: rows per tile (1 or 2)
  int rowpass_budget_kb = -1; // shared-memory stage budget
  int rowpass_wide_slice = -1;// wide rows: max columns per CTA slice
  int rowpass_pf = -1;        // L2 prefetch distance (tiles) of the bulk row pass, 0 = off
  int csr_rowdot = -1;        // 0 heavy-dense + light-CSR 8 rows/step, 1 warp per row (full CSR), 2 hl 2 rows/step,
                              // 3 the two-kernel form (row dots + CSC gather) also for k <= 2048
  int csr_sketch = -1;        // 0 column-stationary light sketch, 1 generate-once slab sketch, 2 stored G
  int csr_heavy_fma = -1;     // stored-G heavy block: 1 = FP64-FMA kernel instead of DMMA
  int csr_all = -1;           // k <= 2048 single-pass kernel: 0 one pair of rows in flight, 6 / 10 pipelined
  int csr_light = -1;         // stored-G light sketch: 10 * (columns per CTA) + (gathers in flight: 2, 4, 8)
};
const Overrides& ovr();
struct OverrideScope {
  explicit OverrideScope(const Overrides* o);
  ~OverrideScope();
  const Overrides* prev;
};

// ---- K2 dense sketch (sketch_dense.cu)
struct SketchDenseArgs {
  const double* X;   // shard rows (row-major, leading dim ld)
  int64_t ld, rows, k, lo, s;
  uint64_t seed;
  int64_t rows_per_split;
  int nsplit;
  double* out;       // [nsplit][s][k]
  int64_t out_split_stride;
  int accumulate = 0;   // 1: out += partial (stream-ordered chunks of A, host-IO streaming)
  double* G = nullptr;  // stored-G mode: buffer of sketch_g_bytes(s, rows) the launch fills with
                        // this launch's G tiles first (rows_per_split a multiple of sketch_g_block_rows())
};
size_t sketch_g_bytes(int64_t s, int64_t rows);
int64_t sketch_g_row_bytes(int64_t s);
int64_t sketch_g_block_rows();
size_t sketch_dense_smem();
void sketch_tile_counts(int64_t s, int64_t k, int64_t* mtiles, int64_t* ntiles, int64_t* bk);
cudaError_t launch_sketch_dense(const SketchDenseArgs& a, cudaStream_t st);   // picks v2 when supported
bool sketch_ws_supported(const SketchDenseArgs& a);
cudaError_t launch_sketch_ws(const SketchDenseArgs& a, cudaStream_t st);
void sketch_ws_tile_dims(int64_t* bm, int64_t* bn, int64_t* bk);
cudaError_t launch_sketch_finish(const double* part, int nsplit, int64_t split_stride, int64_t s, int64_t k,
                                 double sx, double si, int64_t L, uint64_t seed, double* out, cudaStream_t st,
                                 int nsm);
cudaError_t launch_debug_box_muller(const uint32_t* words, int64_t count, int mode, double* out, cudaStream_t st);
cudaError_t launch_debug_gaussian(uint64_t seed, const int64_t* rows, const int64_t* cols, int64_t count,
                                  double* out, cudaStream_t st);

// ---- K5/K6 fused row pass (rowpass.cu)
// For rows j of the row-major R x C matrix Y (scaled by sx):
//   z_j <- c1 z_j + c2 sx (Y_j . t);  acc_j += ca z_j (if acc);  norm2 += z_j^2;  w += sx Y_j z_j
// coef -> {c1, c2, ca}.  Writes per-cluster partials wpart[g][C] and npart[g].
struct RowPassArgs {
  const double* Y;
  int64_t ld, R, C;
  double sx;
  double* z;
  const double* t;
  const double* coef;
  double* acc;
  const int* done;       // nullable: skip the pass when *done != 0
  double* wpart;         // [nparts][C]
  double* npart;         // [nparts]
};
struct RowPassPlan {
  int vpt, cl, tr, nclusters, vec;  // vec: 2 = 16-byte loads
  int64_t rows_per_cluster;
  int bulk = 0;                     // 1: rowpass_bulk_kernel (TMA bulk-copy ring)
  int64_t cq = 0;                   // bulk: columns per CTA slice
  int nst = 0;                      // bulk: pipeline stages
  int keep = 0;                     // bulk: row tile kept in registers between the two phases
  int occ = 1;                      // bulk: CTAs per SM
  int async_x = 0;                  // bulk, cl > 1: pipelined st.async partial-dot exchange
  int nt = 256;                     // bulk: threads per CTA (wide rows: 256, or 512 as a tuning aid)
  int pf = 0;                       // bulk: L2 prefetch distance in tiles beyond the ring (0 = off)
};
// allow_bulk = false forces the register-load kernel (tests compare both)
RowPassPlan plan_rowpass(int64_t R, int64_t C, int64_t ld, const double* Y, int nsm, bool allow_bulk = true);
cudaError_t launch_rowpass(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st);
bool plan_rowpass_bulk(int64_t R, int64_t C, int64_t ld, const double* Y, int nsm, RowPassPlan* p);
cudaError_t launch_rowpass_bulk(const RowPassArgs& a, const RowPassPlan& p, cudaStream_t st);

// Column reduce of the row-pass partials (+ optional Tikhonov identity block):
//   w_c = sum_g wpart[g][c];  if zI: zI_c <- c1 zI_c + c2 sI t_c,  w_c += sI zI_c
//   out[c] = w_c (c < C);  out[C] = sum_g npart[g] + sum_c zI_c^2
struct ColReduceArgs {
  const double* wpart;
  const double* npart;
  int nparts;
  int64_t C;
  double* zI;            // nullable
  const double* t;
  const double* coef;
  double sI;
  double* out;           // C + 1
  double* blockpart;     // scratch, >= colreduce_blocks(C)
  unsigned* counter;     // zero-initialised, self-resetting
  const int* done;
};
int colreduce_blocks(int64_t C);
cudaError_t launch_colreduce(const ColReduceArgs& a, cudaStream_t st);

// ---- compensated row pass (compensated.cu; precision = 1, C18(ii))
struct ExtRowPassArgs {
  const double* Y;
  int64_t ld, R, C;
  double sx;
  double* z;
  const double* t_hi;
  const double* t_lo;
  const double* coef;
  double* acc;
  const int* done;
  double* part_s;        // [nblocks][C]
  double* part_c;        // [nblocks][C]
  double* npart;         // [nblocks]
};
struct ExtColReduceArgs {
  const double* part_s;
  const double* part_c;
  const double* npart;
  int nparts;
  int64_t C;
  double* zI;            // nullable
  const double* t_hi;
  const double* t_lo;
  const double* coef;
  double sI;
  double* out_hi;        // C + 1 (out_hi[C] = ||z||^2)
  double* out_lo;        // C + 1
  const int* done;
};
int ext_rowpass_blocks(int64_t R, int nsm);
cudaError_t launch_ext_rowpass(const ExtRowPassArgs& a, int nblocks, cudaStream_t st);
cudaError_t launch_ext_colreduce(const ExtColReduceArgs& a, cudaStream_t st);

// ---- Krylov scalar / vector steps (krylov.cu)
struct LsqrState {
  double alpha, beta, su, sv, rhobar, phibar, anorm2, bnorm;
  double phi_rho, theta_rho, rnorm, arnorm, tol;
  double cU[3], cV[3];          // pass coefficients {c1, c2, ca}
  int iters, done, converged, adaptive, stop_after, pad_;
};
cudaError_t launch_lsqr_init_state(LsqrState* st_dev, double tol, int adaptive, cudaStream_t st);
// phase 0: after the initial U pass (beta_1); 1: after a U pass inside the loop
cudaError_t launch_lsqr_after_u(LsqrState* s, const double* comm, int64_t C, int phase, cudaStream_t st);
// phase 0: after the initial V pass (alpha_1) -> w_y = sv v; 1: Givens step + y / w_y update.
// ypart: scratch of update-kernel block partials (>= lsqr_update_blocks(n)).
int lsqr_update_blocks(int64_t n);
cudaError_t launch_lsqr_after_v(LsqrState* s, const double* comm, int64_t C, int phase, double* y, double* wy,
                                const double* vstore, int64_t n, double* ypart, unsigned* counter,
                                cudaStream_t st);

// ---- K4 CSR sketch + CSR long pass (csr.cu)
struct CsrBuildArgs {
  const int64_t* rowptr;   // rows + 1 (rowptr[0] may be non-zero)
  const int32_t* colind;
  const double* val;
  int64_t rows, k;
  int* cntc;               // [nchunks][k]
  int64_t* offs;           // [nchunks][k]
  int64_t* total;          // [k]
  const int* colmap;       // [k]: heavy index h >= 0, or -1 (light)
  int64_t* colptr;         // [k + 1] (light columns only)
  int32_t* rowidx;         // [nnz_light]
  double* cval;            // [nnz_light]
  double* D;               // [rows][ld_d] heavy block (nullable when no heavy column)
  int64_t ld_d;
  int* bad;                // validation flags (zeroed by launch_csr_build): 1 column range, 2 order, 4 rowptr
  // light-column CSR (row order, heavy entries removed) for the iteration pass
  int64_t* lrowptr;        // [rows + 1]
  int32_t* lcol;           // [nnz_light]
  double* lval;            // [nnz_light]
  int64_t* lchunk_cnt;     // [nchunks]: light entries per row chunk
  int64_t* lchunk_off;     // [nchunks + 1]: exclusive scan
};
int64_t csr_chunk_rows();
int64_t csr_nchunks(int64_t rows);
int csr_rowdot_blocks(int nsm);
int csr_rowdot_hl_blocks(int nsm, int ND);
int csr_colgather_blocks(int64_t k);
size_t csr_max_k();
cudaError_t launch_csr_build(const CsrBuildArgs& a, cudaStream_t st);   // validate + counts + per-column totals
cudaError_t launch_csr_fill(const CsrBuildArgs& a, cudaStream_t st);    // colptr + CSC + D (needs colmap)

struct CsrSketchArgs {
  const double* D;         // heavy block [rows][ldd] (nd columns used)
  int64_t rows, lo, s, k;
  uint64_t seed;
  int nd, ND, nsplit;
  int ldd;                 // row stride of D (nd rounded up to even)
  int64_t rows_per_split;
  double* part;            // [nsplit][s][ND]
  const int* heavy_cols;   // [nd]
  const int* colmap;
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* cval;
  double* At;              // s x k (row-major), fully written
  int skip_light = 0;      // 1: leave the light columns to launch_csr_sketch_slab
};
cudaError_t launch_csr_sketch(const CsrSketchArgs& a, cudaStream_t st, int nsm);
// Generate-once light sketch (csr.cu, csr_sketch_slab_kernel): the light part of
// At from the CSC copy with the per-chunk column pointers cp[J][c] (launch_csr_chunkptr);
// part: [nsplit][k][s] scratch; the heavy columns of At are left to the heavy path.
struct CsrSlabArgs {
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* cval;
  const int* colmap;
  const int32_t* cp;        // [nchunks + 1][k]
  int64_t k, rows, lo, s, nchunks;
  uint64_t seed;
  int nsplit;
  double* part;             // [nsplit][k][s]
  double* At;
};
int64_t csr_slab_chunk_rows();
int64_t csr_slab_tile_cols();
int64_t csr_slab_row_blocks(int64_t s);
cudaError_t launch_csr_chunkptr(const int64_t* colptr, const int32_t* rowidx, const int* colmap, int64_t k,
                                int64_t nchunks, int32_t* cp, cudaStream_t st, int64_t chunk_rows = 0);
// Stored-G CSR sketch (csr.cu): per chunk of g_rows shard rows, G (g_rows x s2, i contiguous)
// is generated once and read by the heavy and light kernels; Pt: [k][s] light partial.
struct CsrSketchGArgs {
  const double* D;
  int64_t rows, lo, s, s2, k, g_rows;
  uint64_t seed;
  int nd, ND, nsplit, ldd;
  double* part;            // [nsplit][s][ND] heavy partials
  const int* heavy_cols;
  const int* colmap;
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* cval;
  int32_t* cp;             // [nchunks + 1][k] chunk pointers (filled here)
  double* G;               // [g_rows][s2]
  double* Pt;              // [k][s]
  double* At;
};
int64_t csr_g_s2(int64_t s);
cudaError_t launch_csr_sketch_g(const CsrSketchGArgs& a, cudaStream_t st, int nsm);
cudaError_t launch_csr_sketch_slab(const CsrSlabArgs& a, cudaStream_t st);
cudaError_t launch_sketch_add_gblock(double* At, int64_t s, int64_t k, int64_t L, double si, uint64_t seed,
                                     cudaStream_t st, int nsm);

struct CsrRowdotArgs {
  const int64_t* rowptr;
  const int32_t* colind;
  const double* val;
  int64_t rows;
  const double* t;
  const int* colmap;
  const double* coef;      // {c1, c2, ca}
  double sx;               // sigma_X (1/lambda for the wide Tikhonov form)
  double* u;
  double* acc;             // nullable: acc_j += ca u_j (CS, wide form)
  double* npart;           // [nblocks]
  double* wpart;           // [nblocks][ND]
  const int* done;
  int ND, nblocks;
  // heavy-dense + light-CSR form (csr_rowdot_hl_kernel)
  const double* D;         // [rows][ldd] heavy block
  const int* heavy_cols;   // [nd]
  int nd, ldd;
  const int64_t* lrowptr;
  const int32_t* lcol;
  const double* lval;
};
cudaError_t launch_csr_rowdot(const CsrRowdotArgs& a, cudaStream_t st);
cudaError_t launch_csr_rowdot_hl(const CsrRowdotArgs& a, cudaStream_t st);
// single-pass variant for k <= csr_rowdot_all_max_k(): wpart[nblocks][k], then colreduce
int64_t csr_rowdot_all_max_k();
int csr_rowdot_all_default_variant();
int csr_rowdot_all_blocks(int nsm, int64_t k, int variant);
int csr_rowdot_all_blocks_max(int nsm, int64_t k);   // over every variant (workspace)
cudaError_t launch_csr_rowdot_all(const CsrRowdotArgs& a, int64_t k, int variant, cudaStream_t st);

struct CsrGatherArgs {
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* cval;
  int64_t k;
  double sx;
  const double* u;
  const int* colmap;
  const double* wpart;
  int ND;
  const double* npart;
  int nparts;
  double* zI;              // nullable (Tikhonov identity block)
  const double* t;
  const double* coef;
  double sI;
  double* out;             // k + 1
  double* blockpart;       // >= csr_colgather_blocks(k)
  unsigned* counter;
  const int* done;
};
cudaError_t launch_csr_colgather(const CsrGatherArgs& a, cudaStream_t st);

// ---- misc (misc.cu)
cudaError_t launch_fill(double* p, double v, int64_t n, cudaStream_t st);
cudaError_t launch_copy_scale(double* dst, const double* src, double scale, int64_t n, cudaStream_t st);
// row-major s x k -> column-major s x k
cudaError_t launch_transpose(const double* src, int64_t rows, int64_t cols, double* dst, cudaStream_t st);
// R (upper triangle of the k x k leading block of column-major QR, ld) -> dense k x k, zero below
cudaError_t launch_build_jw(const double* qr, int64_t ld, int64_t k, double* JW, cudaStream_t st);
cudaError_t launch_form_nt_jw(const double* E, int64_t lde, const double* ev, int64_t k, int64_t r, double* Nt,
                              cudaStream_t st);
cudaError_t launch_extract_r(const double* qr, int64_t ld, int64_t k, double* R, cudaStream_t st);
// Nt[c][j] = VT[c + j * k] / S[c], c < r, j < k  (Nt row-major r x k == N column-major)
cudaError_t launch_form_nt(const double* VT, const double* S, int64_t k, int64_t r, double* Nt,
                           cudaStream_t st);

// V column-major k x k (gesvdp): Nt[c][j] = V[j + c k] / S[c]
cudaError_t launch_form_nt_v(const double* V, const double* S, int64_t k, int64_t r, double* Nt, cudaStream_t st);
// out[0] = ||A||^2, out[1] = ||B||^2 over n entries (fixed order); part: sumsq2_part_size() doubles
cudaError_t launch_sumsq2(const double* A, const double* B, int64_t n, double* part, double* out, cudaStream_t st);
int sumsq2_part_size();
// flag[0] <- 1.0 if any of p[0..n) is not finite (never cleared here)
cudaError_t launch_check_finite(const double* p, int64_t n, double* flag, cudaStream_t st);

}  // namespace lsrn
