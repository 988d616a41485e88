// C ABI of the LSRN hot path (include/lsrn.h): planning, workspace layout, the
// sketch -> SVD -> iterations pipeline, CUDA-graph capture of the iteration
// loop, NCCL collectives for multi-GPU runs.
//
// Paper map: Alg. 1 / Alg. 2 / Alg. 3 /
// §5 Tikhonov / MPI design P:779-800 (Reduce -> here one NCCL
// allreduce of the partial sketch; one allreduce per iteration).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <cusolverDn.h>
#ifdef LSRN_WITH_NCCL
#include <nccl.h>
#endif

#include "../../include/lsrn.h"
#include "kernels.h"

using namespace lsrn;

namespace {

thread_local std::string g_last_error;

struct Fail {
  lsrn_status code;
};

lsrn_status set_error(lsrn_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define LSRN_CUDA(call)                                                                          \
  do {                                                                                           \
    cudaError_t e__ = (call);                                                                    \
    if (e__ != cudaSuccess) {                                                                    \
      g_last_error = std::string("CUDA error: ") + cudaGetErrorString(e__) + " at " #call;        \
      throw Fail{LSRN_ECUDA};                                                                    \
    }                                                                                            \
  } while (0)

#define LSRN_SOLVER(call)                                                                        \
  do {                                                                                           \
    cusolverStatus_t e__ = (call);                                                               \
    if (e__ != CUSOLVER_STATUS_SUCCESS) {                                                        \
      g_last_error = std::string("cuSOLVER error ") + std::to_string((int)e__) + " at " #call;    \
      throw Fail{LSRN_ESVD};                                                                     \
    }                                                                                            \
  } while (0)

#define LSRN_REQUIRE(cond, code, msg)                                                            \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      g_last_error = (msg);                                                                      \
      throw Fail{code};                                                                          \
    }                                                                                            \
  } while (0)

// ------------------------------------------------------------------ workspace
// Carve-up of the caller's workspace.  Offsets are aligned to 256 bytes of the
// ABSOLUTE address (16-byte vector stores, TMA bulk copies): the base is rounded
// up first, inside the 256 bytes of slack lsrn_workspace_size adds.
struct Arena {
  char* base;
  size_t pad = 0, off = 0;
  explicit Arena(void* b) : base(static_cast<char*>(b)) {
    if (base) pad = off = (256 - (reinterpret_cast<uintptr_t>(base) & 255)) & 255;
  }
  template <typename T>
  T* take(size_t count) {
    off = pad + ((off - pad + 255) & ~size_t(255));
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct Dims {
  bool tall;
  int64_t m, n, L, k, s, cnt, lo;
  double sx, si;      // sigma_X, sigma_I (tall form)
  bool has_I;         // this rank holds the Tikhonov identity block
  int64_t Lz;         // local long-vector length
};

}  // namespace

struct lsrn_ctx {
  cudaStream_t stream = nullptr;
  bool own_stream = false;            // created with stream == NULL: own stream joined to the legacy stream
  cudaEvent_t join_ev[2] = {};
  // options (lsrn_ctx_set_option)
  Overrides ovr;
  int svd_method = LSRN_SVD_AUTO;
  bool graph_reuse = true;
  double hostio_chunk_mb = 32.0;
  int lsqr_sync = 0;
  bool bcast_n = true;
  // host-staged collectives (nranks > 1 without NCCL)
  lsrn_host_allreduce_fn h_allreduce = nullptr;
  lsrn_host_bcast_fn h_bcast = nullptr;
  void* h_user = nullptr;
  std::vector<double> h_buf;
  int nranks = 1, rank = 0, device = 0, nsm = 148;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t params = nullptr;
  std::vector<char> host_ws;          // cuSOLVER 64-bit API host workspace
  // host-IO streaming of A: copy stream + per-chunk events
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ev[16] = {};
  cudaEvent_t io_ev = nullptr;
  // raw sketch cache (λ-path reuse): key of the sketch held in the workspace
  bool sketch_cached = false;
  unsigned char sketch_key[160] = {};
#ifdef LSRN_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  // cached iteration graph
  cudaGraphExec_t gexec = nullptr;
  // the iteration graph is re-captured only when something it bakes in changed
  std::vector<int64_t> graph_key;
  int graph_launches = 0, graph_pass_ev = 0;
  int svd_polar_fallbacks = 0;        // polar SVD results rejected (redone with gesvd)
  int svd_qr_fallbacks = 0;           // QR routes not certified full rank (SVD computed instead)
  double qr_kappa_f = 0.0;            // kappa_F(R) of the last certified QR route
  int svd_used = 0;                   // method that produced N in the last solve
  int collectives = 0;                // collective calls of the current call (reported)
  int graph_collectives = 0;          // ... inside the cached iteration graph
  std::vector<char> gkey;
  // timing
  cudaEvent_t ev[8] = {};
  bool profile = false;
  std::vector<cudaEvent_t> pass_ev;   // pairs around long-pass kernels
  int n_pass_ev = 0;
  bool stats_pending = false;   // stats[1], [2], [4] not yet computed from the pass events
  bool sketch_pending = false;  // stats[0] of the last lsrn_sketch not yet read from ev[1], ev[2]
  double stats[8] = {};
  int launches = 0;
};

namespace {

// Every ABI call that touches the device runs inside a CallScope: the context's
// kernel-plan overrides are installed for the planners (ovr()), and a context
// created on the legacy stream joins its own stream to it at entry and exit.
struct CallScope {
  lsrn_ctx* c;
  OverrideScope os;
  explicit CallScope(lsrn_ctx* c_) : c(c_), os(c_ ? &c_->ovr : nullptr) {
    if (c && c->own_stream) {
      cudaEventRecord(c->join_ev[0], cudaStreamLegacy);
      cudaStreamWaitEvent(c->stream, c->join_ev[0], 0);
    }
  }
  ~CallScope() {
    if (c && c->own_stream) {
      cudaEventRecord(c->join_ev[1], c->stream);
      cudaStreamWaitEvent(cudaStreamLegacy, c->join_ev[1], 0);
    }
  }
};

Dims make_dims(lsrn_ctx* c, const lsrn_matrix* A, double gamma, double lambda, bool allow_partial = false) {
  LSRN_REQUIRE(A != nullptr, LSRN_EINVAL, "A is NULL");
  LSRN_REQUIRE(A->m > 0 && A->n > 0, LSRN_EDIM, "m and n must be positive");
  LSRN_REQUIRE(gamma > 1.0, LSRN_EINVAL, "oversampling factor must exceed 1 (gamma > 1, Alg. 1 step 1)");
  LSRN_REQUIRE(lambda >= 0.0 && std::isfinite(lambda), LSRN_EINVAL, "lambda must be finite and >= 0");
  Dims d{};
  d.m = A->m;
  d.n = A->n;
  d.tall = A->m >= A->n;
  d.L = d.tall ? d.m : d.n;
  d.k = d.tall ? d.n : d.m;
  d.s = (int64_t)std::ceil(gamma * (double)d.k);
  d.lo = A->lo;
  d.cnt = A->cnt;
  LSRN_REQUIRE(d.lo >= 0 && d.cnt >= 0 && d.lo + d.cnt <= d.L, LSRN_EDIM, "shard [lo, lo+cnt) outside the long dimension");
  if (c->nranks == 1 && !allow_partial)
    LSRN_REQUIRE(d.lo == 0 && d.cnt == d.L, LSRN_EDIM, "single rank must hold the whole matrix");
  if (lambda > 0.0) {
    d.sx = d.tall ? 1.0 : 1.0 / lambda;
    d.si = d.tall ? lambda : 1.0;
  } else {
    d.sx = 1.0;
    d.si = 0.0;
  }
  d.has_I = (d.si != 0.0) && (d.lo == 0);   // the shard that starts the long index owns the I block
  d.Lz = d.cnt + (d.has_I ? d.k : 0);
  if (A->kind == LSRN_DENSE) {
    LSRN_REQUIRE(A->ld >= d.k, LSRN_EDIM, "leading dimension ld must be >= min(m, n)");
    LSRN_REQUIRE(A->val != nullptr || d.cnt == 0, LSRN_EINVAL, "A->val is NULL");
  } else if (A->kind == LSRN_CSR) {
    // X is always the long-index-major matrix: CSR of A (m >= n) or CSR of A^T (m < n, i.e. A in CSC)
    LSRN_REQUIRE((size_t)d.k <= csr_max_k(), LSRN_EUNSUPPORTED,
                 "CSR path supports min(m, n) <= " + std::to_string(csr_max_k()));
    LSRN_REQUIRE(A->nnz >= 0, LSRN_EDIM, "nnz must be >= 0");
    LSRN_REQUIRE(d.cnt < ((int64_t)1 << 31), LSRN_EDIM, "CSR shard must have fewer than 2^31 rows (int32 row indices)");
    LSRN_REQUIRE(d.cnt == 0 || A->rowptr != nullptr, LSRN_EINVAL, "A->rowptr is NULL");
    LSRN_REQUIRE(A->nnz == 0 || (A->colind != nullptr && A->val != nullptr), LSRN_EINVAL,
                 "A->colind / A->val is NULL");
  } else {
    throw Fail{set_error(LSRN_EINVAL, "unknown matrix kind")};
  }
  return d;
}

// Iteration counts from the Thm 4.4 bounds: LSQR, Thm 4.5 at alpha = 0
// (§8(c) C5: (log eps - log 2) / log sqrt(r/s)); CS, Alg. 3's K + 1 passes with
// rho = (sU - sL) / (sU + sL) (§8(c) C2).
struct Counts {
  double sigL, sigU;
  int lsqr, cs_passes;
};
Counts iteration_counts(double s, double r, double alpha, double tol) {
  Counts c{};
  c.sigU = 1.0 / ((1.0 - alpha) * std::sqrt(s) - std::sqrt(r));
  c.sigL = 1.0 / ((1.0 + alpha) * std::sqrt(s) + std::sqrt(r));
  const double rate0 = std::sqrt(r / s);
  c.lsqr = (int)std::ceil((std::log(tol) - std::log(2.0)) / std::log(rate0));
  if (c.lsqr < 0) c.lsqr = 0;
  c.cs_passes = 1;
  const double rho = (c.sigU - c.sigL) / (c.sigU + c.sigL);
  if (rho > 0.0) {
    const int K = (int)std::ceil((std::log(tol) - std::log(2.0)) / std::log(rho));
    c.cs_passes = (K > 0 ? K : 0) + 1;
  }
  return c;
}

int choose_nsplit(int64_t s, int64_t k, int64_t rows, int nsm) {
  int64_t mt, nt, bk;
  sketch_tile_counts(s, k, &mt, &nt, &bk);
  const int64_t tiles = mt * nt;
  if (ovr().sketch_nsplit >= 1) return ovr().sketch_nsplit;      // override (testing / tuning)
  // Split-K over rows for whole waves of CTAs: the smallest split whose last wave
  // is >= 99 % full, else the fullest (partials capped at 4 GB).  c2 (500 tiles of
  // 32 x 512): 2 splits (96.5 %) 58.1 ms, 13 splits (99.8 %) 56.5 ms
  // (profiles/r01_sketch_nsplit.jsonl).
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= 16; ++sp) {
    if (sp > 1 && rows / sp < 1024) break;
    if (sp > 1 && (double)sp * (double)s * (double)k * 8.0 > 4.0e9) break;
    const int64_t units = tiles * sp;
    const int64_t waves = (units + nsm - 1) / nsm;
    const double eff = (double)units / (double)(waves * nsm);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
    if (eff >= 0.99) break;
  }
  return best;
}

constexpr int kMaxChunks = 16;   // = size of lsrn_ctx::chunk_ev

struct SketchWs {
  int nsplit = 1;
  int64_t rows_per_split = 0;
  double* part = nullptr;   // nullptr if direct
  // LSRN_HOST_IO streaming: A arrives in nchunk H2D chunks; chunk i is sketched (split-K
  // nsplit inside the chunk) as soon as it lands and accumulated into the nsplit partials
  int nchunk = 0;
  int64_t chunk_r0[kMaxChunks + 1] = {};   // chunk i = rows [chunk_r0[i], chunk_r0[i+1])
  bool host_stream = false;                 // chunks wait on their H2D copy events
  // stored G (ovr().sketch_g != 0): each launch covers <= g_rows rows (a multiple of 16)
  // and first writes its G tiles into G (sketch_gen_g_kernel)
  double* G = nullptr;
  int64_t g_rows = 0;
};

// Stored-G plan: rows per sketch launch so that its G tiles fit the budget (0: the
// in-register path).  Needs the 32 x 512 warp-specialized kernel's layout (even ld
// and k; the kernel / tile overrides select the other kernels).
int64_t stored_g_rows(const Dims& d, int64_t ld) {
  if (ovr().sketch_g == 0 || d.cnt <= 0 || ld % 2 != 0 || d.k % 2 != 0) return 0;
  if (ovr().sketch_kernel == 1 || ovr().sketch_kernel == 2 || ovr().sketch_tile == 0) return 0;
  const double budget = ovr().sketch_g > 0 ? (double)ovr().sketch_g * 1048576.0 : 8.0e9;
  const int64_t bk = sketch_g_block_rows();
  const int64_t rows = (int64_t)(budget / (double)sketch_g_row_bytes(d.s)) / bk * bk;
  return std::max(bk, rows);
}

// split-K of one sketch launch of `rows` rows (stored G: split boundaries on k-blocks)
void launch_split(const lsrn_ctx* c, const Dims& d, int64_t rows, bool g, int* nsplit, int64_t* rps) {
  *nsplit = choose_nsplit(d.s, d.k, rows, c->nsm);
  int64_t r = (rows + *nsplit - 1) / *nsplit;
  if (g) r = (r + 15) / 16 * 16;
  *rps = r > 0 ? r : 16;
}

// Host-IO streaming: A is copied in chunks of >= 128 MB on a second stream and
// each chunk is sketched as soon as it has landed, so the H2D copy of A
// overlaps the sketch (one split-K slot per chunk, summed in fixed order).
// Chunk boundaries (rows) of the streamed host copy of A: geometric sizes (first
// 32 MB, x1.5 each, <= 16 chunks) so that the first sketch launch starts after a
// short copy and later chunks (copied at ~55 GB/s, sketched at ~29 GB/s of A)
// stay ahead of the sketch.  Returns the chunk count (1: no streaming).
int stream_chunks(const Dims& d, int64_t ld, double first_mb, int64_t* r0) {
  const double row_bytes = 8.0 * (double)ld;
  if (8.0 * (double)d.cnt * (double)ld < 2.0 * first_mb * 1024 * 1024 || d.cnt < 512) return 1;
  int n = 0;
  int64_t row = 0;
  double size = first_mb * 1024 * 1024;
  while (row < d.cnt && n < kMaxChunks) {
    r0[n++] = row;
    int64_t nr = std::max<int64_t>(256, (int64_t)(size / row_bytes) / 16 * 16);
    if (n == kMaxChunks || row + nr > d.cnt) nr = d.cnt - row;
    row += nr;
    size *= 1.5;
  }
  r0[n] = d.cnt;
  return n;
}

// the largest split-K over the launches of chunks [chunk_r0] (stored G: sub-launches of <= g_rows)
int max_nsplit(const lsrn_ctx* c, const Dims& d, const SketchWs& w) {
  int ns = 1;
  for (int i = 0; i < w.nchunk; ++i) {
    const int64_t nr = w.chunk_r0[i + 1] - w.chunk_r0[i];
    const int64_t step = w.g_rows > 0 ? w.g_rows : nr;
    for (int64_t sub = 0; sub < nr; sub += step) ns = std::max(ns, choose_nsplit(d.s, d.k, std::min(step, nr - sub), c->nsm));
  }
  return ns;
}

SketchWs plan_sketch(lsrn_ctx* c, const Dims& d, Arena& ar, bool need_finish_flag, bool host_stream = false,
                     int64_t ld = 0) {
  SketchWs w{};
  w.g_rows = stored_g_rows(d, ld);
  auto take_g = [&]() {
    if (w.g_rows > 0) w.G = ar.take<double>(sketch_g_bytes(d.s, std::min(w.g_rows, d.cnt)) / sizeof(double));
  };
  if (host_stream && d.cnt > 0) {
    w.nchunk = stream_chunks(d, ld, c->hostio_chunk_mb, w.chunk_r0);
    if (w.nchunk > 1) {
      w.host_stream = true;
      w.nsplit = max_nsplit(c, d, w);
      w.part = ar.take<double>((size_t)w.nsplit * d.s * d.k);
      take_g();
      return w;
    }
    w.nchunk = 0;
  }
  // Device-resident A larger than 4 GB: one launch per row chunk of <= 4 GB (<= 16
  // chunks), accumulated in stream order.  Within a launch the resident CTAs (one X
  // column stripe, M-tile-fastest raster) read the same rows at nearly the same time
  // and share them through L2; one launch over all of c5's 1e6 rows let them drift
  // apart (each CTA runs ~170 ms) and re-read X from DRAM 27 TB per sketch.
  const double a_bytes = 8.0 * (double)d.cnt * (double)ld;
  int nch = (int)std::ceil(a_bytes / 4.0e9);
  if (ovr().sketch_chunks >= 0) nch = ovr().sketch_chunks;
  if (w.g_rows > 0 && w.g_rows < d.cnt)       // stored G: at least one launch per budget of G tiles
    nch = std::max(nch, (int)((d.cnt + w.g_rows - 1) / w.g_rows));
  nch = std::min(nch, kMaxChunks);
  if (d.cnt > 0 && nch > 1 && d.cnt >= 16 * (int64_t)nch) {
    int64_t per = (d.cnt + nch - 1) / nch;
    per = (per + 15) / 16 * 16;
    w.nchunk = 0;
    for (int64_t row = 0; row < d.cnt && w.nchunk < kMaxChunks; row += per) w.chunk_r0[w.nchunk++] = row;
    w.chunk_r0[w.nchunk] = d.cnt;
    if (w.nchunk > 1) {
      w.nsplit = max_nsplit(c, d, w);
      w.part = ar.take<double>((size_t)w.nsplit * d.s * d.k);
      take_g();
      return w;
    }
    w.nchunk = 0;
  }
  w.g_rows = (w.g_rows > 0 && w.g_rows >= d.cnt) ? w.g_rows : 0;   // one launch (or none: cnt < 16 chunks)
  w.nsplit = choose_nsplit(d.s, d.k, d.cnt, c->nsm);
  int64_t rps = (d.cnt + w.nsplit - 1) / w.nsplit;
  rps = (rps + 15) / 16 * 16;
  w.rows_per_split = rps > 0 ? rps : 16;
  take_g();
  const bool direct = (w.nsplit == 1);
  (void)need_finish_flag;
  w.part = direct ? nullptr : ar.take<double>((size_t)w.nsplit * d.s * d.k);
  return w;
}

// ------------------------------------------------------------------ CSR (K4)
constexpr int kMaxHeavy = 64;

struct CsrWs {
  int* cntc;
  int* bad;
  int64_t *offs, *total, *colptr;
  int *colmap, *heavy_cols;
  int32_t* rowidx;
  double *cval, *D, *part, *npart, *wpart;
  int64_t *lrowptr, *lchunk_cnt, *lchunk_off;   // light-column CSR (iteration pass, k > 2048)
  // generate-once light sketch (csr_sketch_slab_kernel): per-chunk CSC pointers + split partials
  bool slab = false;
  int slab_nsplit = 1;
  int64_t slab_nchunks = 0;
  int32_t* cp = nullptr;
  double* slab_part = nullptr;
  // stored-G sketch (launch_csr_sketch_g): G rows per chunk, G block, chunk pointers, light partial
  bool gstore = false;
  int64_t g_rows = 0;
  double* G = nullptr;
  int32_t* cpg = nullptr;
  double* Pt = nullptr;
  int32_t* lcol;
  double* lval;
  int nsplit;
  int64_t rows_per_split;
  // filled by csr_prepare
  int nd = 0, ND = 0, ldd = 0;   // ldd: row stride of D (nd rounded up to even: 16-byte rows)
  int64_t nnz_light = 0;
};

CsrWs plan_csr(lsrn_ctx* c, const Dims& d, const lsrn_matrix* A, Arena& ar) {
  CsrWs w{};
  const int64_t nch = csr_nchunks(d.cnt);
  const int64_t k = d.k;
  const int64_t nnz = std::max<int64_t>(A->nnz, 1);
  w.cntc = ar.take<int>((size_t)std::max<int64_t>(nch, 1) * k);
  w.bad = ar.take<int>(4);
  w.offs = ar.take<int64_t>((size_t)std::max<int64_t>(nch, 1) * k);
  w.total = ar.take<int64_t>((size_t)k);
  w.colptr = ar.take<int64_t>((size_t)k + 1);
  w.colmap = ar.take<int>((size_t)k);
  w.heavy_cols = ar.take<int>(kMaxHeavy);
  w.rowidx = ar.take<int32_t>((size_t)nnz);
  w.cval = ar.take<double>((size_t)nnz);
  w.D = ar.take<double>((size_t)std::max<int64_t>(d.cnt, 1) * kMaxHeavy);
  w.lrowptr = ar.take<int64_t>((size_t)d.cnt + 1);
  w.lcol = ar.take<int32_t>((size_t)nnz);
  w.lval = ar.take<double>((size_t)nnz);
  w.lchunk_cnt = ar.take<int64_t>((size_t)std::max<int64_t>(nch, 1));
  w.lchunk_off = ar.take<int64_t>((size_t)nch + 1);
  // heavy-part split-K: enough (row block, split) CTAs for two waves
  const int64_t row_blocks = (d.s + 255) / 256;
  int nsplit = (int)std::max<int64_t>(1, (2 * (int64_t)c->nsm + row_blocks - 1) / row_blocks);
  nsplit = (int)std::min<int64_t>(nsplit, std::max<int64_t>(1, d.cnt / 256));
  w.nsplit = nsplit;
  w.rows_per_split = std::max<int64_t>(1, (d.cnt + nsplit - 1) / nsplit);
  w.part = ar.take<double>((size_t)nsplit * d.s * kMaxHeavy);
  w.npart = ar.take<double>((size_t)std::max(csr_rowdot_blocks(c->nsm), csr_rowdot_all_blocks_max(c->nsm, d.k)));
  const size_t wp_heavy = (size_t)csr_rowdot_blocks(c->nsm) * kMaxHeavy;
  const size_t wp_all = d.k <= csr_rowdot_all_max_k() ? (size_t)csr_rowdot_all_blocks_max(c->nsm, d.k) * d.k : 0;
  w.wpart = ar.take<double>(std::max(wp_heavy, wp_all));
  // Sketch of the CSR shard: by default the stored-G kernels (G generated once per chunk
  // of rows, <= 8 GB, and read by the heavy and light kernels): c4 7.33 -> 4.37 s, t4
  // 267 ms (slab) -> 207 ms (profiles/r02_csr_sketch_modes.jsonl).  Overrides (csr_sketch):
  // 0 the per-nonzero kernel regenerating G[:, j] per light nonzero, 1 the generate-once
  // slab kernel (each G[i, j] once per 512-column tile).
  w.slab = d.cnt > 0 && A->nnz > 0 && ovr().csr_sketch == 1;
  w.gstore = d.cnt > 0 && A->nnz > 0 && (ovr().csr_sketch == 2 || ovr().csr_sketch == -1);
  if (w.gstore) {
    // the stored-G heavy kernel holds ~1 CTA per SM (64 accumulators + 16 staged G values
    // per thread): split-K for ~16 nearly full waves
    w.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(16, d.cnt / 256));
    w.rows_per_split = std::max<int64_t>(1, (d.cnt + w.nsplit - 1) / w.nsplit);
    w.part = ar.take<double>((size_t)w.nsplit * d.s * kMaxHeavy);
    const int64_t s2 = csr_g_s2(d.s);
    // G rows per chunk.  Default: as few rows as keep ~256 nonzeros per column and chunk
    // (the light kernel's staging batch; estimated as nnz / k), but a G block of at least
    // 256 MB and at most 8 GB (as the dense G).  Small blocks stay L2-resident between
    // generation and the light gathers: t4 (82000 nonzeros per column) -> 256 MB, 245
    // chunks: 147 -> 123 ms; c4 (7000 per column) keeps 8 GB, smaller blocks are slower
    // there (launches, short heavy GEMMs: 2 GB 2.78 s vs 1.82 s; profiles/r02_csr_light2_*.jsonl).
    double budget = 8.0e9;
    if (ovr().sketch_g > 0) {
      budget = (double)ovr().sketch_g * 1048576.0;
    } else if (d.k > 0 && A->nnz > 0) {
      const double per_col = (double)A->nnz / (double)d.k;
      const double chunks = std::max(1.0, std::floor(per_col / 256.0));
      const double rows_c = std::ceil((double)d.cnt / chunks);
      budget = std::min(8.0e9, std::max(256.0 * 1048576.0, rows_c * 8.0 * (double)s2));
    }
    w.g_rows = std::max<int64_t>(1, std::min<int64_t>(d.cnt, (int64_t)(budget / (8.0 * (double)s2))));
    const int64_t nchg = (d.cnt + w.g_rows - 1) / w.g_rows;
    w.G = ar.take<double>((size_t)w.g_rows * s2);
    w.cpg = ar.take<int32_t>((size_t)(nchg + 1) * d.k);
    w.Pt = ar.take<double>((size_t)d.k * d.s);
  }
  if (w.slab) {
    w.slab_nchunks = (d.cnt + csr_slab_chunk_rows() - 1) / csr_slab_chunk_rows();
    const int64_t tiles = (d.k + csr_slab_tile_cols() - 1) / csr_slab_tile_cols();
    const int64_t ctas = csr_slab_row_blocks(d.s) * tiles;
    int64_t ns = (3 * (int64_t)c->nsm + ctas - 1) / ctas;
    ns = std::max<int64_t>(1, std::min<int64_t>({ns, 16, w.slab_nchunks}));
    w.slab_nsplit = (int)ns;
    w.cp = ar.take<int32_t>((size_t)(w.slab_nchunks + 1) * d.k);
    w.slab_part = ar.take<double>((size_t)w.slab_nsplit * d.k * d.s);
  }
  return w;
}

// CSC copy of the light columns + heavy block D.  One device->host read of the
// column counts (the heavy/light split is a host decision).
void csr_prepare(lsrn_ctx* c, const lsrn_matrix* A, const Dims& d, CsrWs& w) {
  cudaStream_t st = c->stream;
  CsrBuildArgs b{};
  b.rowptr = A->rowptr;
  b.colind = A->colind;
  b.val = A->val;
  b.rows = d.cnt;
  b.k = d.k;
  b.cntc = w.cntc;
  b.offs = w.offs;
  b.total = w.total;
  b.colmap = w.colmap;
  b.colptr = w.colptr;
  b.rowidx = w.rowidx;
  b.cval = w.cval;
  b.D = w.D;
  b.bad = w.bad;
  LSRN_CUDA(launch_csr_build(b, st));
  c->launches += 2;
  std::vector<int64_t> tot((size_t)d.k);
  int bad = 0;
  int64_t rp_ends[2] = {0, 0};   // rowptr[0], rowptr[cnt]: nnz must match before buffers sized from it are filled
  LSRN_CUDA(cudaMemcpyAsync(tot.data(), w.total, sizeof(int64_t) * d.k, cudaMemcpyDeviceToHost, st));
  LSRN_CUDA(cudaMemcpyAsync(&bad, w.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (d.cnt > 0) {
    LSRN_CUDA(cudaMemcpyAsync(&rp_ends[0], A->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaMemcpyAsync(&rp_ends[1], A->rowptr + d.cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  LSRN_CUDA(cudaStreamSynchronize(st));
  LSRN_REQUIRE(rp_ends[1] - rp_ends[0] == A->nnz, LSRN_EDIM,
               "CSR nnz = " + std::to_string(A->nnz) + " but rowptr[cnt] - rowptr[0] = " +
                   std::to_string(rp_ends[1] - rp_ends[0]));
  LSRN_REQUIRE(bad == 0, LSRN_EINVAL,
               std::string("CSR A is not canonical:") + ((bad & 1) ? " column index outside [0, n);" : "") +
                   ((bad & 2) ? " column indices not strictly increasing within a row;" : "") +
                   ((bad & 4) ? " rowptr decreasing;" : ""));
  // heavy: density >= 1/32 of the shard's rows (then one generated G[i, j] serves
  // every heavy column of row j), at most kMaxHeavy, the densest first
  const int64_t thr = std::max<int64_t>(1, (d.cnt + 31) / 32);
  std::vector<int> cand;
  for (int64_t j = 0; j < d.k; ++j)
    if (tot[j] >= thr) cand.push_back((int)j);
  std::stable_sort(cand.begin(), cand.end(), [&](int a, int b2) { return tot[a] > tot[b2]; });
  if (cand.size() > (size_t)kMaxHeavy) cand.resize(kMaxHeavy);
  std::sort(cand.begin(), cand.end());
  w.nd = (int)cand.size();
  w.ND = w.nd == 0 ? 0 : (w.nd <= 16 ? 16 : (w.nd <= 32 ? 32 : 64));
  w.ldd = (w.nd + 1) & ~1;
  std::vector<int> colmap((size_t)d.k, -1);
  for (int h = 0; h < w.nd; ++h) colmap[cand[h]] = h;
  w.nnz_light = 0;
  for (int64_t j = 0; j < d.k; ++j)
    if (colmap[j] < 0) w.nnz_light += tot[j];
  LSRN_CUDA(cudaMemcpyAsync(w.colmap, colmap.data(), sizeof(int) * d.k, cudaMemcpyHostToDevice, st));
  if (w.nd > 0)
    LSRN_CUDA(cudaMemcpyAsync(w.heavy_cols, cand.data(), sizeof(int) * w.nd, cudaMemcpyHostToDevice, st));
  b.D = w.nd > 0 ? w.D : nullptr;
  b.ld_d = w.ldd;
  b.lrowptr = w.lrowptr;
  b.lcol = w.lcol;
  b.lval = w.lval;
  b.lchunk_cnt = w.lchunk_cnt;
  b.lchunk_off = w.lchunk_off;
  LSRN_CUDA(launch_csr_fill(b, st));
  c->launches += 2;
  if (w.slab) {
    LSRN_CUDA(launch_csr_chunkptr(w.colptr, w.rowidx, w.colmap, d.k, w.slab_nchunks, w.cp, st));
    c->launches++;
  }
  LSRN_CUDA(cudaStreamSynchronize(st));   // host vectors above are pageable: keep them alive until copied
}

// Raw sketch S0 = G[:, lo:lo+cnt] X_shard (no scaling, no Tikhonov block) of a CSR shard.
void run_sketch_csr(lsrn_ctx* c, const Dims& d, uint64_t seed, CsrWs& w, double* At) {
  if (w.gstore) {
    CsrSketchGArgs g{};
    g.D = w.D;
    g.rows = d.cnt;
    g.lo = d.lo;
    g.s = d.s;
    g.s2 = csr_g_s2(d.s);
    g.k = d.k;
    g.g_rows = w.g_rows;
    g.seed = seed;
    g.nd = w.nd;
    g.ND = w.ND;
    g.nsplit = w.nsplit;
    g.ldd = w.ldd;
    g.part = w.part;
    g.heavy_cols = w.heavy_cols;
    g.colmap = w.colmap;
    g.colptr = w.colptr;
    g.rowidx = w.rowidx;
    g.cval = w.cval;
    g.cp = w.cpg;
    g.G = w.G;
    g.Pt = w.Pt;
    g.At = At;
    LSRN_CUDA(launch_csr_sketch_g(g, c->stream, c->nsm));
    const int64_t nchg = (d.cnt + w.g_rows - 1) / w.g_rows;
    c->launches += 1 + (int)nchg * (2 + (w.nd > 0 ? 1 : 0)) + (w.nd > 0 ? 1 : 0) + 1;
    return;
  }
  CsrSketchArgs a{};
  a.D = w.D;
  a.rows = d.cnt;
  a.lo = d.lo;
  a.s = d.s;
  a.k = d.k;
  a.seed = seed;
  a.nd = w.nd;
  a.ND = w.ND;
  a.ldd = w.ldd;
  a.nsplit = w.nsplit;
  a.rows_per_split = w.rows_per_split;
  a.part = w.part;
  a.heavy_cols = w.heavy_cols;
  a.colmap = w.colmap;
  a.colptr = w.colptr;
  a.rowidx = w.rowidx;
  a.cval = w.cval;
  a.At = At;
  a.skip_light = w.slab ? 1 : 0;
  LSRN_CUDA(launch_csr_sketch(a, c->stream, c->nsm));
  c->launches += (w.nd > 0 ? 2 : 0) + (w.slab ? 0 : 1);
  if (w.slab) {
    CsrSlabArgs sa{};
    sa.colptr = w.colptr;
    sa.rowidx = w.rowidx;
    sa.cval = w.cval;
    sa.colmap = w.colmap;
    sa.cp = w.cp;
    sa.k = d.k;
    sa.rows = d.cnt;
    sa.lo = d.lo;
    sa.s = d.s;
    sa.nchunks = w.slab_nchunks;
    sa.seed = seed;
    sa.nsplit = w.slab_nsplit;
    sa.part = w.slab_part;
    sa.At = At;
    LSRN_CUDA(launch_csr_sketch_slab(sa, c->stream));
    c->launches += 2;
  }
}

// Raw sketch S0 = G[:, lo:lo+cnt] X_shard of a dense shard (split-K partials summed in fixed order).
void run_sketch(lsrn_ctx* c, const lsrn_matrix* A, const Dims& d, uint64_t seed, const SketchWs& w, double* At) {
  cudaStream_t st = c->stream;
  if (w.nchunk > 1) {          // one launch per row chunk (host IO: each after its copy event)
    LSRN_CUDA(launch_fill(w.part, 0.0, (int64_t)w.nsplit * d.s * d.k, st));
    c->launches++;
    for (int i = 0; i < w.nchunk; ++i) {
      const int64_t c0 = w.chunk_r0[i];
      const int64_t cn = w.chunk_r0[i + 1] - c0;
      if (w.host_stream) LSRN_CUDA(cudaStreamWaitEvent(st, c->chunk_ev[i], 0));
      const int64_t step = w.G ? w.g_rows : cn;            // stored G: <= g_rows rows per launch
      for (int64_t sub = 0; sub < cn; sub += step) {
        const int64_t r0 = c0 + sub, nr = std::min(step, cn - sub);
        SketchDenseArgs a{};
        a.X = A->val + r0 * A->ld;
        a.ld = A->ld;
        a.rows = nr;
        a.k = d.k;
        a.lo = d.lo + r0;
        a.s = d.s;
        a.seed = seed;
        launch_split(c, d, nr, w.G != nullptr, &a.nsplit, &a.rows_per_split);   // nsplit <= w.nsplit
        a.out = w.part;
        a.out_split_stride = d.s * d.k;
        a.accumulate = 1;     // launches are stream-ordered: fixed summation order
        a.G = w.G;
        LSRN_CUDA(launch_sketch_dense(a, st));
        c->launches += w.G ? 2 : 1;
      }
    }
    LSRN_CUDA(launch_sketch_finish(w.part, w.nsplit, d.s * d.k, d.s, d.k, 1.0, 0.0, d.L, seed, At, st, c->nsm));
    c->launches++;
    return;
  }
  if (d.cnt > 0) {
    SketchDenseArgs a{};
    a.X = A->val;
    a.ld = A->ld;
    a.rows = d.cnt;
    a.k = d.k;
    a.lo = d.lo;
    a.s = d.s;
    a.seed = seed;
    a.rows_per_split = w.rows_per_split;
    a.nsplit = w.nsplit;
    a.out = w.part ? w.part : At;
    a.out_split_stride = d.s * d.k;
    a.G = w.G;
    LSRN_CUDA(launch_sketch_dense(a, st));
    c->launches += w.G ? 2 : 1;
  } else if (!w.part) {
    LSRN_CUDA(launch_fill(At, 0.0, d.s * d.k, st));
    c->launches++;
  }
  if (w.part) {
    if (d.cnt == 0) {
      LSRN_CUDA(launch_fill(w.part, 0.0, (int64_t)w.nsplit * d.s * d.k, st));
      c->launches++;
    }
    LSRN_CUDA(launch_sketch_finish(w.part, w.nsplit, d.s * d.k, d.s, d.k, 1.0, 0.0, d.L, seed, At, st, c->nsm));
    c->launches++;
  }
}

void allreduce(lsrn_ctx* c, double* buf, int64_t count);

// Alg. 1/2 step 3 with the §5 blocks, from the raw (allreduced) sketch S0:
//   At = sigma_X S0 + sigma_I G[:, L:L+k]   (every rank; G is deterministic)
// With one rank and a partial shard (lo > 0: a testing / manual-reduction use of
// lsrn_sketch) the block belongs to the shard that starts the long index, so
// that partial sketches still sum to the full one.
void finish_sketch(lsrn_ctx* c, const Dims& d, uint64_t seed, const double* S0, double* At) {
  LSRN_CUDA(launch_copy_scale(At, S0, d.sx, d.s * d.k, c->stream));
  c->launches++;
  if (d.si != 0.0 && (c->nranks > 1 || d.lo == 0)) {
    LSRN_CUDA(launch_sketch_add_gblock(At, d.s, d.k, d.L, d.si, seed, c->stream, c->nsm));
    c->launches++;
  }
}

// The raw sketch of the last call is kept in the workspace (Plan::S0); a later
// call with LSRN_REUSE_SKETCH and the same A, shard, gamma, seed and workspace
// skips the sketch of A and its allreduce -- the λ-path reuse of §5:
// only the Tikhonov block G_W (tall) / G_I (wide) depends on λ.
struct SketchKey {
  const void* val = nullptr;
  const void* rowptr = nullptr;
  const void* colind = nullptr;
  int64_t m = 0, n = 0, lo = 0, cnt = 0, ld = 0, nnz = 0, s = 0;
  int kind = -1;
  uint64_t seed = 0;
  const void* ws = nullptr;
};
static_assert(sizeof(SketchKey) <= 160, "sketch key must fit lsrn_ctx::sketch_key");

SketchKey make_key(const lsrn_matrix* A_user, const Dims& d, uint64_t seed, const void* ws) {
  SketchKey k;
  std::memset(static_cast<void*>(&k), 0, sizeof(k));   // padding takes part in the comparison
  k.val = A_user->val;
  k.rowptr = A_user->rowptr;
  k.colind = A_user->colind;
  k.m = A_user->m;
  k.n = A_user->n;
  k.lo = A_user->lo;
  k.cnt = A_user->cnt;
  k.ld = A_user->ld;
  k.nnz = A_user->nnz;
  k.s = d.s;
  k.kind = A_user->kind;
  k.seed = seed;
  k.ws = ws;
  return k;
}

// Collectives: NCCL on the context stream (capturable into the
// iteration graph), or host-staged through the caller's callbacks
// (lsrn_ctx_set_host_collectives: stream sync, D2H, callback, H2D).
bool host_collectives(const lsrn_ctx* c) {
#ifdef LSRN_WITH_NCCL
  if (c->comm != nullptr) return false;
#endif
  return c->nranks > 1 && c->h_allreduce != nullptr;
}

void host_stage(lsrn_ctx* c, double* buf, int64_t count, bool to_host) {
  if (to_host) {
    if ((int64_t)c->h_buf.size() < count) c->h_buf.resize((size_t)count);
    LSRN_CUDA(cudaMemcpyAsync(c->h_buf.data(), buf, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    LSRN_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    LSRN_CUDA(cudaMemcpyAsync(buf, c->h_buf.data(), sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
    LSRN_CUDA(cudaStreamSynchronize(c->stream));   // h_buf is pageable and reused by the next collective
  }
}

void allreduce(lsrn_ctx* c, double* buf, int64_t count) {
  if (count <= 0) return;
  if (c->nranks > 1 || host_collectives(c)
#ifdef LSRN_WITH_NCCL
      || c->comm != nullptr
#endif
  )
    c->collectives++;
#ifdef LSRN_WITH_NCCL
  if (c->comm != nullptr) {
    ncclResult_t r = ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c->comm, c->stream);
    if (r != ncclSuccess) {
      g_last_error = std::string("NCCL allreduce failed: ") + ncclGetErrorString(r);
      throw Fail{LSRN_ENCCL};
    }
    return;
  }
#endif
  if (c->nranks == 1) return;
  LSRN_REQUIRE(c->h_allreduce != nullptr, LSRN_ENCCL,
               "nranks > 1 needs an NCCL id at lsrn_ctx_create or lsrn_ctx_set_host_collectives");
  host_stage(c, buf, count, true);
  LSRN_REQUIRE(c->h_allreduce(c->h_user, c->h_buf.data(), count) == 0, LSRN_ENCCL, "host allreduce callback failed");
  host_stage(c, buf, count, false);
}

void broadcast(lsrn_ctx* c, double* buf, int64_t count, int root) {
  if (count <= 0) return;
  if (c->nranks > 1) c->collectives++;
#ifdef LSRN_WITH_NCCL
  if (c->comm != nullptr) {
    ncclResult_t r = ncclBroadcast(buf, buf, (size_t)count, ncclDouble, root, c->comm, c->stream);
    if (r != ncclSuccess) {
      g_last_error = std::string("NCCL broadcast failed: ") + ncclGetErrorString(r);
      throw Fail{LSRN_ENCCL};
    }
    return;
  }
#endif
  if (c->nranks == 1) return;
  LSRN_REQUIRE(c->h_bcast != nullptr, LSRN_ENCCL,
               "nranks > 1 needs an NCCL id at lsrn_ctx_create or lsrn_ctx_set_host_collectives");
  if (c->rank == root) host_stage(c, buf, count, true);
  else if ((int64_t)c->h_buf.size() < count) c->h_buf.resize((size_t)count);
  LSRN_REQUIRE(c->h_bcast(c->h_user, c->h_buf.data(), count, root) == 0, LSRN_ENCCL, "host broadcast callback failed");
  if (c->rank != root) host_stage(c, buf, count, false);
}

// ------------------------------------------------------------------ SVD
// Alg. 1/2 steps 4-5: N from the s x k sketch, outside the hot
// path.  Ãt = Q R (geqrf); when R is certified full rank N = R^{-1} (reading C23, in
// svd_local below: same preconditioned singular values as V Sigma^{-1}).  Otherwise
// the SVD of R through the symmetric eigenproblem of its Jordan-Wielandt matrix
// [[0, R^T], [R, 0]], whose eigenpairs are (+-sigma_i, [v_i; +-u_i] / sqrt 2):
// a true SVD (eigenvalues with absolute error ~ eps ||R||, no squaring of
// kappa -- unlike an eigendecomposition of R^T R), the same
// Golub-Kahan idea LAPACK's dbdsvdx uses for bidiagonal SVD.  syevdx computes
// only the k largest eigenpairs.  Measured on the c2 shape (4000 x 2000, rank
// 1800): 80 ms vs 231 ms for cuSOLVER gesvd with equal sigma / subspace
// accuracy (profiles/r01_svd_options.jsonl).
// cuSOLVER's symmetric eigensolvers accept n <= 32768, so for k > 16384 (c4,
// k = 2e4) the default is the polar route: gesvdp of R (polar decomposition
// R = U_p H, then the k x k symmetric eigenproblem of H = V Sigma V^T), 13.4 s
// on a 2e4 x 2e4 R against 47.5-72 s for gesvd, with residual ||RV - US|| / ||R||
// 7e-15 and orthogonality 9e-15 (profiles/r02_svd_options.jsonl).  The polar
// route loses accuracy on (numerically) rank-deficient R (on c2's rank-1800 R
// gesvdp put the 200 null singular values at ~1e-8 sigma_1, above the rank
// threshold, profiles/r01_svd_options.jsonl), so its result is accepted only
// when every sigma_i >= 1e-6 sigma_1 (clearly full rank, kappa <= 1e6); else the
// SVD is redone with gesvd of R, which the rank rule can trust.
constexpr int64_t kMaxJW = 32768;
constexpr double kPolarMinRatio = 1e-6;
constexpr int64_t kPolarMinK = 4096;

struct SvdWs {
  double *W1, *tau, *JW, *S, *Sd, *Nt;   // JW: Jordan-Wielandt matrix, or [R | VT] (gesvd), or [R | U | V] (polar)
  double* flag;                          // non-finite flag (1 double, allreduced)
  void* work;
  size_t work_bytes, host_bytes;
  int* info;
  int method;                            // LSRN_SVD_JW / _GESVD / _POLAR (polar may fall back)
  bool fallback_jw;                      // a rejected polar result is redone with JW (else gesvd)
  bool try_qr;                           // N = R^{-1} when R is certified full rank (C23), else `method`
  double* red;                           // sumsq2 partials + the two norms
};

// 64-bit cuSOLVER API: the c4 shape (s x k = 4e4 x 2e4) needs workspaces beyond
// 2^31 elements.
SvdWs plan_svd(lsrn_ctx* c, const Dims& d, Arena& ar) {
  SvdWs w{};
  const int64_t k = d.k;
  w.method = c->svd_method;
  // auto: the polar route from k = 4096 up (c5, k = 1e4: 2.5 s against 4.4 s for the
  // Jordan-Wielandt eigenproblem, profiles/r02_svd_c5.jsonl), falling back to JW (or
  // gesvd above its limit) when the polar result is rejected; JW below (c2: 80 ms)
  w.try_qr = w.method == LSRN_SVD_AUTO || w.method == LSRN_SVD_QR;
  if (w.method == LSRN_SVD_AUTO || w.method == LSRN_SVD_QR)
    w.method = (k >= kPolarMinK || 2 * k > kMaxJW) ? LSRN_SVD_POLAR : LSRN_SVD_JW;
  w.fallback_jw = (w.method == LSRN_SVD_POLAR) && (2 * k <= kMaxJW);
  LSRN_REQUIRE(!(w.method == LSRN_SVD_JW && 2 * k > kMaxJW), LSRN_EUNSUPPORTED,
               "LSRN_SVD_JW needs min(m, n) <= 16384 (cuSOLVER symmetric eigensolver limit)");
  size_t d1 = 0, h1 = 0, d2 = 0, h2 = 0, d3 = 0, h3 = 0;
  int64_t meig = 0;
  double vl = 0.0, vu = 0.0;
  LSRN_SOLVER(cusolverDnXgeqrf_bufferSize(c->solver, c->params, d.s, k, CUDA_R_64F, nullptr, d.s, CUDA_R_64F,
                                          nullptr, CUDA_R_64F, &d1, &h1));
  if (w.method == LSRN_SVD_JW || w.fallback_jw) {
    LSRN_SOLVER(cusolverDnXsyevdx_bufferSize(c->solver, c->params, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                             CUBLAS_FILL_MODE_LOWER, 2 * k, CUDA_R_64F, nullptr, 2 * k, &vl, &vu,
                                             k + 1, 2 * k, &meig, CUDA_R_64F, nullptr, CUDA_R_64F, &d2, &h2));
  }
  if (w.method != LSRN_SVD_JW) {
    size_t d4 = 0, h4 = 0;
    LSRN_SOLVER(cusolverDnXgesvd_bufferSize(c->solver, c->params, 'N', 'A', k, k, CUDA_R_64F, nullptr, k,
                                            CUDA_R_64F, nullptr, CUDA_R_64F, nullptr, 1, CUDA_R_64F, nullptr, k,
                                            CUDA_R_64F, &d4, &h4));
    d2 = std::max(d2, d4);
    h2 = std::max(h2, h4);
    if (w.method == LSRN_SVD_POLAR)
      LSRN_SOLVER(cusolverDnXgesvdp_bufferSize(c->solver, c->params, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F,
                                               nullptr, k, CUDA_R_64F, nullptr, CUDA_R_64F, nullptr, k, CUDA_R_64F,
                                               nullptr, k, CUDA_R_64F, &d3, &h3));
  }
  size_t d5 = 0, h5 = 0;
  if (w.try_qr)
    LSRN_SOLVER(cusolverDnXtrtri_bufferSize(c->solver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, k, CUDA_R_64F,
                                            nullptr, k, &d5, &h5));
  w.work_bytes = std::max({d1, d2, d3, d5});
  w.host_bytes = std::max({h1, h2, h3, h5});
  w.W1 = ar.take<double>((size_t)d.s * k);
  w.tau = ar.take<double>((size_t)k);
  const int nblk = (w.method == LSRN_SVD_JW || w.fallback_jw) ? 4 : (w.method == LSRN_SVD_POLAR ? 3 : 2);
  w.JW = ar.take<double>((size_t)nblk * k * k);
  w.S = ar.take<double>((size_t)2 * k);
  w.Sd = ar.take<double>((size_t)k);
  w.flag = ar.take<double>(2);
  w.work = ar.take<char>(w.work_bytes + 16);
  w.Nt = ar.take<double>((size_t)k * k);
  w.info = ar.take<int>(4);
  w.red = ar.take<double>((size_t)sumsq2_part_size() + 2);
  return w;
}

// rank rule (reading C4): r = #{sigma_i > max(s, k) 2^-52 sigma_1}
int64_t rank_of(const std::vector<double>& S, int64_t s, int64_t k) {
  const double tau = (double)std::max(s, k) * std::ldexp(1.0, -52) * S[0];
  int64_t r = 0;
  if (S[0] > 0.0)
    for (int64_t i = 0; i < k; ++i)
      if (S[i] > tau) ++r;
  return r;
}

// geqrf of the sketch + SVD of R on this rank.  S_host receives the k singular
// values, descending; Nt (r x k, row-major = N column-major) is formed.  Returns r.
int64_t svd_local(lsrn_ctx* c, const Dims& d, const double* At, const SvdWs& w, std::vector<double>& S_host) {
  cudaStream_t st = c->stream;
  const int64_t k = d.k;
  LSRN_CUDA(launch_transpose(At, d.s, k, w.W1, st));
  c->launches++;
  if (c->host_ws.size() < w.host_bytes + 16) c->host_ws.resize(w.host_bytes + 16);
  LSRN_SOLVER(cusolverDnXgeqrf(c->solver, c->params, d.s, k, CUDA_R_64F, w.W1, d.s, CUDA_R_64F, w.tau, CUDA_R_64F,
                               w.work, w.work_bytes, c->host_ws.data(), w.host_bytes, w.info));
  std::vector<double> ev((size_t)k, 0.0);
  int info[2] = {0, 0};
  auto fetch = [&](const double* sv, const char* what, int64_t meig) {
    LSRN_CUDA(cudaMemcpyAsync(ev.data(), sv, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaMemcpyAsync(info, w.info, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaStreamSynchronize(st));
    LSRN_REQUIRE(info[0] == 0 && info[1] == 0 && meig == k, LSRN_ESVD,
                 std::string("cuSOLVER geqrf/") + what + " info = " + std::to_string(info[0]) + "/" +
                     std::to_string(info[1]) + ", values " + std::to_string(meig));
  };
  double* R = w.JW;                          // gesvd / polar: R (k x k) first
  if (w.try_qr) {
    // Reading C23: N = R^{-1} (Ã = Q R) preconditions exactly as N = V Sigma^{-1}:
    // R^{-1} = V Sigma^{-1} U_R^T, so A R^{-1} = (A V Sigma^{-1}) U_R^T has the same
    // singular values (Lemma 4.2 / Thm 4.4) and LSQR / CS the same iterates up
    // to that rotation of y.  Used only when R is certified full rank under the rank rule
    // C4: kappa_F(R) = ||R||_F ||R^{-1}||_F >= kappa_2(R), required below
    // 1e-2 / (max(s, k) 2^-52); otherwise (rank-deficient or nearly so) the SVD route.
    double* Ri = w.JW + (size_t)k * k;
    LSRN_CUDA(launch_extract_r(w.W1, d.s, k, R, st));
    LSRN_CUDA(launch_extract_r(w.W1, d.s, k, Ri, st));
    c->launches += 2;
    LSRN_SOLVER(cusolverDnXtrtri(c->solver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, k, CUDA_R_64F, Ri, k, w.work,
                                 w.work_bytes, c->host_ws.data(), w.host_bytes, w.info + 1));
    LSRN_CUDA(launch_sumsq2(R, Ri, k * k, w.red, w.red + sumsq2_part_size(), st));
    c->launches += 2;
    double nrm[2] = {0.0, 0.0};
    LSRN_CUDA(cudaMemcpyAsync(nrm, w.red + sumsq2_part_size(), sizeof(nrm), cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaMemcpyAsync(info, w.info, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaStreamSynchronize(st));
    LSRN_REQUIRE(info[0] == 0, LSRN_ESVD, "cuSOLVER geqrf info = " + std::to_string(info[0]));
    const double kf = std::sqrt(nrm[0]) * std::sqrt(nrm[1]);
    const double tau = (double)std::max(d.s, k) * std::ldexp(1.0, -52);
    if (info[1] == 0 && std::isfinite(kf) && nrm[0] > 0.0 && kf * tau < 1e-2) {
      // Nt row-major r x k = N column-major: R^{-1} (column-major, zero below the diagonal)
      LSRN_CUDA(cudaMemcpyAsync(w.Nt, Ri, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
      c->svd_used = LSRN_SVD_QR;
      c->qr_kappa_f = kf;
      S_host.assign((size_t)k, 1.0);         // certified: r = k under C4 (sigma are not computed)
      return k;
    }
    c->svd_qr_fallbacks++;
  }
  auto gesvd = [&]() {
    double* VT = w.JW + (size_t)k * k;
    LSRN_CUDA(launch_extract_r(w.W1, d.s, k, R, st));
    c->launches++;
    LSRN_SOLVER(cusolverDnXgesvd(c->solver, c->params, 'N', 'A', k, k, CUDA_R_64F, R, k, CUDA_R_64F, w.S, CUDA_R_64F,
                                 nullptr, 1, CUDA_R_64F, VT, k, CUDA_R_64F, w.work, w.work_bytes, c->host_ws.data(),
                                 w.host_bytes, w.info + 1));
    fetch(w.S, "gesvd", k);
    c->svd_used = LSRN_SVD_GESVD;
    S_host.assign((size_t)k, 0.0);
    for (int64_t i = 0; i < k; ++i) S_host[i] = std::max(0.0, ev[i]);
    const int64_t r = rank_of(S_host, d.s, k);
    LSRN_REQUIRE(r > 0, LSRN_ERANK0, "sketch has numerical rank 0");
    LSRN_CUDA(launch_form_nt(VT, w.S, k, r, w.Nt, st));
    c->launches++;
    return r;
  };
  auto jw = [&]() {
    int64_t meig = k;
    double vl = 0.0, vu = 0.0;
    LSRN_CUDA(launch_build_jw(w.W1, d.s, k, w.JW, st));
    c->launches++;
    LSRN_SOLVER(cusolverDnXsyevdx(c->solver, c->params, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                  CUBLAS_FILL_MODE_LOWER, 2 * k, CUDA_R_64F, w.JW, 2 * k, &vl, &vu, k + 1, 2 * k, &meig,
                                  CUDA_R_64F, w.S, CUDA_R_64F, w.work, w.work_bytes, c->host_ws.data(), w.host_bytes,
                                  w.info + 1));
    fetch(w.S, "syevdx", meig);
    c->svd_used = LSRN_SVD_JW;
    S_host.assign((size_t)k, 0.0);
    for (int64_t i = 0; i < k; ++i) S_host[i] = std::max(0.0, ev[k - 1 - i]);   // ascending eigenvalues
    const int64_t r = rank_of(S_host, d.s, k);
    LSRN_REQUIRE(r > 0, LSRN_ERANK0, "sketch has numerical rank 0");
    LSRN_CUDA(launch_form_nt_jw(w.JW, 2 * k, w.S, k, r, w.Nt, st));
    c->launches++;
    return r;
  };
  if (w.method == LSRN_SVD_JW) return jw();
  if (w.method == LSRN_SVD_POLAR) {
    double* Up = w.JW + (size_t)k * k;
    double* Vp = w.JW + 2 * (size_t)k * k;
    LSRN_CUDA(launch_extract_r(w.W1, d.s, k, R, st));
    c->launches++;
    double herr = 0.0;
    LSRN_SOLVER(cusolverDnXgesvdp(c->solver, c->params, CUSOLVER_EIG_MODE_VECTOR, 1, k, k, CUDA_R_64F, R, k,
                                  CUDA_R_64F, w.S, CUDA_R_64F, Up, k, CUDA_R_64F, Vp, k, CUDA_R_64F, w.work,
                                  w.work_bytes, c->host_ws.data(), w.host_bytes, w.info + 1, &herr));
    LSRN_CUDA(cudaMemcpyAsync(ev.data(), w.S, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaMemcpyAsync(info, w.info, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaStreamSynchronize(st));
    LSRN_REQUIRE(info[0] == 0, LSRN_ESVD, "cuSOLVER geqrf info = " + std::to_string(info[0]));
    bool ok = info[1] == 0 && ev[0] > 0.0 && std::isfinite(ev[0]);
    for (int64_t i = 0; ok && i < k; ++i)
      ok = std::isfinite(ev[i]) && ev[i] >= kPolarMinRatio * ev[0] && (i == 0 || ev[i] <= ev[i - 1]);
    if (ok) {
      c->svd_used = LSRN_SVD_POLAR;
      S_host.assign(ev.begin(), ev.end());
      LSRN_CUDA(launch_form_nt_v(Vp, w.S, k, k, w.Nt, st));   // r = k (sigma_k >= 1e-6 sigma_1 >> threshold)
      c->launches++;
      return rank_of(S_host, d.s, k);
    }
    c->svd_polar_fallbacks++;
    if (w.fallback_jw) return jw();
  }
  return gesvd();
}

// Alg. 1/2 steps 4-5 across ranks.  With one rank, or LSRN_OPT_BCAST_N = 0, every
// rank computes the SVD itself.  Otherwise rank 0 computes it and broadcasts sigma
// (k doubles) and N^T (r x k) -- the paper's MPI_Bcast of N -- so every
// rank iterates with the same N bit for bit and derives the same r from the same
// sigma.  Returns r; S_host = sigma descending on every rank.
int64_t run_svd(lsrn_ctx* c, const Dims& d, const double* At, const SvdWs& w, std::vector<double>& S_host) {
  const int64_t k = d.k;
  if (c->nranks == 1 || !c->bcast_n) return svd_local(c, d, At, w, S_host);
  cudaStream_t st = c->stream;
  int64_t r = 0;
  if (c->rank == 0) {
    // a failure on rank 0 is still broadcast (sigma = NaN: SVD failure, 0: rank 0) so
    // that no rank waits for an N that never comes
    bool failed = false;
    Fail fail{LSRN_OK};
    try {
      r = svd_local(c, d, At, w, S_host);
    } catch (const Fail& f) {
      if (f.code == LSRN_ECUDA || f.code == LSRN_ENCCL) throw;
      failed = true;
      fail = f;
      S_host.assign((size_t)k, f.code == LSRN_ERANK0 ? 0.0 : std::nan(""));
    }
    LSRN_CUDA(cudaMemcpyAsync(w.Sd, S_host.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
    broadcast(c, w.Sd, k, 0);
    LSRN_CUDA(cudaStreamSynchronize(st));    // S_host is pageable: the copy must finish before it goes out of scope
    if (failed) throw fail;
  } else {
    broadcast(c, w.Sd, k, 0);
    S_host.assign((size_t)k, 0.0);
    LSRN_CUDA(cudaMemcpyAsync(S_host.data(), w.Sd, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaStreamSynchronize(st));
    LSRN_REQUIRE(!std::isnan(S_host[0]), LSRN_ESVD, "the SVD failed on rank 0");
    r = rank_of(S_host, d.s, k);
    LSRN_REQUIRE(r > 0, LSRN_ERANK0, "sketch has numerical rank 0");
  }
  broadcast(c, w.Nt, r * k, 0);
  return r;
}

// ------------------------------------------------------------------ iterations
struct IterWs {
  double *z, *v, *y, *wy, *xL, *wxL, *comm, *tbuf, *xbuf, *wpart, *npart, *blockpart, *ypart, *coef, *consts;
  unsigned* counters;
  LsqrState* state;
  int ncoef;
  // LSRN_COMPENSATED: low parts of the vectors that cross between the passes, a
  // zero vector (the low part of b), and the compensated passes' block partials
  double *comm_lo = nullptr, *tbuf_lo = nullptr, *xbuf_lo = nullptr, *zero_lo = nullptr;
  double *epart_s = nullptr, *epart_c = nullptr, *enpart = nullptr;
  int enb = 0;
};

enum Solver { SOLVER_LSQR = 0, SOLVER_CS = 1 };

IterWs plan_iter(lsrn_ctx* c, const Dims& d, Arena& ar, int max_passes, bool compensated) {
  IterWs w{};
  const int64_t k = d.k;
  const int64_t Lz = d.Lz > 0 ? d.Lz : 1;
  w.z = ar.take<double>((size_t)Lz);
  w.v = ar.take<double>((size_t)k);
  w.y = ar.take<double>((size_t)k);
  w.wy = ar.take<double>((size_t)k);
  w.xL = ar.take<double>((size_t)Lz);
  w.wxL = ar.take<double>((size_t)Lz);
  w.comm = ar.take<double>((size_t)k + 1);
  w.tbuf = ar.take<double>((size_t)k + 1);
  w.xbuf = ar.take<double>((size_t)k + 1);
  const int nparts = 2 * (c->nsm > 0 ? c->nsm : 148);   // row-pass partials: up to 2 CTAs per SM
  w.wpart = ar.take<double>((size_t)nparts * k);
  w.npart = ar.take<double>((size_t)nparts);
  w.blockpart = ar.take<double>((size_t)std::max(colreduce_blocks(k), csr_colgather_blocks(k)) + 1);
  w.ypart = ar.take<double>((size_t)lsqr_update_blocks(Lz > k ? Lz : k) + 1);
  w.ncoef = max_passes * 6 + 16;
  w.coef = ar.take<double>((size_t)w.ncoef);
  w.consts = ar.take<double>(16);
  w.counters = ar.take<unsigned>(4);
  w.state = ar.take<LsqrState>(1);
  if (compensated) {
    w.comm_lo = ar.take<double>((size_t)k + 1);
    w.tbuf_lo = ar.take<double>((size_t)k + 1);
    w.xbuf_lo = ar.take<double>((size_t)k + 1);
    w.zero_lo = ar.take<double>((size_t)k + 1);
    w.enb = 2 * (c->nsm > 0 ? c->nsm : 148);        // >= ext_rowpass_blocks of either pass
    w.epart_s = ar.take<double>((size_t)w.enb * k);
    w.epart_c = ar.take<double>((size_t)w.enb * k);
    w.enpart = ar.take<double>((size_t)w.enb);
  }
  return w;
}

struct Pass {
  lsrn_ctx* c;
  const Dims& d;
  const lsrn_matrix* A;
  const double* Nt;
  int64_t r;
  IterWs& w;
  RowPassPlan plong, pshort;
  const CsrWs* cw = nullptr;   // CSR A: rowdot + colgather instead of the dense row pass
  bool two_sync = false;       // LSRN_OPT_LSQR_SYNC = 1: reduce ||z||^2, then the vector (two collectives)
  bool ext = false;            // LSRN_COMPENSATED: double-double vectors between the passes

  // low part of a pass input / output (ext mode): the buffers that cross between passes
  double* lo_of(const double* p) const {
    if (p == w.comm) return w.comm_lo;
    if (p == w.tbuf) return w.tbuf_lo;
    if (p == w.xbuf) return w.xbuf_lo;
    return w.zero_lo;                      // b (fp64 input)
  }

  // compensated row pass over Y (R x C): z <- c1 z + c2 sY Y t ; out = sY Y^T z (+ I block) ; ||z||^2
  void pass_ext(const double* Y, int64_t ld, int64_t R, double sY, double* z, const double* t, const double* coef,
                double* acc, const int* done, double* out, double* zI, double sI) {
    cudaStream_t st = c->stream;
    const int nb = R > 0 ? std::min(ext_rowpass_blocks(R, c->nsm), w.enb) : 0;
    ExtRowPassArgs a{};
    a.Y = Y;
    a.ld = ld;
    a.R = R;
    a.C = d.k;
    a.sx = sY;
    a.z = z;
    a.t_hi = t;
    a.t_lo = lo_of(t);
    a.coef = coef;
    a.acc = acc;
    a.done = done;
    a.part_s = w.epart_s;
    a.part_c = w.epart_c;
    a.npart = w.enpart;
    if (nb > 0) {
      LSRN_CUDA(launch_ext_rowpass(a, nb, st));
      c->launches++;
    }
    ExtColReduceArgs r{};
    r.part_s = w.epart_s;
    r.part_c = w.epart_c;
    r.npart = w.enpart;
    r.nparts = nb;
    r.C = d.k;
    r.zI = zI;
    r.t_hi = t;
    r.t_lo = lo_of(t);
    r.coef = coef;
    r.sI = sI;
    r.out_hi = out;
    r.out_lo = lo_of(out);
    r.done = done;
    LSRN_CUDA(launch_ext_colreduce(r, st));
    c->launches++;
  }

  void reduce_out(double* out) {
    if (two_sync) {
      allreduce(c, out + d.k, 1);
      allreduce(c, out, d.k);
    } else {
      allreduce(c, out, d.k + 1);
    }
  }

  // CSR long pass (tall only): z <- c1 z + c2 A t ; out = [A^T z (+ I block) ; ||z||^2]
  void long_pass_csr(double* z, const double* t, const double* coef, double* acc, const int* done, double* out) {
    cudaStream_t st = c->stream;
    const int idx = c->n_pass_ev;
    const bool prof = c->profile && idx + 2 <= (int)c->pass_ev.size();
    if (prof) LSRN_CUDA(cudaEventRecordWithFlags(c->pass_ev[idx], st, cudaEventRecordExternal));
    CsrRowdotArgs a{};
    a.rowptr = A->rowptr;
    a.colind = A->colind;
    a.val = A->val;
    a.rows = d.cnt;
    a.t = t;
    a.colmap = cw->colmap;
    a.coef = coef;
    a.sx = d.sx;
    a.u = z;
    a.acc = acc;
    a.npart = cw->npart;
    a.wpart = cw->wpart;
    a.done = done;
    a.ND = cw->ND;
    if (d.k <= csr_rowdot_all_max_k() && ovr().csr_rowdot != 3) {
      // single pass: w for every column accumulated in shared memory, then the fixed-order block sum
      const int var = ovr().csr_all >= 0 ? ovr().csr_all : csr_rowdot_all_default_variant();
      a.nblocks = csr_rowdot_all_blocks(c->nsm, d.k, var);
      LSRN_CUDA(launch_csr_rowdot_all(a, d.k, var, st));
      ColReduceArgs r{};
      r.wpart = cw->wpart;
      r.npart = cw->npart;
      r.nparts = a.nblocks;
      r.C = d.k;
      r.zI = d.has_I ? z + d.cnt : nullptr;
      r.t = t;
      r.coef = coef;
      r.sI = d.si;
      r.out = out;
      r.blockpart = w.blockpart;
      r.counter = w.counters;
      r.done = done;
      LSRN_CUDA(launch_colreduce(r, st));
      if (prof) {
        LSRN_CUDA(cudaEventRecordWithFlags(c->pass_ev[idx + 1], st, cudaEventRecordExternal));
        c->n_pass_ev += 2;
      }
      c->launches += 2;
      reduce_out(out);
      return;
    }
    const bool v1 = ovr().csr_rowdot == 1;   // override: warp per row over the full CSR
    a.nblocks = v1 ? csr_rowdot_blocks(c->nsm) : csr_rowdot_hl_blocks(c->nsm, cw->ND);
    a.D = cw->D;
    a.heavy_cols = cw->heavy_cols;
    a.nd = cw->nd;
    a.ldd = cw->ldd;
    a.lrowptr = cw->lrowptr;
    a.lcol = cw->lcol;
    a.lval = cw->lval;
    if (v1)
      LSRN_CUDA(launch_csr_rowdot(a, st));
    else
      LSRN_CUDA(launch_csr_rowdot_hl(a, st));
    CsrGatherArgs g{};
    g.colptr = cw->colptr;
    g.rowidx = cw->rowidx;
    g.cval = cw->cval;
    g.k = d.k;
    g.sx = d.sx;
    g.u = z;
    g.colmap = cw->colmap;
    g.wpart = cw->wpart;
    g.ND = cw->ND;
    g.npart = cw->npart;
    g.nparts = a.nblocks;
    g.zI = d.has_I ? z + d.cnt : nullptr;
    g.t = t;
    g.coef = coef;
    g.sI = d.si;
    g.out = out;
    g.blockpart = w.blockpart;
    g.counter = w.counters;
    g.done = done;
    LSRN_CUDA(launch_csr_colgather(g, st));
    if (prof) {
      LSRN_CUDA(cudaEventRecordWithFlags(c->pass_ev[idx + 1], st, cudaEventRecordExternal));
      c->n_pass_ev += 2;
    }
    c->launches += 2;
    reduce_out(out);
  }

  // long pass over X: z <- c1 z + c2 sX X t (+ I block), out = [P^T z ; ||z||^2]
  void long_pass(double* z, const double* t, const double* coef, double* acc, const int* done, double* out) {
    if (ext) {
      pass_ext(A->val, A->ld, d.cnt, d.sx, z, t, coef, acc, done, out, d.has_I ? z + d.cnt : nullptr, d.si);
      return;
    }
    if (cw != nullptr) {
      long_pass_csr(z, t, coef, acc, done, out);
      return;
    }
    cudaStream_t st = c->stream;
    const int idx = c->n_pass_ev;
    const bool prof = c->profile && idx + 2 <= (int)c->pass_ev.size();
    if (d.cnt > 0) {
      RowPassArgs a{};
      a.Y = A->val;
      a.ld = A->ld;
      a.sx = d.sx;
      a.R = d.cnt;
      a.C = d.k;
      a.z = z;
      a.t = t;
      a.coef = coef;
      a.acc = acc;
      a.done = done;
      a.wpart = w.wpart;
      a.npart = w.npart;
      if (prof) LSRN_CUDA(cudaEventRecordWithFlags(c->pass_ev[idx], st, cudaEventRecordExternal));
      LSRN_CUDA(launch_rowpass(a, plong, st));
      if (prof) {
        LSRN_CUDA(cudaEventRecordWithFlags(c->pass_ev[idx + 1], st, cudaEventRecordExternal));
        c->n_pass_ev += 2;
      }
      c->launches++;
    }
    ColReduceArgs r{};
    r.wpart = w.wpart;
    r.npart = w.npart;
    r.nparts = d.cnt > 0 ? plong.nclusters : 0;
    r.C = d.k;
    r.zI = d.has_I ? z + d.cnt : nullptr;
    r.t = t;
    r.coef = coef;
    r.sI = d.si;
    r.out = out;
    r.blockpart = w.blockpart;
    r.counter = w.counters;
    r.done = done;
    LSRN_CUDA(launch_colreduce(r, st));
    c->launches++;
    reduce_out(out);
  }

  // short pass over N^T: v <- c1 v + c2 N^T wv, out = [N v ; ||v||^2]
  void short_pass(double* v, const double* wv, const double* coef, double* acc, const int* done, double* out) {
    if (ext) {
      pass_ext(Nt, d.k, r, 1.0, v, wv, coef, acc, done, out, nullptr, 0.0);
      return;
    }
    cudaStream_t st = c->stream;
    RowPassArgs a{};
    a.Y = Nt;
    a.ld = d.k;
    a.sx = 1.0;
    a.R = r;
    a.C = d.k;
    a.z = v;
    a.t = wv;
    a.coef = coef;
    a.acc = acc;
    a.done = done;
    a.wpart = w.wpart;
    a.npart = w.npart;
    LSRN_CUDA(launch_rowpass(a, pshort, st));
    c->launches++;
    ColReduceArgs rr{};
    rr.wpart = w.wpart;
    rr.npart = w.npart;
    rr.nparts = pshort.nclusters;
    rr.C = d.k;
    rr.zI = nullptr;
    rr.t = wv;
    rr.coef = coef;
    rr.sI = 0.0;
    rr.out = out;
    rr.blockpart = w.blockpart;
    rr.counter = w.counters;
    rr.done = done;
    LSRN_CUDA(launch_colreduce(rr, st));
    c->launches++;
  }
};

}  // namespace

// =================================================================== ABI
extern "C" {

const char* lsrn_last_error(void) { return g_last_error.c_str(); }

const char* lsrn_version(void) {
#ifdef LSRN_WITH_NCCL
  return "lsrn-b200 0.1 sm_100a nccl";
#else
  return "lsrn-b200 0.1 sm_100a";
#endif
}

lsrn_status lsrn_nccl_unique_id(void* id_out) {
#ifdef LSRN_WITH_NCCL
  if (!id_out) return set_error(LSRN_EINVAL, "id_out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_error(LSRN_ENCCL, ncclGetErrorString(r));
  std::memcpy(id_out, &id, sizeof(id));
  return LSRN_OK;
#else
  (void)id_out;
  return set_error(LSRN_ENCCL, "built without NCCL");
#endif
}

lsrn_status lsrn_ctx_create(lsrn_ctx** out, void* stream, int nranks, int rank, const void* nccl_id) {
  if (!out) return set_error(LSRN_EINVAL, "ctx out pointer is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(LSRN_EINVAL, "bad nranks / rank");
  lsrn_ctx* c = new lsrn_ctx();
  try {
    c->stream = static_cast<cudaStream_t>(stream);
    c->nranks = nranks;
    c->rank = rank;
    if (c->stream == nullptr || c->stream == cudaStreamLegacy) {
      // the legacy stream cannot be captured: run on an own stream joined to it per call
      LSRN_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
      for (auto& e : c->join_ev) LSRN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    LSRN_CUDA(cudaGetDevice(&c->device));
    LSRN_CUDA(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device));
    LSRN_SOLVER(cusolverDnCreate(&c->solver));
    LSRN_SOLVER(cusolverDnSetStream(c->solver, c->stream));
    LSRN_SOLVER(cusolverDnCreateParams(&c->params));
    for (auto& e : c->ev) LSRN_CUDA(cudaEventCreate(&e));
    LSRN_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (auto& e : c->chunk_ev) LSRN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    LSRN_CUDA(cudaEventCreateWithFlags(&c->io_ev, cudaEventDisableTiming));
    // nranks = 1 with an id: a one-rank communicator, so that the NCCL path (the
    // allreduces, also inside the captured iteration graph) runs on a single GPU
    // nranks > 1 without an id: collectives come from lsrn_ctx_set_host_collectives
    if (nccl_id != nullptr) {
#ifdef LSRN_WITH_NCCL
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
      LSRN_REQUIRE(r == ncclSuccess, LSRN_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
#else
      (void)nccl_id;
      throw Fail{set_error(LSRN_ENCCL, "built without NCCL")};
#endif
    }
  } catch (const Fail& f) {
    lsrn_ctx_destroy(c);
    return f.code;
  }
  *out = c;
  return LSRN_OK;
}

lsrn_status lsrn_ctx_destroy(lsrn_ctx* c) {
  if (!c) return LSRN_OK;
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->pass_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (c->io_ev) cudaEventDestroy(c->io_ev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (auto& e : c->join_ev)
    if (e) cudaEventDestroy(e);
  if (c->own_stream && c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  if (c->params) cusolverDnDestroyParams(c->params);
  if (c->solver) cusolverDnDestroy(c->solver);
#ifdef LSRN_WITH_NCCL
  if (c->comm) ncclCommDestroy(c->comm);
#endif
  delete c;
  return LSRN_OK;
}

lsrn_status lsrn_ctx_set_profiling(lsrn_ctx* c, int on) {
  if (!c) return set_error(LSRN_EINVAL, "ctx is NULL");
  c->profile = on != 0;
  return LSRN_OK;
}

lsrn_status lsrn_ctx_set_option(lsrn_ctx* c, int option, int64_t value) {
  if (!c) return set_error(LSRN_EINVAL, "ctx is NULL");
  auto bad = [&]() {
    return set_error(LSRN_EINVAL, "invalid value " + std::to_string(value) + " for option " + std::to_string(option));
  };
  auto in = [&](int64_t lo, int64_t hi) { return value >= lo && value <= hi; };
  Overrides& o = c->ovr;
  switch (option) {
    case LSRN_OPT_PROFILING: if (!in(0, 1)) return bad(); c->profile = value != 0; break;
    case LSRN_OPT_SVD: if (!in(LSRN_SVD_AUTO, LSRN_SVD_QR)) return bad(); c->svd_method = (int)value; break;
    case LSRN_OPT_GRAPH_REUSE: if (!in(0, 1)) return bad(); c->graph_reuse = value != 0; break;
    case LSRN_OPT_HOSTIO_CHUNK_MB: if (!in(1, 1 << 20)) return bad(); c->hostio_chunk_mb = (double)value; break;
    case LSRN_OPT_LSQR_SYNC: if (!in(0, 1)) return bad(); c->lsqr_sync = (int)value; break;
    case LSRN_OPT_BCAST_N: if (!in(0, 1)) return bad(); c->bcast_n = value != 0; break;
    case LSRN_OPT_SKETCH_KERNEL: if (!in(-1, 2)) return bad(); o.sketch_kernel = (int)value; break;
    case LSRN_OPT_SKETCH_TILE: if (!in(-1, 1)) return bad(); o.sketch_tile = (int)value; break;
    case LSRN_OPT_SKETCH_MAXCL: if (!in(-1, 4)) return bad(); o.sketch_maxcl = (int)value; break;
    case LSRN_OPT_SKETCH_X_L2: if (!in(-1, 1)) return bad(); o.sketch_x_l2 = (int)value; break;
    case LSRN_OPT_SKETCH_CHUNKS: if (!in(-1, 16)) return bad(); o.sketch_chunks = (int)value; break;
    case LSRN_OPT_SKETCH_G: if (!in(-1, 1 << 20)) return bad(); o.sketch_g = (int)value; break;
    case LSRN_OPT_SKETCH_NSPLIT: if (!in(-1, 64) || value == 0) return bad(); o.sketch_nsplit = (int)value; break;
    case LSRN_OPT_ROWPASS_KEEP: if (!in(-1, 1)) return bad(); o.rowpass_keep = (int)value; break;
    case LSRN_OPT_ROWPASS_OCC: if (!in(-1, 2) || value == 0) return bad(); o.rowpass_occ = (int)value; break;
    case LSRN_OPT_ROWPASS_WIDE1: if (!in(-1, 1)) return bad(); o.rowpass_wide1 = (int)value; break;
    case LSRN_OPT_ROWPASS_WIDE2: if (!in(-1, 1)) return bad(); o.rowpass_wide2 = (int)value; break;
    case LSRN_OPT_ROWPASS_ASYNCX: if (!in(-1, 1)) return bad(); o.rowpass_asyncx = (int)value; break;
    case LSRN_OPT_ROWPASS_NT: if (!(value == -1 || value == 256 || value == 512)) return bad(); o.rowpass_nt = (int)value; break;
    case LSRN_OPT_ROWPASS_TR: if (!in(-1, 2) || value == 0) return bad(); o.rowpass_tr = (int)value; break;
    case LSRN_OPT_ROWPASS_BUDGET_KB: if (!(value == -1 || in(16, 227))) return bad(); o.rowpass_budget_kb = (int)value; break;
    case LSRN_OPT_ROWPASS_WIDE_SLICE: if (!(value == -1 || in(512, 1 << 20))) return bad(); o.rowpass_wide_slice = (int)value; break;
    case LSRN_OPT_ROWPASS_PF: if (!in(-1, 8)) return bad(); o.rowpass_pf = (int)value; break;
    case LSRN_OPT_CSR_ROWDOT: if (!in(-1, 3)) return bad(); o.csr_rowdot = (int)value; break;
    case LSRN_OPT_CSR_SKETCH: if (!in(-1, 2)) return bad(); o.csr_sketch = (int)value; break;
    case LSRN_OPT_CSR_HEAVY_FMA: if (!in(-1, 1)) return bad(); o.csr_heavy_fma = (int)value; break;
    case LSRN_OPT_CSR_LIGHT:
      if (!(value == -1 || (value >= 12 && value <= 648 && (value % 10 == 2 || value % 10 == 4 || value % 10 == 8))))
        return bad();
      o.csr_light = (int)value;
      break;
    case LSRN_OPT_CSR_ALL: if (!(value == -1 || value == 0 || value == 6 || value == 10)) return bad(); o.csr_all = (int)value; break;
    default: return set_error(LSRN_EINVAL, "unknown option " + std::to_string(option));
  }
  return LSRN_OK;
}

lsrn_status lsrn_ctx_set_host_collectives(lsrn_ctx* c, lsrn_host_allreduce_fn allreduce_fn, lsrn_host_bcast_fn bcast_fn,
                                          void* user) {
  if (!c) return set_error(LSRN_EINVAL, "ctx is NULL");
  if ((allreduce_fn == nullptr) != (bcast_fn == nullptr))
    return set_error(LSRN_EINVAL, "give both host collectives (or neither, to unset them)");
  c->h_allreduce = allreduce_fn;
  c->h_bcast = bcast_fn;
  c->h_user = user;
  return LSRN_OK;
}

}  // extern "C"
namespace {
extern int g_elapsed_err;
double elapsed_s(cudaEvent_t a, cudaEvent_t b);
}  // namespace
extern "C" {

lsrn_status lsrn_last_stats(lsrn_ctx* c, double* out, int cap) {
  if (!c || !out) return set_error(LSRN_EINVAL, "NULL argument");
  if (c->sketch_pending) {
    c->sketch_pending = false;
    cudaEventSynchronize(c->ev[2]);
    c->stats[0] = elapsed_s(c->ev[1], c->ev[2]) * 1e3;
  }
  if (c->stats_pending) {
    c->stats_pending = false;
    double lp = 0.0;
    int nlp = 0;
    for (int i = 0; i + 1 < c->n_pass_ev; i += 2) {
      lp += elapsed_s(c->pass_ev[i], c->pass_ev[i + 1]) * 1e3;
      ++nlp;
    }
    c->stats[1] = nlp ? lp / nlp : 0.0;
    c->stats[2] = (double)g_elapsed_err;
    c->stats[4] = (double)nlp;
  }
  for (int i = 0; i < cap && i < 8; ++i) out[i] = c->stats[i];
  return LSRN_OK;
}

lsrn_status lsrn_choose_gamma(const lsrn_report* pr, int64_t m, int64_t n, double tol, int solver,
                              double gamma_lo, double gamma_hi, double* gamma_out, double* t_out) {
  if (!pr || !gamma_out) return set_error(LSRN_EINVAL, "NULL argument");
  if (m <= 0 || n <= 0) return set_error(LSRN_EDIM, "m and n must be positive");
  if (!(tol > 0.0 && tol < 1.0)) return set_error(LSRN_EINVAL, "tol must lie in (0, 1)");
  if (solver != LSRN_SOLVER_LSQR && solver != LSRN_SOLVER_CS) return set_error(LSRN_EINVAL, "unknown solver");
  if (!(gamma_lo > 1.0 && gamma_hi >= gamma_lo)) return set_error(LSRN_EINVAL, "need 1 < gamma_lo <= gamma_hi");
  if (pr->s <= 0 || pr->r <= 0 || pr->r >= pr->s || pr->iters <= 0 || !(pr->t_sketch >= 0.0) ||
      !(pr->t_svd >= 0.0) || !(pr->t_iter > 0.0))
    return set_error(LSRN_EINVAL, "probe report unusable (needs s > r > 0, iters > 0, stage times)");
  const double k = (double)std::min(m, n);
  const double s0 = (double)pr->s, r = (double)pr->r;
  const double svd0 = 2.0 * s0 * k * k + 11.0 * k * k * k;
  const double per_it = pr->t_iter / (double)pr->iters;
  double best_t = INFINITY, best_g = 0.0;
  for (int step = 0;; ++step) {
    const double g = gamma_lo + 0.01 * step;
    if (g > gamma_hi + 1e-12) break;
    const double s = std::ceil(g * k);
    const double alpha = 1.0 / std::sqrt(s);
    if (!(alpha < 1.0 - std::sqrt(r / s))) continue;          // Thm 4.4 needs s large enough
    const Counts cn = iteration_counts(s, r, alpha, tol);
    const int it = solver == LSRN_SOLVER_LSQR ? cn.lsqr : cn.cs_passes;
    const double t = pr->t_sketch * s / s0 + pr->t_svd * (2.0 * s * k * k + 11.0 * k * k * k) / svd0 + per_it * it;
    if (t < best_t) {
      best_t = t;
      best_g = g;
    }
  }
  if (!(best_g > 1.0)) return set_error(LSRN_EINVAL, "no gamma in the range gives s with alpha < 1 - sqrt(r/s)");
  *gamma_out = best_g;
  if (t_out) *t_out = best_t;
  return LSRN_OK;
}

}  // extern "C"

// -------------------------------------------------------------- shared driver
namespace {

struct HostIO {
  lsrn_matrix Adev;
  const double* b = nullptr;
  double* x = nullptr;
};

struct Plan {
  Dims d;
  SketchWs sw;
  CsrWs cw;
  SvdWs vw;
  IterWs iw;
  double* At = nullptr;
  double* S0 = nullptr;
  // LSRN_HOST_IO staging (dense: A rows; CSR: rowptr / colind / val)
  double* Astage = nullptr;
  int64_t* rpstage = nullptr;
  int32_t* cistage = nullptr;
  double* bstage = nullptr;
  double* xstage = nullptr;
  bool csr = false;
};

// Carve every buffer of a solve (or of a sketch when `solve` is false) out of
// the workspace; with ar.base == nullptr only the size is computed.
size_t plan_all(lsrn_ctx* c, const lsrn_matrix* A, const lsrn_opts* o, Arena& ar, Plan& P, bool allow_partial,
                bool solve = true) {
  Dims& d = P.d;
  d = make_dims(c, A, o->gamma, o->lambda, allow_partial);
  P.csr = A->kind == LSRN_CSR;
  if (o->flags & LSRN_HOST_IO) {
    if (P.csr) {
      P.rpstage = ar.take<int64_t>((size_t)d.cnt + 1);
      P.cistage = ar.take<int32_t>((size_t)std::max<int64_t>(A->nnz, 1));
      P.Astage = ar.take<double>((size_t)std::max<int64_t>(A->nnz, 1));
    } else {
      P.Astage = ar.take<double>((size_t)d.cnt * A->ld);
    }
    if (solve) {
      P.bstage = ar.take<double>((size_t)(d.tall ? d.cnt : d.m));
      P.xstage = ar.take<double>((size_t)(d.tall ? d.n : d.cnt));
    }
  }
  P.S0 = ar.take<double>((size_t)d.s * d.k);   // raw sketch (kept for LSRN_REUSE_SKETCH)
  if (solve) P.At = ar.take<double>((size_t)d.s * d.k);
  if (P.csr)
    P.cw = plan_csr(c, d, A, ar);
  else
    P.sw = plan_sketch(c, d, ar, c->nranks > 1, (o->flags & LSRN_HOST_IO) && solve, A->ld);
  if (solve) {
    P.vw = plan_svd(c, d, ar);
    // max passes: LSQR cap (2x the count for r = k) or CS passes with r = k; bounded by a generous margin
    const int max_passes = 4096;
    P.iw = plan_iter(c, d, ar, max_passes, (o->flags & LSRN_COMPENSATED) != 0);
  }
  return ar.off;
}

// Alg. 1/2 step 3 (+ §5 blocks) into At: raw sketch S0 of the shard (skipped with
// LSRN_REUSE_SKETCH when the cached S0 matches), its allreduce, then
// At = sigma_X S0 + sigma_I G_block.  Events ev[1..3] bracket sketch / allreduce.
void sketch_stage(lsrn_ctx* c, const lsrn_matrix* A_user, const lsrn_matrix* A, Plan& P, uint64_t seed, int flags,
                  const void* ws, double* At) {
  cudaStream_t st = c->stream;
  const Dims& d = P.d;
  const SketchKey key = make_key(A_user, d, seed, ws);
  const bool reuse = (flags & LSRN_REUSE_SKETCH) != 0;
  const bool hit = c->sketch_cached && std::memcmp(c->sketch_key, &key, sizeof(key)) == 0;
  LSRN_REQUIRE(!reuse || hit, LSRN_EINVAL,
               "LSRN_REUSE_SKETCH: this context holds no sketch of this A (pointers, shard, gamma, seed) in this workspace");
  if (P.csr) csr_prepare(c, A, d, P.cw);   // CSC copy + heavy block (format conversion; also used by the iterations)
  LSRN_CUDA(cudaEventRecord(c->ev[1], st));
  if (!reuse) {
    c->sketch_cached = false;
    if (P.csr)
      run_sketch_csr(c, d, seed, P.cw, P.S0);
    else
      run_sketch(c, A, d, seed, P.sw, P.S0);
  }
  // streamed host IO: everything after the sketch reads all of A
  if (P.sw.host_stream && P.sw.nchunk > 1) LSRN_CUDA(cudaStreamWaitEvent(st, c->chunk_ev[P.sw.nchunk - 1], 0));
  LSRN_CUDA(cudaEventRecord(c->ev[2], st));
  if (!reuse) {
    allreduce(c, P.S0, d.s * d.k);
    std::memcpy(c->sketch_key, &key, sizeof(key));
    c->sketch_cached = true;
  }
  LSRN_CUDA(cudaEventRecord(c->ev[3], st));
  LSRN_CUDA(cudaGetLastError());   // every check precedes the first write to the caller's At
  finish_sketch(c, d, seed, P.S0, At);
}

// Stage host inputs (LSRN_HOST_IO) and return the device view of A.
lsrn_matrix stage_inputs(lsrn_ctx* c, const lsrn_matrix* A_in, const lsrn_opts* o, Plan& P) {
  lsrn_matrix A = *A_in;
  if (!(o->flags & LSRN_HOST_IO)) return A;
  cudaStream_t st = c->stream;
  const Dims& d = P.d;
  if (P.csr) {
    LSRN_REQUIRE(d.cnt == 0 || A_in->rowptr[d.cnt] - A_in->rowptr[0] == A_in->nnz, LSRN_EDIM,
                 "CSR nnz does not equal rowptr[cnt] - rowptr[0]");
    if (d.cnt > 0)
      LSRN_CUDA(cudaMemcpyAsync(P.rpstage, A_in->rowptr, sizeof(int64_t) * (d.cnt + 1), cudaMemcpyHostToDevice, st));
    if (A_in->nnz > 0) {
      LSRN_CUDA(cudaMemcpyAsync(P.cistage, A_in->colind, sizeof(int32_t) * A_in->nnz, cudaMemcpyHostToDevice, st));
      LSRN_CUDA(cudaMemcpyAsync(P.Astage, A_in->val, sizeof(double) * A_in->nnz, cudaMemcpyHostToDevice, st));
    }
    A.rowptr = P.rpstage;
    A.colind = P.cistage;
    A.val = P.Astage;
  } else if (P.sw.host_stream && P.sw.nchunk > 1) {
    // chunks on the copy stream (after everything already queued on the main stream,
    // which may still read the staging buffer); the sketch waits per chunk
    LSRN_CUDA(cudaEventRecord(c->io_ev, st));
    LSRN_CUDA(cudaStreamWaitEvent(c->copy_stream, c->io_ev, 0));
    for (int i = 0; i < P.sw.nchunk; ++i) {
      const int64_t r0 = P.sw.chunk_r0[i];
      const int64_t nr = P.sw.chunk_r0[i + 1] - r0;
      LSRN_CUDA(cudaMemcpyAsync(P.Astage + r0 * A_in->ld, A_in->val + r0 * A_in->ld, sizeof(double) * nr * A_in->ld,
                                cudaMemcpyHostToDevice, c->copy_stream));
      LSRN_CUDA(cudaEventRecord(c->chunk_ev[i], c->copy_stream));
    }
    A.val = P.Astage;
  } else {
    if (d.cnt > 0)
      LSRN_CUDA(cudaMemcpyAsync(P.Astage, A_in->val, sizeof(double) * d.cnt * A_in->ld, cudaMemcpyHostToDevice, st));
    A.val = P.Astage;
  }
  return A;
}

void validate_opts(const lsrn_opts* o) {
  LSRN_REQUIRE(o != nullptr, LSRN_EINVAL, "opts is NULL");
  LSRN_REQUIRE(o->tol > 0.0 && o->tol < 1.0, LSRN_EINVAL, "tol must lie in (0, 1)");
  LSRN_REQUIRE(o->mode == LSRN_MODE_PREDICTABLE || o->mode == LSRN_MODE_ADAPTIVE, LSRN_EINVAL, "unknown mode");
  LSRN_REQUIRE(o->max_iter >= 0, LSRN_EINVAL, "max_iter must be >= 0");
}

int g_elapsed_err = 0;
double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaError_t e = cudaEventElapsedTime(&ms, a, b);
  if (e != cudaSuccess) {
    if (!g_elapsed_err) g_elapsed_err = (int)e;
    cudaGetLastError();
    return 0.0;
  }
  return ms * 1e-3;
}

lsrn_status solve_impl(lsrn_ctx* c, const lsrn_matrix* A_in, const double* b_in, const lsrn_opts* o, void* ws,
                       size_t ws_bytes, double* x_out, lsrn_report* rep, Solver solver) {
  CallScope scope(c);
  try {
    LSRN_REQUIRE(c != nullptr, LSRN_EINVAL, "ctx is NULL");
    validate_opts(o);
    LSRN_REQUIRE(A_in != nullptr && b_in != nullptr && x_out != nullptr, LSRN_EINVAL, "A, b or x is NULL");
    Arena ar(ws);
    Plan PL{};
    const size_t need = plan_all(c, A_in, o, ar, PL, false);
    Dims& d = PL.d;
    SvdWs& vw = PL.vw;
    IterWs& iw = PL.iw;
    double* At = PL.At;
    double* xstage = PL.xstage;
    LSRN_REQUIRE(ws != nullptr && ws_bytes >= need, LSRN_ENOMEM,
                 "workspace too small: need " + std::to_string(need) + " bytes");
    LSRN_REQUIRE(!(o->mode == LSRN_MODE_ADAPTIVE && !d.tall && c->nranks > 1), LSRN_EUNSUPPORTED,
                 "adaptive LSQR on a sharded wide problem is not supported (use predictable mode)");
    const bool ext = (o->flags & LSRN_COMPENSATED) != 0;
    LSRN_REQUIRE(!ext || (A_in->kind == LSRN_DENSE && c->nranks == 1), LSRN_EUNSUPPORTED,
                 "LSRN_COMPENSATED supports dense A on one rank");
    cudaStream_t st = c->stream;
    c->launches = 0;
    c->collectives = 0;
    c->svd_used = 0;
    c->n_pass_ev = 0;
    const double* b = b_in;
    double* x = x_out;
    LSRN_CUDA(cudaEventRecord(c->ev[0], st));
    if (o->flags & LSRN_HOST_IO) {
      // streamed A: b goes first on the copy stream (st waits for the last chunk of A
      // before the iterations); st itself then issues no H2D copy the sketch could queue behind
      cudaStream_t bs = (PL.sw.host_stream && PL.sw.nchunk > 1) ? c->copy_stream : st;
      if (bs != st) {
        LSRN_CUDA(cudaEventRecord(c->io_ev, st));
        LSRN_CUDA(cudaStreamWaitEvent(bs, c->io_ev, 0));
      }
      LSRN_CUDA(cudaMemcpyAsync(PL.bstage, b_in, sizeof(double) * (d.tall ? d.cnt : d.m), cudaMemcpyHostToDevice, bs));
      b = PL.bstage;
      x = xstage;
    }
    lsrn_matrix A = stage_inputs(c, A_in, o, PL);
    // ---- sketch (Alg. 1/2 step 3; §5 blocks)
    sketch_stage(c, A_in, &A, PL, o->seed, o->flags, ws, At);
    // ---- non-finite inputs: NaN / Inf anywhere in A reaches the sketch (every
    // G[i, j] is non-zero), so the s x k sketch and b are checked; the flag is
    // allreduced so that every rank takes the same decision
    LSRN_CUDA(cudaMemsetAsync(vw.flag, 0, sizeof(double), st));
    LSRN_CUDA(launch_check_finite(At, d.s * d.k, vw.flag, st));
    LSRN_CUDA(launch_check_finite(b, d.tall ? d.cnt : d.m, vw.flag, st));
    c->launches += 2;
    allreduce(c, vw.flag, 1);
    {
      double nf = 0.0;
      LSRN_CUDA(cudaMemcpyAsync(&nf, vw.flag, sizeof(double), cudaMemcpyDeviceToHost, st));
      LSRN_CUDA(cudaStreamSynchronize(st));
      LSRN_REQUIRE(nf == 0.0, LSRN_ENONFINITE, "non-finite value (NaN / Inf) in b or in the sketch of A");
    }
    // ---- SVD + N (steps 4-5), outside the hot path
    std::vector<double> S;
    const int64_t r = run_svd(c, d, At, vw, S);
    LSRN_CUDA(cudaEventRecord(c->ev[4], st));
    // ---- bounds and counts (Thm 4.4, Thm 4.5, Alg. 3)
    const double s = (double)d.s;
    double alpha = o->alpha < 0.0 ? 1.0 / std::sqrt(s) : o->alpha;
    LSRN_REQUIRE(alpha > 0.0 && alpha < 1.0 - std::sqrt((double)r / s), LSRN_EINVAL,
                 "alpha must lie in (0, 1 - sqrt(r/s)) (Thm 4.4)");
    const Counts cnts = iteration_counts(s, (double)r, alpha, o->tol);
    const double sigU = cnts.sigU, sigL = cnts.sigL;
    const int kl = cnts.lsqr;
    const int passes = cnts.cs_passes;
    int iters_graph = 0;
    if (solver == SOLVER_LSQR)
      iters_graph = (o->mode == LSRN_MODE_PREDICTABLE) ? kl : (o->max_iter > 0 ? o->max_iter : 2 * kl);
    LSRN_REQUIRE(iters_graph <= 4000 && passes <= 4000, LSRN_EINVAL, "iteration count too large");

    // ---- iteration plans
    Pass P{c, d, &A, vw.Nt, r, iw, {}, {}};
    P.two_sync = solver == SOLVER_LSQR && c->lsqr_sync == 1;
    P.ext = ext;
    const bool eager = host_collectives(c);   // host round trips cannot live in a graph
    if (PL.csr)
      P.cw = &PL.cw;
    else
      P.plong = plan_rowpass(d.cnt, d.k, A.ld, A.val, c->nsm);
    P.pshort = plan_rowpass(r, d.k, d.k, vw.Nt, c->nsm);

    // coefficient table (device): consts + CS schedule
    std::vector<double> coefh((size_t)iw.ncoef, 0.0);
    // consts: [0..2] = {1, 0, 0} copy; [3..5] = {0, 1, 0} load-only
    std::vector<double> consts(16, 0.0);
    consts[0] = 1.0;
    consts[4] = 1.0;
    if (solver == SOLVER_CS) {
      const double dd = (sigU * sigU + sigL * sigL) / 2.0, cc = (sigU * sigU - sigL * sigL) / 2.0;
      double al = 0.0;
      for (int kp = 0; kp < passes; ++kp) {
        double be;
        if (kp == 0) {
          be = 0.0;
          al = 1.0 / dd;
        } else if (kp == 1) {
          be = 0.5 * (cc / dd) * (cc / dd);
          al = 1.0 / (dd - cc * cc / (2.0 * dd));   // reading C1 (P:706 prints the reciprocal)
        } else {
          be = (al * cc / 2.0) * (al * cc / 2.0);
          al = 1.0 / (dd - al * cc * cc / 4.0);
        }
        double* e = &coefh[(size_t)kp * 6];
        // v-side pass: v <- beta v + 1 * Abar^T r (scaled), acc += alpha v
        e[0] = be;
        e[1] = 1.0;
        e[2] = al;
        // r-side pass: r <- r - alpha Abar v
        e[3] = 1.0;
        e[4] = -al;
        e[5] = 0.0;
      }
    }
    LSRN_CUDA(cudaMemcpyAsync(iw.coef, coefh.data(), sizeof(double) * coefh.size(), cudaMemcpyHostToDevice, st));
    LSRN_CUDA(cudaMemcpyAsync(iw.consts, consts.data(), sizeof(double) * 16, cudaMemcpyHostToDevice, st));

    // ---- zero state
    LSRN_CUDA(cudaMemsetAsync(iw.counters, 0, 4 * sizeof(unsigned), st));
    const int64_t Lz = d.Lz;
    LSRN_CUDA(launch_fill(iw.z, 0.0, Lz, st));
    LSRN_CUDA(launch_fill(iw.xL, 0.0, Lz, st));
    LSRN_CUDA(launch_fill(iw.wxL, 0.0, Lz, st));
    LSRN_CUDA(launch_fill(iw.v, 0.0, d.k, st));
    LSRN_CUDA(launch_fill(iw.y, 0.0, d.k, st));
    LSRN_CUDA(launch_fill(iw.wy, 0.0, d.k, st));
    LSRN_CUDA(launch_fill(iw.comm, 0.0, d.k + 1, st));
    LSRN_CUDA(launch_fill(iw.tbuf, 0.0, d.k + 1, st));
    LSRN_CUDA(launch_fill(iw.xbuf, 0.0, d.k + 1, st));
    c->launches += 9;
    if (ext) {
      for (double* q : {iw.comm_lo, iw.tbuf_lo, iw.xbuf_lo, iw.zero_lo}) LSRN_CUDA(launch_fill(q, 0.0, d.k + 1, st));
      c->launches += 4;
    }
    if (solver == SOLVER_LSQR) {
      LSRN_CUDA(launch_lsqr_init_state(iw.state, o->tol, o->mode == LSRN_MODE_ADAPTIVE ? 1 : 0, st));
      c->launches++;
    }
    if (d.tall && d.cnt > 0) {
      LSRN_CUDA(launch_copy_scale(iw.z, b, 1.0, d.cnt, st));
      c->launches++;
    }
    LSRN_CUDA(cudaEventRecord(c->ev[5], st));

    // ---- the iteration loop, captured once as a CUDA graph
    if (c->profile) {
      const size_t need_ev = 2 * (size_t)(std::max(iters_graph, passes) + 4);
      while (c->pass_ev.size() < need_ev) {
        cudaEvent_t e;
        LSRN_CUDA(cudaEventCreate(&e));
        c->pass_ev.push_back(e);
      }
    }
    const int launches_before = c->launches;
    // Everything the captured graph holds by value: pointers, sizes, plans, counts,
    // the CSR heavy/light split and the profiling events.  Coefficients, LSQR state
    // and the stop flag live in device memory and are re-initialised above, so an
    // identical key means the previous graph is this solve's graph.
    std::vector<int64_t> gk;
    auto kp = [&](const void* v) { gk.push_back((int64_t)reinterpret_cast<uintptr_t>(v)); };
    auto ki = [&](int64_t v) { gk.push_back(v); };
    auto kd = [&](double v) {
      int64_t bits;
      std::memcpy(&bits, &v, sizeof(bits));
      gk.push_back(bits);
    };
    auto kplan = [&](const RowPassPlan& q) {
      for (int64_t v : {(int64_t)q.vpt, (int64_t)q.cl, (int64_t)q.tr, (int64_t)q.nclusters, (int64_t)q.vec,
                        q.rows_per_cluster, (int64_t)q.bulk, q.cq, (int64_t)q.nst, (int64_t)q.keep, (int64_t)q.occ,
                        (int64_t)q.async_x, (int64_t)q.nt, (int64_t)q.pf})
        ki(v);
    };
    kp(A.val), kp(A.rowptr), kp(A.colind), kp(ws), kp(b), kp(x), kp(c->pass_ev.empty() ? nullptr : c->pass_ev.data());
    // workspace carve-up (offsets move when the plan changes, e.g. the SVD fallback)
    for (const void* q : {(const void*)iw.z, (const void*)iw.v, (const void*)iw.y, (const void*)iw.wy,
                          (const void*)iw.xL, (const void*)iw.wxL, (const void*)iw.comm, (const void*)iw.tbuf,
                          (const void*)iw.xbuf, (const void*)iw.wpart, (const void*)iw.npart,
                          (const void*)iw.blockpart, (const void*)iw.ypart, (const void*)iw.coef,
                          (const void*)iw.consts, (const void*)iw.counters, (const void*)iw.state,
                          (const void*)vw.Nt})
      kp(q);
    if (PL.csr)
      for (const void* q : {(const void*)PL.cw.colptr, (const void*)PL.cw.rowidx, (const void*)PL.cw.cval,
                            (const void*)PL.cw.D, (const void*)PL.cw.colmap, (const void*)PL.cw.heavy_cols,
                            (const void*)PL.cw.wpart, (const void*)PL.cw.npart, (const void*)PL.cw.lrowptr,
                            (const void*)PL.cw.lcol, (const void*)PL.cw.lval})
        kp(q);
    ki(A.ld), ki(A.nnz), ki(r), ki(iters_graph), ki(passes), ki(solver), ki(o->mode), ki(c->profile ? 1 : 0);
    ki((int64_t)c->pass_ev.size()), ki(PL.csr ? 1 : 0), ki(ovr().csr_rowdot), ki(ovr().csr_all), ki(P.two_sync ? 1 : 0);
    if (PL.csr) ki(PL.cw.nd), ki(PL.cw.ND), ki(PL.cw.ldd), ki(PL.cw.nnz_light);
    ki(d.tall ? 1 : 0), ki(d.m), ki(d.n), ki(d.L), ki(d.k), ki(d.s), ki(d.cnt), ki(d.lo), kd(d.sx), kd(d.si);
    ki(d.has_I ? 1 : 0), ki(d.Lz), ki(ext ? 1 : 0);
    kplan(P.plong), kplan(P.pshort);
    const bool graph_hit = !eager && c->gexec && c->graph_key == gk && c->graph_reuse;
    cudaGraph_t graph = nullptr;
    const int coll_before = c->collectives;
    if (graph_hit) {
      c->launches += c->graph_launches;
      c->n_pass_ev = c->graph_pass_ev;
      c->collectives += c->graph_collectives;
    } else {
    c->graph_key.clear();
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    if (!eager)
      LSRN_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    else
      LSRN_CUDA(cudaEventRecord(c->ev[6], st));   // eager loop: runs right here
    try {
      const double* one = iw.consts;        // {1, 0, 0}
      const double* load = iw.consts + 3;   // {0, 1, 0}
      LsqrState* S_ = iw.state;
      const int* done = solver == SOLVER_LSQR ? &S_->done : nullptr;
      if (solver == SOLVER_LSQR) {
        if (d.tall) {
          P.long_pass(iw.z, iw.tbuf, one, nullptr, done, iw.comm);          // ||b||^2, w = P^T b
          LSRN_CUDA(launch_lsqr_after_u(S_, iw.comm, d.k, 0, st));
          P.short_pass(iw.v, iw.comm, S_->cV, nullptr, done, iw.tbuf);
          LSRN_CUDA(launch_lsqr_after_v(S_, iw.tbuf, d.k, 0, iw.y, iw.wy, iw.v, r, iw.ypart, iw.counters + 1, st));
          c->launches += 2;
          for (int it = 0; it < iters_graph; ++it) {
            P.long_pass(iw.z, iw.tbuf, S_->cU, nullptr, done, iw.comm);
            LSRN_CUDA(launch_lsqr_after_u(S_, iw.comm, d.k, 1, st));
            P.short_pass(iw.v, iw.comm, S_->cV, nullptr, done, iw.tbuf);
            LSRN_CUDA(launch_lsqr_after_v(S_, iw.tbuf, d.k, 1, iw.y, iw.wy, iw.v, r, iw.ypart, iw.counters + 1, st));
            c->launches += 2;
          }
          P.short_pass(iw.y, iw.comm, one, nullptr, nullptr, iw.xbuf);    // x = N y
        } else {
          P.short_pass(iw.v, b, load, nullptr, done, iw.tbuf);             // u = N^T b, t = N u
          LSRN_CUDA(launch_lsqr_after_u(S_, iw.tbuf, d.k, 0, st));
          c->launches++;
          P.long_pass(iw.z, iw.tbuf, S_->cV, nullptr, done, iw.comm);
          LSRN_CUDA(launch_lsqr_after_v(S_, iw.comm, d.k, 0, iw.xL, iw.wxL, iw.z, Lz, iw.ypart, iw.counters + 1, st));
          c->launches++;
          for (int it = 0; it < iters_graph; ++it) {
            P.short_pass(iw.v, iw.comm, S_->cU, nullptr, done, iw.tbuf);
            LSRN_CUDA(launch_lsqr_after_u(S_, iw.tbuf, d.k, 1, st));
            c->launches++;
            P.long_pass(iw.z, iw.tbuf, S_->cV, nullptr, done, iw.comm);
            LSRN_CUDA(launch_lsqr_after_v(S_, iw.comm, d.k, 1, iw.xL, iw.wxL, iw.z, Lz, iw.ypart, iw.counters + 1, st));
            c->launches++;
          }
        }
      } else {
        if (d.tall) {
          P.long_pass(iw.z, iw.tbuf, one, nullptr, nullptr, iw.comm);       // w = P^T b
          for (int kp = 0; kp < passes; ++kp) {
            const double* e = iw.coef + (size_t)kp * 6;
            P.short_pass(iw.v, iw.comm, e, iw.y, nullptr, iw.tbuf);         // v = b v + N^T w; y += a v
            if (kp + 1 < passes) P.long_pass(iw.z, iw.tbuf, e + 3, nullptr, nullptr, iw.comm);
          }
          P.short_pass(iw.y, iw.comm, one, nullptr, nullptr, iw.xbuf);     // x = N y
        } else {
          P.short_pass(iw.v, b, load, nullptr, nullptr, iw.tbuf);          // r = N^T b, t = N r
          for (int kp = 0; kp < passes; ++kp) {
            const double* e = iw.coef + (size_t)kp * 6;
            P.long_pass(iw.z, iw.tbuf, e, iw.xL, nullptr, iw.comm);  // v = b v + P t; x += a v
            if (kp + 1 < passes) P.short_pass(iw.v, iw.comm, e + 3, nullptr, nullptr, iw.tbuf);
          }
        }
      }
    } catch (...) {
      if (!eager) {
        cudaGraph_t g2 = nullptr;
        cudaStreamEndCapture(st, &g2);
        if (g2) cudaGraphDestroy(g2);
      }
      throw;
    }
    if (!eager) {
      LSRN_CUDA(cudaStreamEndCapture(st, &graph));
      LSRN_CUDA(cudaGraphInstantiate(&c->gexec, graph, 0));
      cudaGraphDestroy(graph);
      c->graph_key = gk;
      c->graph_launches = c->launches - launches_before;
      c->graph_pass_ev = c->n_pass_ev;
      c->graph_collectives = c->collectives - coll_before;
    }
    }   // capture
    const int graph_launches = c->launches - launches_before;
    if (!eager) {
      LSRN_CUDA(cudaEventRecord(c->ev[6], st));
      LSRN_CUDA(cudaGraphLaunch(c->gexec, st));
    }
    LSRN_CUDA(cudaEventRecord(c->ev[7], st));
    // ---- recover x (Alg. 1 step 7 / §5 x = z / lambda)
    if (d.tall) {
      LSRN_CUDA(launch_copy_scale(x, iw.xbuf, 1.0, d.n, st));
    } else if (d.cnt > 0) {
      LSRN_CUDA(launch_copy_scale(x, iw.xL, d.sx, d.cnt, st));
    }
    c->launches++;
    if (o->flags & LSRN_HOST_IO) {
      LSRN_CUDA(cudaMemcpyAsync(x_out, xstage, sizeof(double) * (d.tall ? d.n : d.cnt), cudaMemcpyDeviceToHost, st));
    }
    LsqrState hs{};
    if (solver == SOLVER_LSQR)
      LSRN_CUDA(cudaMemcpyAsync(&hs, iw.state, sizeof(LsqrState), cudaMemcpyDeviceToHost, st));
    LSRN_CUDA(cudaStreamSynchronize(st));
    LSRN_CUDA(cudaGetLastError());
    // ---- report
    if (rep) {
      std::memset(rep, 0, sizeof(*rep));
      rep->s = d.s;
      rep->r = r;
      rep->sigma_L = sigL;
      rep->sigma_U = sigU;
      rep->alpha = alpha;
      if (solver == SOLVER_LSQR) {
        rep->iters = hs.iters;
        rep->converged = hs.converged;
        rep->rnorm_est = hs.rnorm;
      } else {
        rep->iters = passes;
        rep->converged = 1;
      }
      rep->t_sketch = elapsed_s(c->ev[1], c->ev[2]);
      rep->t_allreduce = elapsed_s(c->ev[2], c->ev[3]);
      rep->t_svd = elapsed_s(c->ev[3], c->ev[4]);
      rep->t_iter = elapsed_s(c->ev[6], c->ev[7]);
      rep->t_total = elapsed_s(c->ev[0], c->ev[7]);
      rep->svd_used = c->svd_used;
      rep->collectives = c->collectives;
    }
    // ---- stats
    c->stats[0] = elapsed_s(c->ev[1], c->ev[2]) * 1e3;
    c->sketch_pending = false;
    // per-pass kernel times are read lazily by lsrn_last_stats (the events stay valid
    // until the next call): no host work between back-to-back solves
    c->stats_pending = true;
    c->stats[3] = (double)c->launches;
    // algorithmic bytes of one long pass: dense rows (8k + 16 per row);
    // CSR: the CSR stream (12 B per nonzero + 8 B rowptr + 16 B u per row) + the light CSC (12 B per entry)
    // (k <= 2048: single pass over the CSR, no CSC read in the iterations)
    // k > 2048: the heavy block D (8 B per heavy entry, nd per row) + the light CSR (12 B per entry,
    // 8 B row pointer) + u (16 B per row) + the light CSC (12 B per entry)
    const bool two_pass = d.k > csr_rowdot_all_max_k() || ovr().csr_rowdot == 3;
    const bool hl = two_pass && ovr().csr_rowdot != 1;
    const double csc_bytes = two_pass ? 12.0 * (double)PL.cw.nnz_light : 0.0;
    const double nnz_b = hl ? 8.0 * (double)PL.cw.nd * (double)d.cnt + 12.0 * (double)PL.cw.nnz_light
                            : 12.0 * (double)A_in->nnz;
    c->stats[5] = PL.csr ? (nnz_b + 24.0 * (double)d.cnt + csc_bytes)
                         : (double)d.cnt * ((double)d.k * 8.0 + 16.0);
    c->stats[6] = 2.0 * (double)d.s * (double)d.k * (double)d.cnt;
    c->stats[7] = (double)graph_launches;
    return LSRN_OK;
  } catch (const Fail& f) {
    if (c) {
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(c->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
      }
    }
    return f.code;
  } catch (...) {
    return set_error(LSRN_ECUDA, "unexpected C++ exception");
  }
}

}  // namespace

extern "C" {

lsrn_status lsrn_workspace_size(lsrn_ctx* c, const lsrn_matrix* A, const lsrn_opts* o, size_t* bytes) {
  CallScope scope(c);
  try {
    LSRN_REQUIRE(c != nullptr && bytes != nullptr, LSRN_EINVAL, "NULL argument");
    validate_opts(o);
    Arena ar(nullptr);
    Plan PL{};
    *bytes = plan_all(c, A, o, ar, PL, true, (o->flags & LSRN_SKETCH_ONLY) == 0) + 256;
    return LSRN_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

lsrn_status lsrn_sketch(lsrn_ctx* c, const lsrn_matrix* A, double gamma, double lambda, uint64_t seed, void* ws,
                        size_t ws_bytes, double* At, int64_t* s_out) {
  CallScope scope(c);
  try {
    LSRN_REQUIRE(c != nullptr && At != nullptr && A != nullptr, LSRN_EINVAL, "ctx, A or At is NULL");
    lsrn_opts o{};
    o.gamma = gamma;
    o.lambda = lambda;
    o.tol = 0.5;
    o.seed = seed;
    Arena ar(ws);
    Plan PL{};
    plan_all(c, A, &o, ar, PL, /*allow_partial=*/true, /*solve=*/false);
    const Dims& d = PL.d;
    LSRN_REQUIRE(ar.off == 0 || (ws != nullptr && ws_bytes >= ar.off), LSRN_ENOMEM,
                 "workspace too small for the sketch: need " + std::to_string(ar.off) + " bytes");
    c->launches = 0;
    c->n_pass_ev = 0;
    c->stats_pending = false;
    c->stats[1] = c->stats[4] = 0.0;
    sketch_stage(c, A, A, PL, seed, 0, ws, At);   // At is written by its last step only
    c->sketch_pending = true;                      // stats[0] read lazily from ev[1], ev[2]
    c->stats[6] = 2.0 * (double)d.s * (double)d.k * (double)d.cnt;
    if (s_out) *s_out = d.s;
    return LSRN_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

lsrn_status lsrn_solve_lsqr(lsrn_ctx* c, const lsrn_matrix* A, const double* b, const lsrn_opts* o, void* ws,
                            size_t ws_bytes, double* x, lsrn_report* rep) {
  return solve_impl(c, A, b, o, ws, ws_bytes, x, rep, SOLVER_LSQR);
}

lsrn_status lsrn_solve_cs(lsrn_ctx* c, const lsrn_matrix* A, const double* b, const lsrn_opts* o, void* ws,
                          size_t ws_bytes, double* x, lsrn_report* rep) {
  return solve_impl(c, A, b, o, ws, ws_bytes, x, rep, SOLVER_CS);
}

lsrn_status lsrn_debug_box_muller(lsrn_ctx* c, const uint32_t* words, int64_t count, int mode, double* out) {
  if (!c || !words || !out) return set_error(LSRN_EINVAL, "NULL argument");
  CallScope scope(c);
  if (mode < 0 || mode > 2) return set_error(LSRN_EINVAL, "mode must be 0 (fp64 table), 1 (libm) or 2 (integer)");
  if (count <= 0) return LSRN_OK;
  cudaError_t e = launch_debug_box_muller(words, count, mode, out, c->stream);
  if (e != cudaSuccess) return set_error(LSRN_ECUDA, cudaGetErrorString(e));
  return LSRN_OK;
}

lsrn_status lsrn_debug_rowpass(lsrn_ctx* c, const double* Y, int64_t R, int64_t C, int64_t ld, const double* t,
                               const double* coef, double sx, double* z, double* acc, double* out, int reps,
                               double* ms_out) {
  if (!c || !Y || !t || !coef || !z || !out) return set_error(LSRN_EINVAL, "NULL argument");
  if (R <= 0 || C <= 0 || ld < C || reps < 1) return set_error(LSRN_EDIM, "need R, C > 0, ld >= C, reps >= 1");
  CallScope scope(c);
  cudaStream_t st = c->stream;
  const RowPassPlan pl = plan_rowpass(R, C, ld, Y, c->nsm);
  double *wpart = nullptr, *npart = nullptr, *blockpart = nullptr;
  unsigned* counter = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaMallocAsync(&wpart, sizeof(double) * (size_t)pl.nclusters * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&npart, sizeof(double) * (size_t)pl.nclusters, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&blockpart, sizeof(double) * ((size_t)colreduce_blocks(C) + 1), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&counter, sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  RowPassArgs a{};
  a.Y = Y;
  a.ld = ld;
  a.sx = sx;
  a.R = R;
  a.C = C;
  a.z = z;
  a.t = t;
  a.coef = coef;
  a.acc = acc;
  a.wpart = wpart;
  a.npart = npart;
  ColReduceArgs r{};
  r.wpart = wpart;
  r.npart = npart;
  r.nparts = pl.nclusters;
  r.C = C;
  r.t = t;
  r.coef = coef;
  r.out = out;
  r.blockpart = blockpart;
  r.counter = counter;
  // reps > 1 (timing): the pass is repeated on the same z (z, acc change every repetition)
  for (int i = 0; i < reps && e == cudaSuccess; ++i) {
    if (i == reps - 1 && ms_out) e = cudaEventRecord(e0, st);
    if (e == cudaSuccess) e = launch_rowpass(a, pl, st);
    if (i == reps - 1 && ms_out && e == cudaSuccess) e = cudaEventRecord(e1, st);
    if (e == cudaSuccess) e = launch_colreduce(r, st);
  }
  if (e == cudaSuccess && ms_out) {
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms;
  }
  if (wpart) cudaFreeAsync(wpart, st);
  if (npart) cudaFreeAsync(npart, st);
  if (blockpart) cudaFreeAsync(blockpart, st);
  if (counter) cudaFreeAsync(counter, st);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e != cudaSuccess) return set_error(LSRN_ECUDA, cudaGetErrorString(e));
  return LSRN_OK;
}

lsrn_status lsrn_debug_gaussian(lsrn_ctx* c, uint64_t seed, const int64_t* rows, const int64_t* cols, int64_t count,
                                double* out) {
  if (!c || !rows || !cols || !out) return set_error(LSRN_EINVAL, "NULL argument");
  if (count <= 0) return LSRN_OK;
  CallScope scope(c);
  cudaError_t e = launch_debug_gaussian(seed, rows, cols, count, out, c->stream);
  if (e != cudaSuccess) return set_error(LSRN_ECUDA, cudaGetErrorString(e));
  return LSRN_OK;
}

}  // extern "C"
