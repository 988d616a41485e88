/*
 * lsrn.h -- C ABI of the B200 (sm_100a) LSRN hot path.
 *
 * LSRN: Meng, Saunders & Mahoney, "LSRN: a parallel iterative solver for
 * strongly over- or under-determined systems", arXiv 1109.5981.  Citations
 * "P:n" are lines of the paper text; "§8(c) Cn" are
 * the readings recorded in DESIGN.md ("Readings of the paper").
 *
 * Problem (§1): x* = argmin ||Ax - b||_2 of minimum length,
 * A m x n strongly over- (m >> n, Alg. 1) or under-determined
 * (m << n, Alg. 2), possibly rank deficient, optionally with
 * Tikhonov regularisation W = lambda I (§5):
 *     x_lambda = argmin 1/2 ||Ax - b||^2 + 1/2 lambda^2 ||x||^2.
 *
 * Conventions shared by every entry point
 *   - All array arguments are DEVICE pointers (CUDA global memory of the
 *     context's device), owned by the caller, unless opts->flags has
 *     LSRN_HOST_IO (then A, b and x are host pointers; pinned host memory is
 *     recommended; the library stages them through the workspace).
 *   - fp64 everywhere (P:991-992 tolerance 1e-14 implies double; §8(c) C8).
 *   - Layout of dense A ("long-index-major"): the long index is the major one.
 *       m >= n (tall): A row-major,   element (i, j) at val[(i - lo) * ld + j];
 *       m <  n (wide): A column-major, element (i, j) at val[(j - lo) * ld + i].
 *     i.e. the library always sees X = A (tall) or X = A^T (wide) as a
 *     row-major L x k matrix, L = max(m, n), k = min(m, n).  ld >= k, and the
 *     fast (16-byte vector) paths need ld even and val 16-byte aligned.
 *   - CSR (kind LSRN_CSR): the long-index-major X in CSR -- X = A for m >= n,
 *     X = A^T for m < n (i.e. a wide A given in CSC).  Rows [lo, lo+cnt) of X; rowptr has
 *     cnt+1 entries (rowptr[0] may be non-zero: entry e of local row r is
 *     colind/val[rowptr[r] - rowptr[0] + e]), colind int32 in [0, k),
 *     k = min(m, n), strictly increasing within each row (canonical CSR:
 *     sorted, no duplicates), val fp64.  A violation returns LSRN_EINVAL.
 *     k <= 24576 (the CSC build keeps one cursor per column in shared memory).
 *   - Multi-GPU: every rank calls with the SAME opts/seed; A is sharded along
 *     the long index (rows of a tall A, columns of a wide A): rank p holds
 *     [lo, lo + cnt).  b is the rank's shard of b (tall) or the full b (wide).
 *     x is the full x (tall, replicated on every rank) or the rank's shard of x
 *     (wide).  The sketch partials are combined with one NCCL allreduce
 *     (MPI_Reduce in the paper) and every iteration does one
 *     allreduce of k+1 doubles.
 *   - Every call is asynchronous on the context stream except for one
 *     device->host read of the singular values after the SVD (to get r).
 *   - Outputs are written only when the call returns LSRN_OK: every argument,
 *     shape and format check (and, for solves, the non-finite check) happens
 *     before the first write to an output.  A fault inside an asynchronous
 *     kernel surfaces as LSRN_ECUDA from this or a later call (standard CUDA
 *     semantics); output contents are then undefined.  A and b are never
 *     modified.  No C++ exception crosses the ABI; on error a thread-local
 *     message is available from lsrn_last_error().
 *   - The library performs no device allocation: every buffer lives in the
 *     caller's workspace (size from lsrn_workspace_size; any alignment -- the
 *     library aligns its carve-up to 256 bytes inside the slack it asks for).
 */
#ifndef LSRN_H
#define LSRN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LSRN_OK = 0,
  LSRN_EINVAL = -1,      /* gamma <= 1, lambda < 0, tol not in (0,1), alpha not in
                            (0, 1 - sqrt(r/s)), unknown kind/solver/mode, NULL pointer */
  LSRN_EDIM = -2,        /* inconsistent dims / shard / leading dimension */
  LSRN_ENONFINITE = -3,  /* solves: NaN / Inf in b or in the sketch of A (so in A) */
  LSRN_ERANK0 = -4,      /* "sketch has numerical rank 0" */
  LSRN_ESVD = -5,        /* cuSOLVER failed */
  LSRN_ENOMEM = -6,      /* workspace smaller than lsrn_workspace_size() */
  LSRN_ECUDA = -7,       /* CUDA runtime / launch error */
  LSRN_ENCCL = -8,       /* NCCL error or NCCL unavailable for nranks > 1 */
  LSRN_EUNSUPPORTED = -9 /* valid request this build does not implement (message says which) */
} lsrn_status;

enum { LSRN_DENSE = 0, LSRN_CSR = 1 };
enum { LSRN_MODE_PREDICTABLE = 0, LSRN_MODE_ADAPTIVE = 1 };
enum {
  LSRN_HOST_IO = 1,
  LSRN_SKETCH_ONLY = 2,    /* lsrn_workspace_size: size for lsrn_sketch only */
  /* λ-path reuse (§5: "we can reuse GA and only re-sketch W"):
   * skip the sketch of A and its allreduce and reuse the raw sketch G·A that
   * the previous call on this context left in this workspace.  Valid only if
   * A (the same pointers and values), its shard, gamma and seed are unchanged;
   * pointer / shard / gamma / seed / workspace mismatches return LSRN_EINVAL.
   * lambda may change: only the Tikhonov block depends on it. */
  LSRN_REUSE_SKETCH = 4,
  /* precision = 1 (SURVEY §8(b) lsrn_opts.precision; reading C18(ii)):
   * the iteration products A (N v) and N^T (A^T u) carry N v and A^T u as
   * double-double pairs and accumulate every dot product and column sum with
   * error-free transformations (TwoProd / TwoSum), removing the ~kappa(A) u
   * cancellation floor of plain fp64 products; the Krylov recurrences stay
   * fp64.  Dense A and nranks == 1 only (else LSRN_EUNSUPPORTED), like the
   * oracle's long-double product mode.  Slower than the fp64 passes (two
   * launches per pass, Y read twice, ~10x the arithmetic). */
  LSRN_COMPENSATED = 8
};

typedef struct lsrn_ctx lsrn_ctx;

typedef struct {
  int32_t kind;          /* LSRN_DENSE or LSRN_CSR */
  int32_t pad_;
  int64_t m, n;          /* GLOBAL dims of A */
  int64_t lo, cnt;       /* this rank's shard of the long index: [lo, lo + cnt) */
  const double* val;     /* dense: shard base (cnt rows of X, leading dim ld); CSR: values */
  int64_t ld;            /* dense leading dimension (>= k) */
  const int64_t* rowptr; /* CSR: cnt + 1 entries */
  const int32_t* colind; /* CSR: column indices (global, in [0, n)) */
  int64_t nnz;           /* CSR: must equal rowptr[cnt] - rowptr[0] (checked on the device
                            copy of rowptr before any buffer is sized from it: LSRN_EDIM);
                            cnt < 2^31 */
} lsrn_matrix;

typedef struct {
  double gamma;          /* oversampling factor > 1; s = ceil(gamma * min(m, n)) */
  double lambda;         /* Tikhonov lambda >= 0 (W = lambda I, §5); 0 = plain LS */
  double tol;            /* epsilon in (0, 1); paper default 1e-14 */
  double alpha;          /* Thm 4.4 alpha; < 0 selects the default 1/sqrt(s) (§8(c) C3) */
  uint64_t seed;         /* Philox key of G (§8(c) C9) */
  int32_t mode;          /* LSQR: LSRN_MODE_PREDICTABLE (Thm 4.5 count at alpha = 0, §8(c) C5)
                            or LSRN_MODE_ADAPTIVE (Paige-Saunders tests, capped) */
  int32_t max_iter;      /* adaptive cap; 0 = 2 x the Thm 4.5 count */
  int32_t flags;         /* LSRN_HOST_IO, LSRN_SKETCH_ONLY (workspace query), LSRN_REUSE_SKETCH,
                            LSRN_COMPENSATED */
  int32_t pad_;
} lsrn_opts;

typedef struct {
  int64_t s, r;          /* sketch size and detected rank of the sketch (§8(c) C4) */
  int32_t iters;         /* LSQR iterations / CS loop passes performed */
  int32_t converged;     /* adaptive LSQR: 1 if a stopping test fired; otherwise 1 */
  double sigma_L, sigma_U, alpha;   /* Thm 4.4 bounds used */
  double t_sketch, t_allreduce, t_svd, t_iter, t_total;  /* seconds (CUDA events) */
  double rnorm_est;      /* LSQR phibar estimate of ||Abar y - bbar|| (0 for CS) */
  int32_t svd_used;      /* method that produced N: LSRN_SVD_QR (N = R^{-1}) / _JW / _GESVD / _POLAR
                            (a rejected polar result redone with gesvd reports LSRN_SVD_GESVD) */
  int32_t collectives;   /* collective calls issued by this rank during the solve (sketch
                            allreduce, non-finite flag, sigma / N broadcasts, per-pass reductions);
                            0 with one rank and no communicator */
} lsrn_report;

/* Human-readable message of the last failing call on this thread ("" if none). */
const char* lsrn_last_error(void);

/* Library version string, build flags. */
const char* lsrn_version(void);

/* NCCL unique id (128 bytes) for lsrn_ctx_create on rank 0; LSRN_ENCCL if this
 * build has no NCCL. */
lsrn_status lsrn_nccl_unique_id(void* id_out /* 128 bytes */);

/* Create a context on the current CUDA device.
 *   stream : cudaStream_t every call is ordered on.  NULL means the legacy
 *     default stream: the context then runs on a stream of its own (the
 *     iteration loop is captured as a CUDA graph, which the legacy stream does
 *     not allow) that waits for the legacy stream at the start of every call and
 *     that the legacy stream waits for at its end, so the ordering seen by the
 *     caller is that of the legacy stream;
 *   nranks, rank : process group (1, 0 for single GPU); nccl_id from rank 0's
 *   lsrn_nccl_unique_id, identical on all ranks.  For nranks > 1 either an
 *   nccl_id (NCCL communicator, the normal multi-GPU path) or, afterwards,
 *   lsrn_ctx_set_host_collectives is required.  With nranks == 1 an id is
 *   optional and, if given, builds a one-rank communicator so the NCCL path runs
 *   on a single GPU (a testing aid).
 * Creates the cuSOLVER handle and the NCCL communicator (when an id is given). */
lsrn_status lsrn_ctx_create(lsrn_ctx** ctx, void* stream, int nranks, int rank,
                            const void* nccl_id);
lsrn_status lsrn_ctx_destroy(lsrn_ctx* ctx);

/* Context options (lsrn_ctx_set_option).  Values are validated (LSRN_EINVAL on
 * an unknown option or value).  The product options:
 *   LSRN_OPT_PROFILING      0/1, as lsrn_ctx_set_profiling.
 *   LSRN_OPT_SVD            how N is obtained from the s x k sketch (Alg. 1/2 steps 4-5,
 *                           P:489-495; outside the hot path).  Every SVD method is a
 *                           true SVD (no Gram matrix):
 *                           LSRN_SVD_AUTO (default) = LSRN_SVD_QR, falling back to the
 *                             Jordan-Wielandt eigenproblem of R for k <= 4095 and to
 *                             LSRN_SVD_POLAR above;
 *                           LSRN_SVD_QR: geqrf, then N = R^{-1} (trtri) when R is
 *                             certified full rank under the rank rule (kappa_F(R) <
 *                             1e-2 / (max(s, k) 2^-52); C23): the same
 *                             preconditioned singular values as V Sigma^{-1}; otherwise
 *                             the SVD as for AUTO;
 *                           LSRN_SVD_JW: geqrf, then syevdx on [[0, R^T], [R, 0]]
 *                             (k <= 16384, cuSOLVER's symmetric-eigensolver limit);
 *                           LSRN_SVD_GESVD: geqrf, then gesvd of R;
 *                           LSRN_SVD_POLAR: geqrf, then gesvdp of R (polar
 *                             decomposition + symmetric eigensolver, k x k).  Its
 *                             result is accepted only when every sigma_i >= 1e-6
 *                             sigma_1 (clearly full rank, where the polar route is
 *                             accurate); otherwise the SVD is redone with gesvd, so
 *                             the rank rule (C4) always sees exact
 *                             singular values.
 *   LSRN_OPT_GRAPH_REUSE    1 (default): reuse the captured iteration graph when
 *                           nothing it holds by value changed; 0: capture every solve.
 *   LSRN_OPT_HOSTIO_CHUNK_MB  first chunk (MB, default 32) of the streamed
 *                           LSRN_HOST_IO copy of dense A.
 *   LSRN_OPT_LSQR_SYNC      collectives per LSQR half-step with nranks > 1:
 *                           0 (default) one -- the vector A^T u and ||u||^2 are
 *                           reduced together (lazy normalisation);
 *                           1 two -- ||u||^2 first, then the vector, the
 *                           synchronisation count of textbook LSQR that the paper
 *                           compares CS against.
 *   LSRN_OPT_BCAST_N        nranks > 1: 1 (default) rank 0 computes the SVD and
 *                           broadcasts sigma and N to every rank (the paper's
 *                           MPI_Bcast), so all ranks iterate with the same
 *                           N bit for bit; 0: every rank computes the SVD itself.
 * Kernel-plan overrides (testing / tuning; -1 = the planner's shape-based
 * choice).  Each selects among kernels computing the same quantities (results
 * may differ by summation order only):
 *   LSRN_OPT_SKETCH_KERNEL  0 warp-specialized DMMA kernel, 1 non-specialized kernel
 *   LSRN_OPT_SKETCH_TILE    0: 64 x 256 tile, 1: 32 x 512 tile (default)
 *   LSRN_OPT_SKETCH_MAXCL   cap on the G-sharing cluster size
 *   LSRN_OPT_SKETCH_NSPLIT  split-K factor of the dense sketch (>= 1)
 *   LSRN_OPT_SKETCH_X_L2    1: X tiles of the dense sketch loaded with an L2 evict_last policy
 *   LSRN_OPT_SKETCH_CHUNKS  dense sketch of a device-resident A: number of row chunks
 *                           launched in stream order (default: one per 4 GB of A, <= 16)
 *   LSRN_OPT_SKETCH_G       dense sketch: -1 (default) each launch first writes its G tiles
 *                           once into a workspace buffer of <= 8 GB and the DMMA kernel streams
 *                           them; 0 G generated in registers by every CTA that needs it, never
 *                           stored; N > 0 stored with an N-MB budget (same G values either way)
 *   LSRN_OPT_ROWPASS_*      row-pass plan fields; _PF: L2 prefetch distance
 *   LSRN_OPT_CSR_ROWDOT     CSR long pass: 0 heavy-dense + light-CSR, 8 rows per step;
 *                           1 warp per row over the full CSR; 2 as 0 with 2 rows per step;
 *                           3 the two-kernel form (row dots, then A^T u gathered from the
 *                           CSC copy) also for k <= 2048
 *   LSRN_OPT_CSR_SKETCH     CSR sketch: 0 column-stationary light part, G regenerated per
 *                           nonzero; 1 generate-once row-stationary slab;
 *                           2 (default) G generated once per chunk of rows (<= 8 GB, or the
 *                           LSRN_OPT_SKETCH_G budget) and read by the heavy and light kernels
 *   LSRN_OPT_CSR_HEAVY_FMA  stored-G heavy block: 1 = FP64-FMA kernel instead of the DMMA GEMM
 *   LSRN_OPT_CSR_ALL        CSR single pass (k <= 2048): 0 one pair of rows in flight per warp
 *                           (round 1); 6 a register load pipeline of 8-row groups, one group
 *                           in flight; 10 (default) the same with t in shared memory
 *   LSRN_OPT_CSR_LIGHT      stored-G light sketch kernel: 10 * (columns per CTA, 1-64) +
 *                           (gathers in flight per thread: 2, 4 or 8) */
enum {
  LSRN_OPT_PROFILING = 1,
  LSRN_OPT_SVD = 2,
  LSRN_OPT_GRAPH_REUSE = 3,
  LSRN_OPT_HOSTIO_CHUNK_MB = 4,
  LSRN_OPT_LSQR_SYNC = 5,
  LSRN_OPT_BCAST_N = 6,
  LSRN_OPT_SKETCH_KERNEL = 100,
  LSRN_OPT_SKETCH_TILE = 101,
  LSRN_OPT_SKETCH_MAXCL = 102,
  LSRN_OPT_SKETCH_NSPLIT = 103,
  LSRN_OPT_SKETCH_X_L2 = 104,
  LSRN_OPT_SKETCH_CHUNKS = 105,
  LSRN_OPT_SKETCH_G = 106,
  LSRN_OPT_ROWPASS_KEEP = 110,
  LSRN_OPT_ROWPASS_OCC = 111,
  LSRN_OPT_ROWPASS_WIDE1 = 112,
  LSRN_OPT_ROWPASS_WIDE2 = 113,
  LSRN_OPT_ROWPASS_ASYNCX = 114,
  LSRN_OPT_ROWPASS_NT = 115,
  LSRN_OPT_ROWPASS_TR = 116,
  LSRN_OPT_ROWPASS_BUDGET_KB = 117,
  LSRN_OPT_ROWPASS_WIDE_SLICE = 118,
  LSRN_OPT_ROWPASS_PF = 119,
  LSRN_OPT_CSR_ROWDOT = 120,
  LSRN_OPT_CSR_SKETCH = 121,
  LSRN_OPT_CSR_HEAVY_FMA = 123,
  LSRN_OPT_CSR_ALL = 124,
  LSRN_OPT_CSR_LIGHT = 126
};
enum { LSRN_SVD_AUTO = 0, LSRN_SVD_JW = 1, LSRN_SVD_GESVD = 2, LSRN_SVD_POLAR = 3, LSRN_SVD_QR = 4 };
lsrn_status lsrn_ctx_set_option(lsrn_ctx* ctx, int option, int64_t value);

/* Host-staged collectives for nranks > 1 without NCCL (any host transport: MPI,
 * gloo, ... -- the paper's own cluster runs used MPI).  The library
 * synchronises its stream, copies the operand to host memory, calls the
 * callback and copies the result back:
 *   allreduce(user, buf, count): in-place elementwise sum of buf[0..count) over
 *     all ranks (every rank calls it in the same order with the same count);
 *   bcast(user, buf, count, root): buf[0..count) of rank `root` to every rank.
 * Callbacks return 0 on success (non-zero -> LSRN_ENCCL).  With host
 * collectives the iteration loop is launched eagerly (a CUDA graph cannot hold
 * the host round trips).  Only used when the context has no NCCL communicator. */
typedef int (*lsrn_host_allreduce_fn)(void* user, double* buf, int64_t count);
typedef int (*lsrn_host_bcast_fn)(void* user, double* buf, int64_t count, int root);
lsrn_status lsrn_ctx_set_host_collectives(lsrn_ctx* ctx, lsrn_host_allreduce_fn allreduce, lsrn_host_bcast_fn bcast,
                                          void* user);

/* Record CUDA events around every long-pass (K6) launch of the next solves so
 * lsrn_last_stats reports its average duration (adds event nodes to the graph). */
lsrn_status lsrn_ctx_set_profiling(lsrn_ctx* ctx, int on);

/* Bytes of device workspace needed by lsrn_sketch / lsrn_solve_* for this
 * matrix shard and options (includes host-IO staging when LSRN_HOST_IO). */
lsrn_status lsrn_workspace_size(lsrn_ctx* ctx, const lsrn_matrix* A, const lsrn_opts* opts,
                                size_t* bytes);

/* Alg. 1/2 step 3 + §5 blocks, in the tall form:
 *   At = sigma_X * G[:, 0:L] X + sigma_I * G[:, L:L+k]              (s x k, row-major)
 * with (sigma_X, sigma_I) = (1, lambda) if m >= n, (1/lambda, 1) if m < n and
 * lambda > 0, (1, 0) if lambda == 0; G[i, j] = Box-Muller(Philox4x32-10(seed;
 * i >> 1, j, 0)) generated in registers, never stored (§8(c) C9).  For m < n
 * the paper's Ã = A G (m x s) is At^T.  With nranks > 1 the result is the
 * allreduced (global) sketch on every rank.  s_out receives s = ceil(gamma k).
 * At must hold s * k doubles (device). */
lsrn_status lsrn_sketch(lsrn_ctx* ctx, const lsrn_matrix* A, double gamma, double lambda,
                        uint64_t seed, void* ws, size_t ws_bytes, double* At, int64_t* s_out);

/* Full LSRN solve (Alg. 1 or 2, §5 when lambda > 0) with LSQR (Paige &
 * Saunders 1982, cited P:107-109) on the preconditioned system.  Sketch ->
 * SVD (cuSOLVER, outside the hot path, timed in t_svd) -> N = V_r Sigma_r^-1 ->
 * fused single-pass iterations captured in one CUDA graph -> x.
 *   b : length cnt (tall, rank's rows) or m (wide, replicated);
 *   x : length n (tall, replicated) or cnt (wide, rank's columns).
 * b = 0 gives x = 0 and iters = 0. */
lsrn_status lsrn_solve_lsqr(lsrn_ctx* ctx, const lsrn_matrix* A, const double* b,
                            const lsrn_opts* opts, void* ws, size_t ws_bytes, double* x,
                            lsrn_report* report);

/* Same with the Chebyshev semi-iterative method, Alg. 3 with the
 * k = 1 step 1/(d - c^2/(2d)) (§8(c) C1) and K + 1 passes (§8(c) C2) from the
 * Thm 4.4 bounds. */
lsrn_status lsrn_solve_cs(lsrn_ctx* ctx, const lsrn_matrix* A, const double* b,
                          const lsrn_opts* opts, void* ws, size_t ws_bytes, double* x,
                          lsrn_report* report);

enum { LSRN_SOLVER_LSQR = 0, LSRN_SOLVER_CS = 1 };

/* Oversampling choice (NEXT-4), §6.3: "initialize LSRN by measuring
 * randn/sec and flops/sec ... and then determine the best value of gamma by
 * minimizing the total running time".  Host-only (no device work).  The rates
 * come from a probe solve's report (any gamma): for s = ceil(gamma k),
 * k = min(m, n),
 *   T(gamma) = t_sketch s / s0                                (randn + mult, linear in s)
 *            + t_svd (2 s k^2 + 11 k^3) / (2 s0 k^2 + 11 k^3)  (SVD cost)
 *            + t_iter / it0 * it(s)                           (it = Thm 4.5 LSQR count or
 *                                                              Alg. 3 K + 1 passes, P:643, P:694,
 *                                                              at the probe's rank r, alpha = 1/sqrt(s))
 * minimised over gamma on a 0.01 grid of [gamma_lo, gamma_hi] (s > r required).
 * probe: a report filled by lsrn_solve_lsqr / _cs for the same (m, n) and
 * solver (iters > 0); solver: LSRN_SOLVER_LSQR or _CS.  Returns LSRN_EINVAL on
 * an unusable probe or range; *gamma_out and (optional) *t_out = the model's
 * time at the choice. */
lsrn_status lsrn_choose_gamma(const lsrn_report* probe, int64_t m, int64_t n, double tol, int solver,
                              double gamma_lo, double gamma_hi, double* gamma_out, double* t_out);

/* Testing aid (K1 parity): out[t] = G[rows[t], cols[t]] for t < count
 * (rows/cols/out device arrays), the in-kernel Philox + Box-Muller. */
lsrn_status lsrn_debug_gaussian(lsrn_ctx* ctx, uint64_t seed, const int64_t* rows,
                                const int64_t* cols, int64_t count, double* out);

/* Testing aid (K1 parity on chosen Philox outputs): for t < count, the
 * Box-Muller pair (z0, z1) of the four 32-bit Philox words words[4t .. 4t+3]
 * (w0 = words[4t] | words[4t+1] << 32, w1 = words[4t+2] | words[4t+3] << 32,
 * §8(c) C9) into out[2t], out[2t+1].  mode 0: the table-driven fp64 transform
 * (CSR sketch, Tikhonov blocks); mode 1: CUDA libm (log, sqrt, sincospi); mode 2:
 * the integer fixed-point transform of the dense sketch.  Device arrays. */
lsrn_status lsrn_debug_box_muller(lsrn_ctx* ctx, const uint32_t* words, int64_t count, int mode, double* out);

/* Testing / tuning aid (K5/K6 parity): one fused row pass of the iterations
 * on a device matrix Y (R x C, row-major, leading
 * dimension ld), with the kernel plan the solver uses for that shape:
 *   z_j <- c1 z_j + c2 sx (Y_j . t);  acc_j += ca z_j (acc nullable);
 *   out[0:C] = sx Y^T z;  out[C] = ||z||^2,
 * coef = {c1, c2, ca} (device, 3 doubles); t (C), z (R), out (C + 1) device.
 * reps > 1 repeats the pass (z, acc updated each time) and, with ms_out, returns
 * the kernel time of the last repetition (CUDA events).  Allocates its scratch
 * with cudaMallocAsync on the context stream. */
lsrn_status lsrn_debug_rowpass(lsrn_ctx* ctx, const double* Y, int64_t R, int64_t C, int64_t ld, const double* t,
                               const double* coef, double sx, double* z, double* acc, double* out, int reps,
                               double* ms_out);

/* Kernel statistics of the last lsrn_sketch / lsrn_solve_* call on ctx:
 * CUDA-event durations (ms) of the dominant kernels, averaged per launch, and
 * the number of kernel launches.  Fills up to `cap` doubles:
 *  [0] sketch stage ms, [1] long-pass kernel ms (avg/launch, needs profiling),
 *  [2] reserved, [3] kernel launches of the last call, [4] long-pass launches
 *  timed, [5] algorithmic bytes of A per long pass, [6] sketch flops
 *  (2 s k L_local), [7] kernel launches inside the iteration graph. */
lsrn_status lsrn_last_stats(lsrn_ctx* ctx, double* out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* LSRN_H */
