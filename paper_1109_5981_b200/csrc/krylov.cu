// K8: LSQR scalar recurrences and the y / w_y update, on the device.
//
// LSQR (Paige & Saunders 1982, cited at P:107-109), applied to Abar = A N
// (Alg. 1) or Abar = M^T A (Alg. 2).  Vectors are kept
// un-normalised ("lazy" scales su, sv: u_i = su * u_store, v_i = sv * v_store)
// so that each Golub-Kahan half-step is ONE fused pass (rowpass.cu):
//   U pass:  u_store <- (-alpha su) u_store + sv * Abar v_store    -> beta^2
//   V pass:  v_store <- (-beta sv) v_store + su * Abar^T u_store  -> alpha^2
// followed by the Givens rotation and
//   y <- y + (phi / rho) w_y ;  w_y <- sv v_store - (theta / rho) w_y.
// The scalars never leave the GPU: the loop has no host synchronisation and is
// captured once as a CUDA graph.  Termination (exact breakdown alpha or beta = 0,
// or the adaptive Paige-Saunders tests of DESIGN.md reading C5) sets `done`,
// which turns every remaining kernel of the graph into a no-op.
#include "common.cuh"
#include "kernels.h"

namespace lsrn {

__global__ void lsqr_init_state_kernel(LsqrState* s, double tol, int adaptive) {
  LsqrState z = {};
  z.tol = tol;
  z.adaptive = adaptive;
  z.converged = adaptive ? 0 : 1;
  *s = z;
}

cudaError_t launch_lsqr_init_state(LsqrState* st_dev, double tol, int adaptive, cudaStream_t st) {
  lsqr_init_state_kernel<<<1, 1, 0, st>>>(st_dev, tol, adaptive);
  return cudaGetLastError();
}

// comm[C] holds ||u_store||^2 after the U pass.
__global__ void lsqr_after_u_kernel(LsqrState* s, const double* comm, int64_t C, int phase) {
  if (s->done) return;
  const double beta = sqrt(comm[C]);
  if (phase == 0) {
    s->bnorm = beta;
    s->phibar = beta;
    s->rnorm = beta;
    if (beta == 0.0) {        // b = 0 (or M^T b = 0): x = 0, no iterations
      s->done = 1;
      s->converged = 1;
      return;
    }
    s->beta = beta;
    s->su = 1.0 / beta;
    s->cV[0] = 0.0;           // v_1 = Abar^T u_1 (no previous v)
    s->cV[1] = s->su;
    s->cV[2] = 0.0;
    return;
  }
  s->anorm2 += s->alpha * s->alpha + beta * beta;
  const double su_new = (beta > 0.0) ? 1.0 / beta : 0.0;
  s->cV[0] = -beta * s->sv;
  s->cV[1] = su_new;
  s->cV[2] = 0.0;
  s->beta = beta;
  s->su = su_new;
  if (beta == 0.0) s->stop_after = 1;
}

// Scalar part of the V step; every block recomputes it (deterministically) and
// block 0 publishes the new state.  Then the vector update on this block's slice.
__global__ void lsqr_after_v_kernel(LsqrState* s, const double* comm, int64_t C, int phase, double* y,
                                    double* wy, const double* vstore, int64_t n, double* ypart,
                                    unsigned* counter) {
  __shared__ double sh[8];
  __shared__ bool last;
  if (s->done) return;
  const double alpha = sqrt(comm[C]);
  const double sv_new = (alpha > 0.0) ? 1.0 / alpha : 0.0;
  if (phase == 0) {
    // w_1 = v_1, y_0 = 0, rhobar_1 = alpha_1
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      wy[i] = sv_new * vstore[i];
      y[i] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s->alpha = alpha;
      s->sv = sv_new;
      s->rhobar = alpha;
      if (alpha == 0.0) {     // A^T b = 0: y = 0 is the solution
        s->done = 1;
        s->converged = 1;
        s->arnorm = 0.0;
        return;
      }
      s->cU[0] = -alpha * s->su;
      s->cU[1] = sv_new;
      s->cU[2] = 0.0;
    }
    return;
  }
  const double beta = s->beta;
  const double rho = hypot(s->rhobar, beta);
  const double c = s->rhobar / rho;
  const double sn = beta / rho;
  const double theta = sn * alpha;
  const double phi = c * s->phibar;
  const double phibar = sn * s->phibar;
  const double phi_rho = phi / rho;
  const double theta_rho = theta / rho;
  double yn = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double w = wy[i];
    const double yi = fma(phi_rho, w, y[i]);
    y[i] = yi;
    wy[i] = fma(-theta_rho, w, sv_new * vstore[i]);
    yn = fma(yi, yi, yn);
  }
  double t = warp_sum(yn);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += sh[w];
    ypart[blockIdx.x] = b;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!(last && threadIdx.x < 32)) return;
  __threadfence();
  const double ynorm2 = warp_sum_l2(ypart, gridDim.x);
  if (threadIdx.x != 0) return;
  *counter = 0u;
  // publish the new scalars (single writer)
  s->alpha = alpha;
  s->sv = sv_new;
  s->rhobar = -c * alpha;
  s->phibar = phibar;
  s->phi_rho = phi_rho;
  s->theta_rho = theta_rho;
  s->rnorm = phibar;
  s->arnorm = phibar * alpha * fabs(c);
  s->iters += 1;
  s->cU[0] = -alpha * s->su;
  s->cU[1] = sv_new;
  s->cU[2] = 0.0;
  if (alpha == 0.0 || s->stop_after) {     // bidiagonalisation terminated: y exact
    s->done = 1;
    s->converged = 1;
    return;
  }
  if (s->adaptive) {
    const double anorm = sqrt(s->anorm2);
    const double tol = s->tol;
    if (s->rnorm <= tol * s->bnorm + tol * anorm * sqrt(ynorm2) || s->arnorm <= tol * anorm * s->rnorm) {
      s->done = 1;
      s->converged = 1;
    }
  }
}

int lsqr_update_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 296) b = 296;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_lsqr_after_u(LsqrState* s, const double* comm, int64_t C, int phase, cudaStream_t st) {
  lsqr_after_u_kernel<<<1, 1, 0, st>>>(s, comm, C, phase);
  return cudaGetLastError();
}

cudaError_t launch_lsqr_after_v(LsqrState* s, const double* comm, int64_t C, int phase, double* y, double* wy,
                                const double* vstore, int64_t n, double* ypart, unsigned* counter,
                                cudaStream_t st) {
  lsqr_after_v_kernel<<<lsqr_update_blocks(n), 256, 0, st>>>(s, comm, C, phase, y, wy, vstore, n, ypart,
                                                             counter);
  return cudaGetLastError();
}

}  // namespace lsrn
