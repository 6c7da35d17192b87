// steps.cu -- device kernels behind the step-wise solver API
// (BatchSolver.step_xy / step_psi / step_d_obs / update_multipliers /
// compute_residuals, reference solver.py:288-410).  Not on the timed path:
// one thread per instance column, coalesced over the (rows, L) layout.
#include <cuda_runtime.h>

#include "am_args.h"
#include "common.cuh"

namespace bmpc {

// out (nb, L) = F_axis^T g for g (m*n + 2n, L) (mode 0: rows [obstacles; accel;
// nonholonomic] against [P; Pddot; Pdot], obstacle-sum-first), or P^T g for
// g (n, L) (mode 1).
__global__ void k_project(int mode, int n, int npad, int nb, int m, long long L,
                          const double* __restrict__ PT, const double* __restrict__ g,
                          double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)nb * L) return;
  const int i = (int)(e / L);
  const long long c = e - (long long)i * L;
  const double* P = PT + (size_t)i * npad;
  const double* Pd = PT + (size_t)(nb + i) * npad;
  const double* Pdd = PT + (size_t)(2 * nb + i) * npad;
  double acc = 0.0;
  if (mode == 1) {
    for (int k = 0; k < n; ++k) acc = fma(P[k], g[(long long)k * L + c], acc);
  } else {
    const long long mn = (long long)m * n;
    for (int k = 0; k < n; ++k) {
      double gs = 0.0;
      for (int j = 0; j < m; ++j) gs += g[((long long)j * n + k) * L + c];
      acc = fma(P[k], gs, acc);
      acc = fma(Pdd[k], g[(mn + k) * L + c], acc);
      acc = fma(Pd[k], g[(mn + n + k) * L + c], acc);
    }
  }
  out[e] = acc;
}

// Refined KKT apply per column (solver.py:164-176): [c; mu] = K^-1 rhs, one
// refinement step against K; writes the nb coefficient rows.  which 0: the xy
// system, rhs (2nb+12, L) = [x rows; y rows; b_x (6); b_y (6)]; which 1: psi,
// rhs (nb+4, L).
__global__ void k_kkt_apply(int which, int nb, long long L, const double* __restrict__ Kf,
                            const double* __restrict__ Ka, int ks, const double* __restrict__ rhs,
                            double* __restrict__ out_x, double* __restrict__ out_y) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L) return;
  const int R = which == 0 ? nb + 6 : nb + 4;
  const int naxes = which == 0 ? 2 : 1;
  double r[22], s[22], q[22];
  for (int ax = 0; ax < naxes; ++ax) {
    for (int row = 0; row < R; ++row) {
      int src;
      if (which == 0) src = row < nb ? ax * nb + row : 2 * nb + 6 * ax + (row - nb);
      else src = row;
      r[row] = rhs[(long long)src * L + c];
    }
    for (int row = 0; row < R; ++row) {
      double a = 0.0;
      for (int j = 0; j < R; ++j) a = fma(Kf[row * ks + j], r[j], a);
      s[row] = a;
    }
    for (int row = 0; row < R; ++row) {
      double a = 0.0;
      for (int j = 0; j < R; ++j) a = fma(Ka[row * ks + j], s[j], a);
      q[row] = r[row] - a;
    }
    double* out = ax == 0 ? out_x : out_y;
    for (int row = 0; row < nb; ++row) {
      double a = 0.0;
      for (int j = 0; j < R; ++j) a = fma(Kf[row * ks + j], q[j], a);
      out[(long long)row * L + c] = s[row] + a;
    }
  }
}

// theta (n, L) = unwrap(atan2(Pdot c_y, Pdot c_x), axis=0) (solver.py:316-318),
// numpy's unwrap semantics exactly.
__global__ void k_heading(int n, int npad, int nb, long long L, const double* __restrict__ PT,
                          const double* __restrict__ c_x, const double* __restrict__ c_y,
                          double* __restrict__ theta) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L) return;
  const double* Pd = PT + (size_t)nb * npad;
  const double period = 6.283185307179586, hi = period / 2.0;
  double cum = 0.0, prev = 0.0;
  for (int k = 0; k < n; ++k) {
    double xd = 0.0, yd = 0.0;
    for (int i = 0; i < nb; ++i) {
      xd = fma(Pd[i * npad + k], c_x[(long long)i * L + c], xd);
      yd = fma(Pd[i * npad + k], c_y[(long long)i * L + c], yd);
    }
    const double p = atan2(yd, xd);
    if (k > 0) {
      const double dd = p - prev;
      double ddmod = np_mod(dd - (-hi), period) + (-hi);
      if (ddmod == -hi && dd > 0.0) ddmod = hi;
      double ph = ddmod - dd;
      if (fabs(dd) < hi) ph = 0.0;
      cum = cum + ph;
      theta[(long long)k * L + c] = p + cum;
    } else {
      theta[c] = p;
    }
    prev = p;
  }
}

// d-step given alpha (solver.py:342-354): d = max(1, num/den).
__global__ void k_d_obs(int n, long long l, long long mn, const double* __restrict__ x,
                        const double* __restrict__ y, const double* __restrict__ xi_x,
                        const double* __restrict__ xi_y, const double* __restrict__ alpha,
                        double a, double b, double* __restrict__ d) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= mn * l) return;
  const long long row = e / l, c = e - row * l;
  const long long k = row % n;
  const double wx = __dsub_rn(x[k * l + c], xi_x[row]);
  const double wy = __dsub_rn(y[k * l + c], xi_y[row]);
  const double ca = cos(alpha[e]), sa = sin(alpha[e]);
  const double num = __dadd_rn(__dmul_rn(__dmul_rn(a, ca), wx), __dmul_rn(__dmul_rn(b, sa), wy));
  const double den = __dadd_rn(__dmul_rn(__dmul_rn(a, ca), __dmul_rn(a, ca)),
                               __dmul_rn(__dmul_rn(b, sa), __dmul_rn(b, sa)));
  const double q = num / den;
  d[e] = q < 1.0 ? 1.0 : q;  // np.maximum(1.0, q), NaN propagates
}

// Block norms of the residual vectors (solver.py:396-410): out (3, l).
__global__ void k_block_norms(int n, long long l, long long mn, const double* __restrict__ r_x,
                              const double* __restrict__ r_y, double* __restrict__ out) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= l) return;
  const long long bounds[4] = {0, mn, mn + n, mn + 2LL * n};
  for (int blk = 0; blk < 3; ++blk) {
    double sx = 0.0, sy = 0.0;
    for (long long row = bounds[blk]; row < bounds[blk + 1]; ++row) {
      const double vx = r_x[row * l + c], vy = r_y[row * l + c];
      sx = fma(vx, vx, sx);
      sy = fma(vy, vy, sy);
    }
    out[blk * l + c] = sqrt(sx + sy);
  }
}

// Ellipse separation ratios recomputed from positions (planner.py:219-230):
// out (m*n, l), row j*n + k = sqrt(((x_k - xi_x)/a)^2 + ((y_k - xi_y)/b)^2), every
// operation rounded on its own as numpy does (no contraction).
__global__ void k_collision_ratios(int n, long long l, long long mn, const double* __restrict__ x,
                                   const double* __restrict__ y, const double* __restrict__ xi_x,
                                   const double* __restrict__ xi_y, double a, double b,
                                   double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= mn * l) return;
  const long long row = e / l, c = e - row * l;
  const long long k = row % n;
  const double wx = __ddiv_rn(__dsub_rn(x[k * l + c], xi_x[row]), a);
  const double wy = __ddiv_rn(__dsub_rn(y[k * l + c], xi_y[row]), b);
  out[e] = __dsqrt_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)));
}

static inline int blocks_for(long long n, int tb) { return (int)((n + tb - 1) / tb); }

cudaError_t op_project(const bmpc_dev_consts& C, int mode, int m, long long L, const double* g,
                       double* out, cudaStream_t st) {
  const long long tot = (long long)C.nb * L;
  if (tot > 0)
    k_project<<<blocks_for(tot, 128), 128, 0, st>>>(mode, C.n, C.npad, C.nb, m, L, C.PT, g, out);
  return cudaGetLastError();
}
cudaError_t op_kkt_apply(const bmpc_dev_consts& C, int which, long long L, const double* rhs,
                         double* out_x, double* out_y, cudaStream_t st) {
  if (L > 0) {
    if (which == 0)
      k_kkt_apply<<<blocks_for(L, 128), 128, 0, st>>>(0, C.nb, L, C.Kxf, C.Kxa, C.kxs, rhs, out_x, out_y);
    else
      k_kkt_apply<<<blocks_for(L, 128), 128, 0, st>>>(1, C.nb, L, C.Kpf, C.Kpa, C.kps, rhs, out_x, nullptr);
  }
  return cudaGetLastError();
}
cudaError_t op_heading(const bmpc_dev_consts& C, long long L, const double* c_x, const double* c_y,
                       double* theta, cudaStream_t st) {
  if (L > 0) k_heading<<<blocks_for(L, 128), 128, 0, st>>>(C.n, C.npad, C.nb, L, C.PT, c_x, c_y, theta);
  return cudaGetLastError();
}
cudaError_t op_d_obs(int n, long long l, long long mn, const double* x, const double* y,
                     const double* xi_x, const double* xi_y, const double* alpha, double a,
                     double b, double* d, cudaStream_t st) {
  if (mn * l > 0)
    k_d_obs<<<blocks_for(mn * l, 256), 256, 0, st>>>(n, l, mn, x, y, xi_x, xi_y, alpha, a, b, d);
  return cudaGetLastError();
}
cudaError_t op_collision_ratios(int n, long long l, long long mn, const double* x, const double* y,
                                const double* xi_x, const double* xi_y, double a, double b,
                                double* out, cudaStream_t st) {
  if (mn * l > 0)
    k_collision_ratios<<<blocks_for(mn * l, 256), 256, 0, st>>>(n, l, mn, x, y, xi_x, xi_y, a, b, out);
  return cudaGetLastError();
}
cudaError_t op_block_norms(int n, long long l, long long mn, const double* r_x, const double* r_y,
                           double* out, cudaStream_t st) {
  if (l > 0) k_block_norms<<<blocks_for(l, 128), 128, 0, st>>>(n, l, mn, r_x, r_y, out);
  return cudaGetLastError();
}

}  // namespace bmpc
