// score.cuh -- per-instance planner scoring shared by the stand-alone scoring
// kernel (ops.cu: k_score) and the fused epilogue of the persistent AM kernel.
//
// planner.py:412-423 (sample_plan: v = |(xdot, ydot)| unclipped), :219-245
// (collision ratios recomputed from positions, heading / residual / collision
// filters), :210-216 (cruise and highspeed meta costs).  Every basic operation
// is an explicit IEEE-rounded intrinsic, so both call sites produce the same
// bits whatever their -fmad setting.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace bmpc {

struct ScoreParams {
  int n, m, kind;  // kind 0 cruise, 1 highspeed
  double a, b, v_cruise, v_max, y_rl, w1, w2;
  double heading_limit, residual_tol, ratio_min;
};

// Warp-cooperative: lane handles samples k = lane, lane+32, ...; `sample(k, x,
// y, v, psi)` provides sample k (v = |(xdot, ydot)|).  Returns (on every lane)
// the meta cost, min ratio, max |psi| and the filter bits (bit0 heading, bit1
// residual, bit2 collision) given the instance's final block residuals.
template <class SampleFn>
__device__ __forceinline__ void score_samples(const ScoreParams& S, const double2* __restrict__ xi,
                                              SampleFn sample, double r0, double r1, double r2,
                                              double& cost_out, double& rmin_out,
                                              double& hmax_out, unsigned char& flags_out) {
  const int lane = threadIdx.x & 31;
  double hmax = 0.0, rmin = INFINITY, cost = 0.0;
  bool any_nan = false;
  for (int k = lane; k < S.n; k += 32) {
    double x, y, v, ps;
    sample(k, x, y, v, ps);
    const double ah = fabs(ps);
    if (ah != ah) any_nan = true;
    hmax = fmax(hmax, ah);
    // ratio^2 (a b)^2 = (b (x - qx))^2 + (a (y - qy))^2: no division per term
    // (the sweep's outside test); the one division and square root come after
    // the minimum
#pragma unroll 4
    for (int j = 0; j < S.m; ++j) {
      const double2 q = __ldg(xi + j * S.n + k);
      const double px = __dmul_rn(S.b, __dsub_rn(x, q.x)), py = __dmul_rn(S.a, __dsub_rn(y, q.y));
      rmin = fmin(rmin, __fma_rn(px, px, __dmul_rn(py, py)));
    }
    if (S.kind == 0) {
      const double dv = __dsub_rn(v, S.v_cruise);
      cost = __dadd_rn(cost, __dmul_rn(dv, dv));
    } else {
      const double dv = __dsub_rn(v, S.v_max), dy = __dsub_rn(y, S.y_rl);
      cost = __dadd_rn(cost, __dadd_rn(__dmul_rn(S.w1, __dmul_rn(dv, dv)),
                                       __dmul_rn(S.w2, __dmul_rn(dy, dy))));
    }
  }
  hmax = warp_max(hmax);
  rmin = __ddiv_rn(__dsqrt_rn(warp_min(rmin)), __dmul_rn(S.a, S.b));
  cost = warp_sum(cost);
  if (__any_sync(BMPC_FULL, any_nan)) hmax = NAN;  // np.abs(psi).max() propagates NaN
  const double rmax = (r0 != r0 || r1 != r1 || r2 != r2) ? NAN : fmax(r0, fmax(r1, r2));
  unsigned char f = 0;
  if (hmax <= S.heading_limit) f |= 1;
  if (rmax <= S.residual_tol) f |= 2;
  if (rmin >= S.ratio_min) f |= 4;
  cost_out = cost;
  rmin_out = rmin;
  hmax_out = hmax;
  flags_out = f;
}

// As score_samples, with `sample(k, x, y, xd, yd, psi)` evaluating the basis:
// v = sqrt(xd^2 + yd^2) unclipped (planner.py:412-423).
template <class SampleFn>
__device__ __forceinline__ void score_instance(const ScoreParams& S, const double2* __restrict__ xi,
                                               SampleFn sample, double r0, double r1, double r2,
                                               double& cost_out, double& rmin_out,
                                               double& hmax_out, unsigned char& flags_out) {
  auto sv = [&](int k, double& x, double& y, double& v, double& ps) {
    double xd, yd;
    sample(k, x, y, xd, yd, ps);
    v = __dsqrt_rn(__dadd_rn(__dmul_rn(xd, xd), __dmul_rn(yd, yd)));
  };
  score_samples(S, xi, sv, r0, r1, r2, cost_out, rmin_out, hmax_out, flags_out);
}

}  // namespace bmpc
