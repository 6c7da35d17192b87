// ops.cu -- operator-level sm_100a kernels behind the reference's `kernels`
// plugin API (/root/reference/pkg/src/batchmpc/kernels/__init__.py:49-86), plus
// the scoring / argmin / sampling kernels of the planner path.
//
// Compiled with -fmad=false: every basic double operation is an IEEE-rounded
// add/mul exactly as in the reference's scalar C (Cython, -O3 without FMA), and
// sqrt / division are the correctly-rounded CUDA defaults, so these kernels
// agree with the reference to the last bit except where libm's and CUDA's
// atan2/sin/cos differ by an ulp.
//
// Layouts are the reference's: (rows, l) row-major with the instance index
// fastest; obstacle rows j*n + k.
#include <cuda_runtime.h>
#include <stdint.h>

#include "am_args.h"
#include "common.cuh"
#include "score.cuh"

namespace bmpc {

constexpr int kTB = 256;
static inline int nblk(long long total) { return (int)((total + kTB - 1) / kTB); }

// ---------------------------------------------------------------- op kernels --
// _speedups.pyx:12-39
__global__ void k_obstacle_update(int n, int l, long long mn, const double* __restrict__ x,
                                  const double* __restrict__ y, const double* __restrict__ xi_x,
                                  const double* __restrict__ xi_y, double a, double b,
                                  double* __restrict__ alpha, double* __restrict__ d) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= mn * l) return;
  const long long row = e / l;
  const int c = (int)(e - row * l);
  const int k = (int)(row % n);
  const double wx = x[(long long)k * l + c] - xi_x[row];
  const double wy = y[(long long)k * l + c] - xi_y[row];
  const double al = atan2(a * wy, b * wx);
  const double ca = cos(al), sa = sin(al);
  const double num = a * ca * wx + b * sa * wy;
  const double den = (a * ca) * (a * ca) + (b * sa) * (b * sa);
  double dd = num / den;
  if (dd < 1.0) dd = 1.0;
  alpha[e] = al;
  d[e] = dd;
}

// _speedups.pyx:42-60
__global__ void k_accel_update(long long nl, const double* __restrict__ xdd,
                               const double* __restrict__ ydd, double a_max,
                               double* __restrict__ alpha_a, double* __restrict__ d_a) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nl) return;
  const double ax = xdd[e], ay = ydd[e];
  alpha_a[e] = atan2(ay, ax);
  double mag = sqrt(ax * ax + ay * ay);
  if (mag > a_max) mag = a_max;
  d_a[e] = mag;
}

// _speedups.pyx:63-78
__global__ void k_v_update(long long nl, const double* __restrict__ xd,
                           const double* __restrict__ yd, double v_min, double v_max,
                           double* __restrict__ v) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nl) return;
  double s = sqrt(xd[e] * xd[e] + yd[e] * yd[e]);
  if (s < v_min) s = v_min;
  else if (s > v_max) s = v_max;
  v[e] = s;
}

// _speedups.pyx:81-111
__global__ void k_assemble_g(int n, int l, long long mn, const double* __restrict__ xi_x,
                             const double* __restrict__ xi_y, const double* __restrict__ alpha,
                             const double* __restrict__ d, const double* __restrict__ alpha_a,
                             const double* __restrict__ d_a, const double* __restrict__ v,
                             const double* __restrict__ psi, double a, double b,
                             double* __restrict__ g_x, double* __restrict__ g_y) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long rows = mn + 2LL * n;
  if (e >= rows * l) return;
  const long long row = e / l;
  const long long c = e - row * l;
  if (row < mn) {
    const double ang = alpha[e], ad = d[e];
    g_x[e] = xi_x[row] + a * ad * cos(ang);
    g_y[e] = xi_y[row] + b * ad * sin(ang);
  } else if (row < mn + n) {
    const long long s = (row - mn) * l + c;
    g_x[e] = d_a[s] * cos(alpha_a[s]);
    g_y[e] = d_a[s] * sin(alpha_a[s]);
  } else {
    const long long s = (row - mn - n) * l + c;
    g_x[e] = v[s] * cos(psi[s]);
    g_y[e] = v[s] * sin(psi[s]);
  }
}

// _speedups.pyx:321-355
__global__ void k_residual_vectors(int n, int l, long long mn, const double* __restrict__ x,
                                   const double* __restrict__ y, const double* __restrict__ xd,
                                   const double* __restrict__ yd, const double* __restrict__ xdd,
                                   const double* __restrict__ ydd, const double* __restrict__ psi,
                                   const double* __restrict__ xi_x, const double* __restrict__ xi_y,
                                   const double* __restrict__ alpha, const double* __restrict__ d,
                                   const double* __restrict__ alpha_a,
                                   const double* __restrict__ d_a, const double* __restrict__ v,
                                   double a, double b, double* __restrict__ r_x,
                                   double* __restrict__ r_y) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long rows = mn + 2LL * n;
  if (e >= rows * l) return;
  const long long row = e / l;
  const long long c = e - row * l;
  if (row < mn) {
    const long long s = (row % n) * l + c;
    const double ang = alpha[e], ad = d[e];
    r_x[e] = x[s] - xi_x[row] - a * ad * cos(ang);
    r_y[e] = y[s] - xi_y[row] - b * ad * sin(ang);
  } else if (row < mn + n) {
    const long long s = (row - mn) * l + c;
    r_x[e] = xdd[s] - d_a[s] * cos(alpha_a[s]);
    r_y[e] = ydd[s] - d_a[s] * sin(alpha_a[s]);
  } else {
    const long long s = (row - mn - n) * l + c;
    r_x[e] = xd[s] - v[s] * cos(psi[s]);
    r_y[e] = yd[s] - v[s] * sin(psi[s]);
  }
}

// _speedups.pyx:114-218 (with_angles=false) and :221-318 (tail_update, with_angles=true).
// One thread per (row, instance) element: rows [0, mn) are the obstacle terms,
// rows [mn, mn + n) sample k of the acceleration and the non-holonomic block.
// Every element's arithmetic is the reference's statement order (compiled with
// -fmad=false); the per-instance squared block sums are taken afterwards by
// k_tail_sums from the stored residuals, walking the rows in the reference's
// order, so they accumulate in the same sequence.
template <bool WITH_ANGLES>
__global__ void k_tail(int n, int l, long long mn, const double* __restrict__ x,
                       const double* __restrict__ y, const double* __restrict__ xd,
                       const double* __restrict__ yd, const double* __restrict__ xdd,
                       const double* __restrict__ ydd, const double* __restrict__ psi,
                       const double* __restrict__ xi_x, const double* __restrict__ xi_y,
                       double v_min, double v_max, double a_max, double a, double b,
                       double* __restrict__ alpha, double* __restrict__ d,
                       double* __restrict__ alpha_a, double* __restrict__ d_a,
                       double* __restrict__ v, double* __restrict__ r_x,
                       double* __restrict__ r_y, double* __restrict__ g_x,
                       double* __restrict__ g_y) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (mn + n) * l) return;
  const long long row = t / l;
  const long long c = t - row * l;
  if (row < mn) {
    const long long k = row % n;
    const long long e = row * l + c;
    const double wx = x[k * l + c] - xi_x[row];
    const double wy = y[k * l + c] - xi_y[row];
    const double px = b * wx, py = a * wy;
    const double r = sqrt(px * px + py * py);
    if (WITH_ANGLES) alpha[e] = atan2(py, px);
    double ca, sa;
    if (r > 0.0) {
      ca = px / r;
      sa = py / r;
    } else {
      ca = 1.0;
      sa = 0.0;
    }
    double dd = r / (a * b);
    if (dd < 1.0) dd = 1.0;
    d[e] = dd;
    const double adca = a * dd * ca, bdsa = b * dd * sa;
    r_x[e] = wx - adca;
    r_y[e] = wy - bdsa;
    g_x[e] = xi_x[row] + adca;
    g_y[e] = xi_y[row] + bdsa;
    return;
  }
  const long long k = row - mn;
  const long long i = k * l + c;
  const double ax = xdd[i], ay = ydd[i];
  const double mag = sqrt(ax * ax + ay * ay);
  if (WITH_ANGLES) alpha_a[i] = atan2(ay, ax);
  double caa, saa;
  if (mag > 0.0) {
    caa = ax / mag;
    saa = ay / mag;
  } else {
    caa = 1.0;
    saa = 0.0;
  }
  const double dd = mag < a_max ? mag : a_max;
  d_a[i] = dd;
  const double daca = dd * caa, dasa = dd * saa;
  const long long ea = (mn + k) * l + c;
  r_x[ea] = ax - daca;
  r_y[ea] = ay - dasa;
  g_x[ea] = daca;
  g_y[ea] = dasa;
  double s = sqrt(xd[i] * xd[i] + yd[i] * yd[i]);
  if (s < v_min) s = v_min;
  else if (s > v_max) s = v_max;
  v[i] = s;
  const double cp = cos(psi[i]), sp = sin(psi[i]);
  const double vcp = s * cp, vsp = s * sp;
  const long long en = (mn + n + k) * l + c;
  r_x[en] = xd[i] - vcp;
  r_y[en] = yd[i] - vsp;
  g_x[en] = vcp;
  g_y[en] = vsp;
}

// Per-instance squared block sums of tail_core (_speedups.pyx:176, :198, :216):
// s += rx rx + ry ry over the block's rows in increasing order, one thread per
// instance column (coalesced across columns).
__global__ void k_tail_sums(int n, int l, long long mn, const double* __restrict__ r_x,
                            const double* __restrict__ r_y, double* __restrict__ sq_obs,
                            double* __restrict__ sq_acc, double* __restrict__ sq_nonhol) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= l) return;
  const int blk = blockIdx.y;  // 0 obstacle, 1 acceleration, 2 non-holonomic rows
  const long long r0 = blk == 0 ? 0 : (blk == 1 ? mn : mn + n);
  const long long r1 = blk == 0 ? mn : (blk == 1 ? mn + n : mn + 2LL * n);
  double s = 0.0;
#pragma unroll 8
  for (long long row = r0; row < r1; ++row) {
    const double rx = r_x[row * l + c], ry = r_y[row * l + c];
    s += rx * rx + ry * ry;
  }
  (blk == 0 ? sq_obs : (blk == 1 ? sq_acc : sq_nonhol))[c] = s;
}

// ------------------------------------------------------------------ sampling --
// (n, L) samples of P c for the planner (planner.py:412-423) and end-of-solve
// materialisation (solver.py:442-450).  PT is the [3][nb][npad] transposed basis.
__global__ void k_sample(int n, int npad, int nb, int L, const double* __restrict__ PT,
                         const double* __restrict__ c_x, const double* __restrict__ c_y,
                         const double* __restrict__ c_psi, double* x, double* y, double* xd,
                         double* yd, double* xdd, double* ydd, double* psi, double* psid,
                         double* v) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * L) return;
  const int k = (int)(e / L);
  const long long c = e - (long long)k * L;
  const double* P = PT;
  const double* Pd = PT + (long long)nb * npad;
  const double* Pdd = PT + 2LL * nb * npad;
  double sx = 0, sy = 0, sxd = 0, syd = 0, sxdd = 0, sydd = 0, sp = 0, spd = 0;
  for (int i = 0; i < nb; ++i) {
    const double p = P[i * npad + k], pd = Pd[i * npad + k], pdd = Pdd[i * npad + k];
    const double cx = c_x ? c_x[(long long)i * L + c] : 0.0;
    const double cy = c_y ? c_y[(long long)i * L + c] : 0.0;
    const double cp = c_psi ? c_psi[(long long)i * L + c] : 0.0;
    sx = __fma_rn(p, cx, sx);
    sy = __fma_rn(p, cy, sy);
    sxd = __fma_rn(pd, cx, sxd);
    syd = __fma_rn(pd, cy, syd);
    sxdd = __fma_rn(pdd, cx, sxdd);
    sydd = __fma_rn(pdd, cy, sydd);
    sp = __fma_rn(p, cp, sp);
    spd = __fma_rn(pd, cp, spd);
  }
  if (x) x[e] = sx;
  if (y) y[e] = sy;
  if (xd) xd[e] = sxd;
  if (yd) yd[e] = syd;
  if (xdd) xdd[e] = sxdd;
  if (ydd) ydd[e] = sydd;
  if (psi) psi[e] = sp;
  if (psid) psid[e] = spd;
  if (v) v[e] = sqrt(sxd * sxd + syd * syd);
}

// ---------------------------------------------------------- fused scoring --
// Warp per instance: sample_plan + collision_ratios + filter_candidates +
// meta_cost (planner.py:210-245, :412-423) straight from the coefficients.
using ScoreArgs = bmpc_score_args;

__global__ void k_score(const ScoreArgs S) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= S.L) return;
  const int inst = warp;
  const double2* xi = reinterpret_cast<const double2*>(S.xi) + (size_t)(inst / S.l) * S.m * S.n;
  const double* P = S.PT;
  const double* Pd = S.PT + (size_t)S.nb * S.npad;
  const ScoreParams sp{S.n, S.m, S.kind, S.a, S.b, S.v_cruise, S.v_max, S.y_rl, S.w1, S.w2,
                       S.heading_limit, S.residual_tol, S.ratio_min};
  auto sample = [&](int k, double& x, double& y, double& xd, double& yd, double& ps) {
    x = y = xd = yd = ps = 0.0;
    for (int i = 0; i < S.nb; ++i) {
      const double p = P[i * S.npad + k], pd = Pd[i * S.npad + k];
      const size_t o = (size_t)i * S.L + inst;
      x = __fma_rn(p, S.c_x[o], x);
      y = __fma_rn(p, S.c_y[o], y);
      xd = __fma_rn(pd, S.c_x[o], xd);
      yd = __fma_rn(pd, S.c_y[o], yd);
      ps = __fma_rn(p, S.c_psi[o], ps);
    }
  };
  double cost, rmin, hmax;
  unsigned char f;
  score_instance(sp, xi, sample, S.res_final[inst], S.res_final[(size_t)S.L + inst],
                 S.res_final[2 * (size_t)S.L + inst], cost, rmin, hmax, f);
  if (lane == 0) {
    S.meta[inst] = cost;
    S.min_ratio[inst] = rmin;
    S.heading_max[inst] = hmax;
    S.flags[inst] = f;
  }
}

// Warp per instance: the same scoring from already-sampled (n, L) arrays --
// the reference-API filter_candidates / rank, which read a RankedPlan's own
// x, y, psi, v (planner.py:219-257).  res: (3, L) block residuals, or null
// (the residual filter bit is then never set).
__global__ void k_score_samples(const ScoreParams sp, int l, int L, const double2* __restrict__ xi,
                                const double* __restrict__ x, const double* __restrict__ y,
                                const double* __restrict__ psi, const double* __restrict__ v,
                                const double* __restrict__ res, double* meta, double* min_ratio,
                                double* heading_max, uint8_t* flags) {
  const int inst = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (inst >= L) return;
  const double2* q = xi + (size_t)(inst / l) * sp.m * sp.n;
  auto sample = [&](int k, double& sx, double& sy, double& sv, double& sps) {
    const size_t e = (size_t)k * L + inst;
    sx = x[e];
    sy = y[e];
    sv = v[e];
    sps = psi[e];
  };
  const double r0 = res ? res[inst] : NAN, r1 = res ? res[(size_t)L + inst] : NAN,
               r2 = res ? res[2 * (size_t)L + inst] : NAN;
  double cost, rmin, hmax;
  unsigned char f;
  score_samples(sp, q, sample, r0, r1, r2, cost, rmin, hmax, f);
  if ((threadIdx.x & 31) == 0) {
    meta[inst] = cost;
    min_ratio[inst] = rmin;
    heading_max[inst] = hmax;
    flags[inst] = f;
  }
}

// ------------------------------------------------------------------ argmin --
// One block per scene: numpy argmin semantics (first minimum; NaN wins) over
// where(mask, cost, inf) for three masks; -1 encodes "None".
__device__ __forceinline__ bool better(double c, long long i, double bc, long long bi) {
  const bool cn = c != c, bn = bc != bc;
  if (bi < 0) return true;
  if (cn || bn) return cn && (!bn || i < bi);
  return c < bc || (c == bc && i < bi);
}

__global__ void k_argmin(int l, const double* __restrict__ meta, const uint8_t* __restrict__ flags,
                         long long* best, long long* best_all, long long* best_hc,
                         long long* nfeas) {
  const int s = blockIdx.x;
  constexpr int kW = 8;  // warps per block (launched with 256 threads)
  __shared__ double sc[3][kW];
  __shared__ long long si[3][kW];
  __shared__ int scount[kW], shc[kW];
  double bc[3] = {INFINITY, INFINITY, INFINITY};
  long long bi[3] = {-1, -1, -1};
  int cnt = 0, cnt_hc = 0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    const long long g = (long long)s * l + i;
    const double c = meta[g];
    const uint8_t f = flags[g];
    const double cf = (f == 7) ? c : INFINITY;
    const double chc = ((f & 5) == 5) ? c : INFINITY;
    cnt += (f == 7);
    cnt_hc += ((f & 5) == 5);
    if (better(cf, i, bc[0], bi[0])) { bc[0] = cf; bi[0] = i; }
    if (better(c, i, bc[1], bi[1])) { bc[1] = c; bi[1] = i; }
    if (better(chc, i, bc[2], bi[2])) { bc[2] = chc; bi[2] = i; }
  }
  // warp tree, then the 8 warp winners (the comparison is order-independent:
  // lexicographic on (cost, index) with numpy's NaN rule)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double oc = __shfl_xor_sync(BMPC_FULL, bc[q], o);
      const long long oi = __shfl_xor_sync(BMPC_FULL, bi[q], o);
      if (oi >= 0 && better(oc, oi, bc[q], bi[q])) { bc[q] = oc; bi[q] = oi; }
    }
    cnt += __shfl_xor_sync(BMPC_FULL, cnt, o);
    cnt_hc += __shfl_xor_sync(BMPC_FULL, cnt_hc, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    for (int q = 0; q < 3; ++q) { sc[q][w] = bc[q]; si[q][w] = bi[q]; }
    scount[w] = cnt;
    shc[w] = cnt_hc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0, tot_hc = 0;
    for (int t = 0; t < (int)(blockDim.x >> 5); ++t) {
      tot += scount[t];
      tot_hc += shc[t];
      for (int q = 0; q < 3; ++q)
        if (si[q][t] >= 0 && better(sc[q][t], si[q][t], bc[q], bi[q])) {
          bc[q] = sc[q][t];
          bi[q] = si[q][t];
        }
    }
    // mask semantics: the filtered argmin is None when nothing passes
    const bool any_f = tot > 0;
    const bool any_hc = tot_hc > 0;
    best[s] = any_f ? bi[0] : -1;
    best_all[s] = l > 0 ? bi[1] : -1;
    best_hc[s] = any_hc ? bi[2] : -1;
    nfeas[s] = tot;
  }
}

// ------------------------------------------------------------------- misc --
// (xi_x, xi_y) pairs, and optionally the pairs scaled to the ellipse frame
// (b xi_x, a xi_y) that the sweep's outside test reads.
// With `scaled`, also the fp32 copy of the ellipse-frame pairs the sweep's
// prefilter reads (am_solve_kernel.cuh obstacle_block): rounded to nearest, and
// NaN when a coordinate exceeds the prefilter's magnitude bound (the fp32 test
// then never decides that term, the fp64 test does).
__global__ void k_pack_xi(long long total, const double* __restrict__ xi_x,
                          const double* __restrict__ xi_y, double2* __restrict__ out,
                          double2* __restrict__ scaled, double a, double b, int* zero,
                          int nzero) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nzero) zero[e] = 0;  // the solve's scratch flags (saves a memset call)
  if (e >= total) return;
  const double x = xi_x[e], y = xi_y[e];
  out[e] = make_double2(x, y);
  if (scaled) {
    const double sx = b * x, sy = a * y;
    scaled[e] = make_double2(sx, sy);
    const double lim = prefilter_lim(a, b);
    const bool ok = fabs(sx) <= lim && fabs(sy) <= lim;
    reinterpret_cast<float2*>(scaled + total)[e] =
        ok ? make_float2(__double2float_rn(sx), __double2float_rn(sy)) : make_float2(NAN, NAN);
  }
}

// Bounding box of every obstacle's ellipse-frame predictions over every
// 32-sample slot (the sweep's culling, am_solve_kernel.cuh obstacle_block):
// (min x, max x, min y, max y) rounded outward to fp32; unbounded when a
// prediction is NaN.  Entry (scene * nslots + slot) * m + j.
__global__ void k_obstacle_boxes(long long count, int m, int n, int nslots,
                                 const double2* __restrict__ xis, float4* __restrict__ box) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  const int j = (int)(e % m);
  const long long r = e / m;
  const int sl = (int)(r % nslots);
  const long long sc = r / nslots;
  const double2* q = xis + ((size_t)sc * m + j) * n;
  double lx = INFINITY, hx = -INFINITY, ly = INFINITY, hy = -INFINITY;
  bool nan = false;
  const int k1 = min(n, 32 * sl + 32);
  for (int k = 32 * sl; k < k1; ++k) {
    const double2 v = q[k];
    nan |= v.x != v.x || v.y != v.y;
    lx = fmin(lx, v.x);
    hx = fmax(hx, v.x);
    ly = fmin(ly, v.y);
    hy = fmax(hy, v.y);
  }
  box[e] = nan ? make_float4(-INFINITY, INFINITY, -INFINITY, INFINITY)
               : make_float4(__double2float_rd(lx), __double2float_ru(hx), __double2float_rd(ly),
                             __double2float_ru(hy));
}

// ---------------------------------------------------------------- launchers --
cudaError_t op_obstacle_update(int n, int l, long long mn, const double* x, const double* y,
                               const double* xi_x, const double* xi_y, double a, double b,
                               double* alpha, double* d, cudaStream_t st) {
  if (mn * l > 0) k_obstacle_update<<<nblk(mn * l), kTB, 0, st>>>(n, l, mn, x, y, xi_x, xi_y, a, b, alpha, d);
  return cudaGetLastError();
}
cudaError_t op_accel_update(long long nl, const double* xdd, const double* ydd, double a_max,
                            double* alpha_a, double* d_a, cudaStream_t st) {
  if (nl > 0) k_accel_update<<<nblk(nl), kTB, 0, st>>>(nl, xdd, ydd, a_max, alpha_a, d_a);
  return cudaGetLastError();
}
cudaError_t op_v_update(long long nl, const double* xd, const double* yd, double v_min,
                        double v_max, double* v, cudaStream_t st) {
  if (nl > 0) k_v_update<<<nblk(nl), kTB, 0, st>>>(nl, xd, yd, v_min, v_max, v);
  return cudaGetLastError();
}
cudaError_t op_assemble_g(int n, int l, long long mn, const double* xi_x, const double* xi_y,
                          const double* alpha, const double* d, const double* alpha_a,
                          const double* d_a, const double* v, const double* psi, double a,
                          double b, double* g_x, double* g_y, cudaStream_t st) {
  const long long tot = (mn + 2LL * n) * l;
  if (tot > 0)
    k_assemble_g<<<nblk(tot), kTB, 0, st>>>(n, l, mn, xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi, a, b, g_x, g_y);
  return cudaGetLastError();
}
cudaError_t op_residual_vectors(int n, int l, long long mn, const double* x, const double* y,
                                const double* xd, const double* yd, const double* xdd,
                                const double* ydd, const double* psi, const double* xi_x,
                                const double* xi_y, const double* alpha, const double* d,
                                const double* alpha_a, const double* d_a, const double* v,
                                double a, double b, double* r_x, double* r_y, cudaStream_t st) {
  const long long tot = (mn + 2LL * n) * l;
  if (tot > 0)
    k_residual_vectors<<<nblk(tot), kTB, 0, st>>>(n, l, mn, x, y, xd, yd, xdd, ydd, psi, xi_x, xi_y,
                                                  alpha, d, alpha_a, d_a, v, a, b, r_x, r_y);
  return cudaGetLastError();
}
cudaError_t op_tail(bool with_angles, int n, int l, long long mn, const double* x, const double* y,
                    const double* xd, const double* yd, const double* xdd, const double* ydd,
                    const double* psi, const double* xi_x, const double* xi_y, double v_min,
                    double v_max, double a_max, double a, double b, double* alpha, double* d,
                    double* alpha_a, double* d_a, double* v, double* r_x, double* r_y,
                    double* g_x, double* g_y, double* sq_obs, double* sq_acc, double* sq_nonhol,
                    cudaStream_t st) {
  if (l <= 0) return cudaSuccess;
  const long long tot = (mn + n) * (long long)l;
  if (with_angles) {
    k_tail<true><<<nblk(tot), kTB, 0, st>>>(n, l, mn, x, y, xd, yd, xdd, ydd, psi, xi_x, xi_y, v_min,
                                            v_max, a_max, a, b, alpha, d, alpha_a, d_a, v, r_x, r_y, g_x,
                                            g_y);
  } else {
    k_tail<false><<<nblk(tot), kTB, 0, st>>>(n, l, mn, x, y, xd, yd, xdd, ydd, psi, xi_x, xi_y, v_min,
                                             v_max, a_max, a, b, alpha, d, alpha_a, d_a, v, r_x, r_y, g_x,
                                             g_y);
    k_tail_sums<<<dim3((l + 31) / 32, 3), 32, 0, st>>>(n, l, mn, r_x, r_y, sq_obs, sq_acc, sq_nonhol);
  }
  return cudaGetLastError();
}
cudaError_t op_sample(int n, int npad, int nb, int L, const double* PT, const double* c_x,
                      const double* c_y, const double* c_psi, double* x, double* y, double* xd,
                      double* yd, double* xdd, double* ydd, double* psi, double* psid, double* v,
                      cudaStream_t st) {
  const long long tot = (long long)n * L;
  if (tot > 0)
    k_sample<<<nblk(tot), kTB, 0, st>>>(n, npad, nb, L, PT, c_x, c_y, c_psi, x, y, xd, yd, xdd, ydd,
                                        psi, psid, v);
  return cudaGetLastError();
}
cudaError_t op_score(const ScoreArgs& S, cudaStream_t st) {
  if (S.L <= 0) return cudaSuccess;
  const int warps = 8;
  k_score<<<(S.L + warps - 1) / warps, warps * 32, 0, st>>>(S);
  return cudaGetLastError();
}
cudaError_t op_score_samples(const ScoreParams& sp, int l, int L, const double* xi2, const double* x,
                             const double* y, const double* psi, const double* v, const double* res,
                             double* meta, double* min_ratio, double* heading_max, uint8_t* flags,
                             cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  const int warps = 8;
  k_score_samples<<<(L + warps - 1) / warps, warps * 32, 0, st>>>(
      sp, l, L, reinterpret_cast<const double2*>(xi2), x, y, psi, v, res, meta, min_ratio,
      heading_max, flags);
  return cudaGetLastError();
}
cudaError_t op_argmin(int S, int l, const double* meta, const uint8_t* flags, long long* best,
                      long long* best_all, long long* best_hc, long long* nfeas, cudaStream_t st) {
  if (S > 0) k_argmin<<<S, 256, 0, st>>>(l, meta, flags, best, best_all, best_hc, nfeas);
  return cudaGetLastError();
}
cudaError_t op_obstacle_boxes(int S, int m, int n, const double* xis, float* boxes, cudaStream_t st) {
  const int nslots = (n + 31) / 32;
  const long long count = (long long)S * nslots * m;
  if (count > 0)
    k_obstacle_boxes<<<nblk(count), kTB, 0, st>>>(count, m, n, nslots, reinterpret_cast<const double2*>(xis),
                                                  reinterpret_cast<float4*>(boxes));
  return cudaGetLastError();
}
cudaError_t op_pack_xi(long long total, const double* xi_x, const double* xi_y, double* out,
                       cudaStream_t st, double* scaled, double a, double b, int* zero, int nzero) {
  const long long work = total > nzero ? total : nzero;
  if (work > 0)
    k_pack_xi<<<nblk(work), kTB, 0, st>>>(total, xi_x, xi_y, reinterpret_cast<double2*>(out),
                                          reinterpret_cast<double2*>(scaled), a, b, zero, nzero);
  return cudaGetLastError();
}

// Early-stop decision in one launch (solver.py:437-439): t* = the first sweep no
// instance flagged as not converged; re-run t* + 1 sweeps unless that is all
// of them (0 = no re-run); {iterations, converged} into status (and status2).
__global__ void k_early_stop(int max_iter, const unsigned long long* __restrict__ notconv, int* rerun,
                             int* status, int* status2) {
  __shared__ int wbest[8];
  int best = 0x7f7f7f7f;
  for (int t = threadIdx.x; t < max_iter; t += blockDim.x)
    if ((notconv[t] >> 32) == 0ull) best = min(best, t);
  for (int o = 16; o >= 1; o >>= 1) best = min(best, __shfl_xor_sync(BMPC_FULL, best, o));
  if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = min(best, wbest[w]);
  const bool conv = best < max_iter;
  const int iters = conv ? best + 1 : max_iter;
  *rerun = (conv && iters < max_iter) ? iters : 0;
  status[0] = iters;
  status[1] = conv ? 1 : 0;
  if (status2) {
    status2[0] = iters;
    status2[1] = conv ? 1 : 0;
  }
}

cudaError_t op_early_stop(int max_iter, const unsigned long long* notconv, int* rerun, int* status, int* status2,
                          cudaStream_t st) {
  k_early_stop<<<1, 256, 0, st>>>(max_iter, notconv, rerun, status, status2);
  return cudaGetLastError();
}
// Device-side early-stop decision: the re-run sweep count (0 = none) and the
// {iterations, converged} status of the solve.

}  // namespace bmpc

// ---------------------------------------------------------- math checks --
// Device-math validation hook for the tests: fn 0 atan2_nb, 1 CUDA atan2,
// 2 rsqrt_nb, 3 sincos_nb, 4 CUDA sincos, 5 div_nb.
namespace bmpc {
__global__ void k_math_check(int fn, long long n, const double* __restrict__ a,
                             const double* __restrict__ b, double* out, double* out2) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double x = a[e], y = b ? b[e] : 0.0;
  double s = 0.0, c = 0.0;
  switch (fn) {
    case 0: out[e] = atan2_nb(x, y); break;
    case 1: out[e] = atan2(x, y); break;
    case 2: out[e] = rsqrt_nb(x); break;
    case 3: sincos_nb(x, &s, &c); out[e] = s; out2[e] = c; break;
    case 4: sincos(x, &s, &c); out[e] = s; out2[e] = c; break;
    case 5: out[e] = div_nb(x, y); break;
    case 6: out[e] = atan2_o0(x, y); break;
    case 7: sincos_q0(x, &s, &c); out[e] = s; out2[e] = c; break;
    default: break;
  }
}
cudaError_t op_math_check(int fn, long long n, const double* a, const double* b, double* out,
                          double* out2, cudaStream_t st) {
  if (n > 0) k_math_check<<<nblk(n), kTB, 0, st>>>(fn, n, a, b, out, out2);
  return cudaGetLastError();
}
}  // namespace bmpc

// ------------------------------------------------------- scene assembly --
// Device-side build_batch for S stacked scenes (planner.py:336-360,
// traffic.py:199-233): select_nearest (stable sort by squared distance, pad
// with virtual vehicles at ego + 1e4), predict_constant_velocity
// (x + vx * (t_k - t_0)) and boundary_vectors.  Same roundings as the
// reference's Python/numpy (this unit is compiled with -fmad=false).
namespace bmpc {
__global__ void k_assemble_xi(int S, int V, int m, int n, const double* __restrict__ veh,
                              const int* __restrict__ nveh, const double* __restrict__ ego,
                              const double* __restrict__ rel, double* xi_x, double* xi_y) {
  extern __shared__ double sh[];
  double* d = sh;                        // V squared distances
  double* pick = sh + V;                 // m x 4 picked states
  const int s = blockIdx.x;
  const int nv = min(nveh[s], V);
  const double ex = ego[s * 8 + 0], ey = ego[s * 8 + 3];
  const double* vs = veh + (size_t)s * V * 4;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const double dx = __dadd_rn(vs[i * 4 + 0], -ex), dy = __dadd_rn(vs[i * 4 + 1], -ey);
    d[i] = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) {  // virtual padding
    pick[j * 4 + 0] = __dadd_rn(ex, 1.0e4);
    pick[j * 4 + 1] = __dadd_rn(ey, 1.0e4);
    pick[j * 4 + 2] = 0.0;
    pick[j * 4 + 3] = 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {  // stable rank = sorted position
    const double di = d[i];
    int r = 0;
    for (int j = 0; j < nv; ++j) r += (d[j] < di) || (d[j] == di && j < i);
    if (r < m)
      for (int q = 0; q < 4; ++q) pick[r * 4 + q] = vs[i * 4 + q];
  }
  __syncthreads();
  const size_t base = (size_t)s * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int j = e / n, k = e - j * n;
    xi_x[base + e] = __dadd_rn(pick[j * 4 + 0], __dmul_rn(pick[j * 4 + 2], rel[k]));
    xi_y[base + e] = __dadd_rn(pick[j * 4 + 1], __dmul_rn(pick[j * 4 + 3], rel[k]));
  }
}

__global__ void k_assemble_b(int S, int l, const double* __restrict__ ego,
                             const double* __restrict__ goals, double* b_xy, double* b_psi) {
  const long long L = (long long)S * l;
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L) return;
  const double* e = ego + (c / l) * 8;
  const double* g = goals + c * 6;
  const double col[12] = {e[0], e[1], e[2], g[0], g[1], g[2], e[3], e[4], e[5], g[3], g[4], g[5]};
#pragma unroll
  for (int r = 0; r < 12; ++r) b_xy[r * L + c] = col[r];
  b_psi[0 * L + c] = e[6];
  b_psi[1 * L + c] = e[7];
  b_psi[2 * L + c] = 0.0;
  b_psi[3 * L + c] = 0.0;
}

cudaError_t op_assemble(int S, int V, int m, int n, int l, const double* veh, const int* nveh,
                        const double* ego, const double* goals, const double* rel, double* xi_x,
                        double* xi_y, double* b_xy, double* b_psi, cudaStream_t st) {
  if (S > 0 && m > 0) {
    const size_t smem = (size_t)(V + 4 * m) * sizeof(double);
    k_assemble_xi<<<S, 256, smem, st>>>(S, V, m, n, veh, nveh, ego, rel, xi_x, xi_y);
  }
  const long long L = (long long)S * l;
  if (L > 0) k_assemble_b<<<nblk(L), kTB, 0, st>>>(S, l, ego, goals, b_xy, b_psi);
  return cudaGetLastError();
}
}  // namespace bmpc
