#pragma once
// am_solve.cu -- persistent fused alternating-minimization kernel (sm_100a, fp64).
//
// One warp owns one trajectory instance for the whole solve; all AM sweeps run
// inside a single launch and every iterate stays on chip (registers + a few
// hundred bytes of per-warp shared memory).  Per sweep (reference
// /root/reference/pkg/src/batchmpc/solver.py:458-500):
//
//   1. xy QP     [c; mu] = K_axis^-1 [rho*G + lambda ; b], one refinement step
//                (solver.py:302-312, :164-168)
//   2. sampling  xdot, ydot = Pdot c ; theta = unwrap(atan2(ydot, xdot)) (:474-477)
//   3. psi QP    c_psi = K_psi^-1 [rho*P^T theta + lambda_psi ; b_psi], refined (:322-328)
//   4. tail      closed forms for d, d_a, v; residual blocks; next targets
//                (kernels/_speedups.pyx:114-218), contracted on the fly:
//                G = F_axis^T g = P^T sum_j g_obs,j + Pddot^T g_acc + Pdot^T g_nh
//                R = F_axis^T r (same split), lambda -= rho*R (:491-494)
//
// Lanes split the horizon samples k (k = lane + 32*r); lane i owns coefficient i
// of the x axis (and of psi), lane 16+i coefficient i of the y axis.  The
// contractions over k are warp reduce-scatters with a fixed summation tree, so
// an instance's arithmetic never depends on the batch size, its column index
// or the GPU shard it lands on.
//
// The obstacle block uses the minimal formulation of SURVEY.md finding 8:
// obstacle-sum-first projections and rsqrt-and-multiply in place of sqrt and
// three divisions (parity measured at <=1e-10 relative on stable columns).
#include <cuda_runtime.h>
#include <stdio.h>

#include "am_args.h"
#include "common.cuh"

namespace bmpc {

struct WarpScratch {
  double* bc;    // 64: KKT right-hand sides (x at 0, y at 32)
  double* sol;   // 64: first solve  Kinv * rhs
  double* res;   // 64: refinement residual rhs - K * sol
  double* cxy;   // 32: (c_x[i], c_y[i]) pairs
  double* cp;    // 16: c_psi
  double* th;    // npad: theta (unwrapped heading target) per sample
};
constexpr int kWarpScratch = 256;

// One row of a KKT apply.  The QP steps run the reference's refined solve
// (solver.py:164-168) -- sol = K^-1 rhs; sol += K^-1 (rhs - K sol) -- with the
// LU factors replaced by the explicit inverse; without the refinement step the
// explicit inverse loses up to 5e-8 relative at the c4 shape (cond 3.9e6).
template <int LEN>
__device__ __forceinline__ double kkt_row_dot(const double* __restrict__ kr,
                                              const double* __restrict__ v) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < LEN; ++j) s = fma(kr[j], v[j], s);
  return s;
}

template <int NB, int NKM>
__global__ void __launch_bounds__(256) am_solve_kernel(const bmpc_dev_consts C,
                                                       const bmpc_solve_args A) {
  extern __shared__ __align__(16) double sm[];
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n = C.n, npad = C.npad;
  const int nk = npad >> 5;
  const int L = A.L;
  constexpr int RX = NB + 6, RP = NB + 4;

  double* sPT = sm;                          // P^T, Pdot^T, Pddot^T
  double* sKxf = sPT + 3 * NB * npad;
  double* sKxa = sKxf + RX * C.kxs;
  double* sKpf = sKxa + RX * C.kxs;
  double* sKpa = sKpf + RP * C.kps;
  double* sTau = sKpa + RP * C.kps;
  double* wbase = sTau + npad + warp * (kWarpScratch + npad);
  WarpScratch ws{wbase, wbase + 64, wbase + 128, wbase + 192, wbase + 224, wbase + kWarpScratch};

  for (int t = threadIdx.x; t < 3 * NB * npad; t += blockDim.x) sPT[t] = C.PT[t];
  for (int t = threadIdx.x; t < RX * C.kxs; t += blockDim.x) {
    sKxf[t] = C.Kxf[t];
    sKxa[t] = C.Kxa[t];
  }
  for (int t = threadIdx.x; t < RP * C.kps; t += blockDim.x) {
    sKpf[t] = C.Kpf[t];
    sKpa[t] = C.Kpa[t];
  }
  for (int t = threadIdx.x; t < npad; t += blockDim.x) sTau[t] = C.tau[t];
  __syncthreads();

  const int inst = blockIdx.x * W + warp;
  if (inst >= L) return;  // no block-wide barriers below this point

  const double* __restrict__ sP = sPT;
  const double* __restrict__ sPd = sPT + NB * npad;
  const double* __restrict__ sPdd = sPT + 2 * NB * npad;
  const double2* __restrict__ xi =
      reinterpret_cast<const double2*>(A.xi) + (size_t)(inst / A.l) * A.m * n;
  const int m = A.m;
  const double a = A.a, b = A.b, rho = C.rho;
  const double inv_ab = 1.0 / (a * b);

  const int li = lane & 15;
  const bool yax = lane >= 16;
  const bool owner = li < NB;

  // persistent per-lane state (owner lanes)
  double lam = 0.0, G = 0.0;   // lane i: lambda_x[i], G_x[i]; lane 16+i: lambda_y[i], G_y[i]
  double lamp = 0.0;           // lane i: lambda_psi[i]
  double bnd = 0.0, bps = 0.0;
  double cown = 0.0, cpown = 0.0;
  if (li < 6) bnd = A.b_xy[(size_t)(yax ? 6 + li : li) * L + inst];
  if (yax && li < 4) bps = A.b_psi[(size_t)li * L + inst];

  // ---------------------------------------------------------------- init ----
  if (A.init_mode == BMPC_INIT_RESUME) {
    const double* cr = A.carry + (size_t)inst * 5 * NB;
    if (owner) {
      lam = cr[(yax ? 1 : 0) * NB + li];
      lamp = cr[2 * NB + li];
      G = cr[(yax ? 4 : 3) * NB + li];
    }
  } else {
    // Initial targets g = assemble_g(alpha, d, alpha_a, d_a, v, psi) contracted
    // to G = F_axis^T g (solver.py:431, :281-286; kernels/_speedups.pyx:81-111).
    double ax[16], ay[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { ax[i] = 0.0; ay[i] = 0.0; }
    const bool cold = A.init_mode == BMPC_INIT_COLD;
    double x0 = 0, xf = 0, y0 = 0, yf = 0, speed0 = 0;
    if (cold) {
      // straight start->goal line (solver.py:226-252)
      x0 = A.b_xy[0 * (size_t)L + inst];
      xf = A.b_xy[3 * (size_t)L + inst];
      y0 = A.b_xy[6 * (size_t)L + inst];
      yf = A.b_xy[9 * (size_t)L + inst];
      const double vx0 = A.b_xy[1 * (size_t)L + inst], vy0 = A.b_xy[7 * (size_t)L + inst];
      speed0 = sqrt(__dadd_rn(__dmul_rn(vx0, vx0), __dmul_rn(vy0, vy0)));
      speed0 = fmin(fmax(speed0, A.v_min), A.v_max);
      if (owner) {
        lam = 0.0;
        lamp = 0.0;
      }
    } else {
      if (owner) {
        lam = A.w_lx ? (yax ? A.w_ly : A.w_lx)[(size_t)li * L + inst] : 0.0;
        lamp = A.w_lp ? A.w_lp[(size_t)li * L + inst] : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < NKM; ++r) {
      const int k = lane + 32 * r;
      if (r < nk && k < n) {
        double gsx = 0.0, gsy = 0.0, gax = 0.0, gay = 0.0, gnx = 0.0, gny = 0.0;
        if (cold) {
          const double xl = __dadd_rn(x0, __dmul_rn(sTau[k], __dsub_rn(xf, x0)));
          const double yl = __dadd_rn(y0, __dmul_rn(sTau[k], __dsub_rn(yf, y0)));
          for (int j = 0; j < m; ++j) {
            const double2 q = __ldg(xi + j * n + k);
            const double wx = xl - q.x, wy = yl - q.y;
            const double al = atan2(a * wy, b * wx);
            double sa, ca;
            sincos(al, &sa, &ca);
            const double num = __dadd_rn(__dmul_rn(__dmul_rn(a, ca), wx), __dmul_rn(__dmul_rn(b, sa), wy));
            const double den = __dadd_rn(__dmul_rn(a * ca, a * ca), __dmul_rn(b * sa, b * sa));
            double d = num / den;
            d = d < 1.0 ? 1.0 : d;
            gsx += q.x + __dmul_rn(a * d, ca);
            gsy += q.y + __dmul_rn(b * d, sa);
          }
          gnx = speed0;  // v cos(psi) with psi = P c_psi = 0, alpha_a = d_a = 0
        } else {
          double ps = 0.0;
#pragma unroll
          for (int i = 0; i < NB; ++i) ps = fma(sP[i * npad + k], A.w_cpsi[(size_t)i * L + inst], ps);
          for (int j = 0; j < m; ++j) {
            const double2 q = __ldg(xi + j * n + k);
            const size_t row = (size_t)(j * n + k) * L + inst;
            const double al = A.w_alpha[row], d = A.w_d[row];
            double sa, ca;
            sincos(al, &sa, &ca);
            gsx += q.x + __dmul_rn(a * d, ca);
            gsy += q.y + __dmul_rn(b * d, sa);
          }
          const size_t kr = (size_t)k * L + inst;
          double sa, ca;
          sincos(A.w_alpha_a[kr], &sa, &ca);
          gax = A.w_d_a[kr] * ca;
          gay = A.w_d_a[kr] * sa;
          sincos(ps, &sa, &ca);
          gnx = A.w_v[kr] * ca;
          gny = A.w_v[kr] * sa;
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double p = sP[i * npad + k], pd = sPd[i * npad + k], pdd = sPdd[i * npad + k];
          ax[i] = fma(p, gsx, ax[i]);
          ax[i] = fma(pdd, gax, ax[i]);
          ax[i] = fma(pd, gnx, ax[i]);
          ay[i] = fma(p, gsy, ay[i]);
          ay[i] = fma(pdd, gay, ay[i]);
          ay[i] = fma(pd, gny, ay[i]);
        }
      }
    }
    double v32[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v32[i] = i < NB ? ax[i] : 0.0;
      v32[16 + i] = i < NB ? ay[i] : 0.0;
    }
    G = reduce_scatter32(v32);
  }

  // ----------------------------------------------------------- AM sweeps ----
  for (int t = 0; t < A.iters; ++t) {
    const bool last = t == A.iters - 1;
    // (1) xy QP: [c; mu] = K^-1 [rho*G + lambda ; b] plus one refinement step,
    //     the 2*(nb+6) rows of both axes spread over the lanes (two per lane max)
    {
      double* rb = ws.bc + (yax ? 32 : 0);
      if (owner) rb[li] = rho * G + lam;
      if (li < 6) rb[NB + li] = bnd;
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = lane + 32 * h;
        if (q < 2 * RX) {
          const int ax = q >= RX ? 1 : 0, row = q - ax * RX;
          ws.sol[ax * 32 + row] = kkt_row_dot<RX>(sKxf + row * C.kxs, ws.bc + ax * 32);
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = lane + 32 * h;
        if (q < 2 * RX) {
          const int ax = q >= RX ? 1 : 0, row = q - ax * RX;
          ws.res[ax * 32 + row] =
              ws.bc[ax * 32 + row] - kkt_row_dot<RX>(sKxa + row * C.kxs, ws.sol + ax * 32);
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = lane + 32 * h;
        if (q < 2 * RX) {
          const int ax = q >= RX ? 1 : 0, row = q - ax * RX;
          if (row < NB)
            ws.cxy[2 * row + ax] =
                ws.sol[ax * 32 + row] + kkt_row_dot<RX>(sKxf + row * C.kxs, ws.res + ax * 32);
        }
      }
      __syncwarp();
      if (owner) cown = ws.cxy[2 * li + (yax ? 1 : 0)];
    }
    const double2* __restrict__ cxy = reinterpret_cast<const double2*>(ws.cxy);

    // (2) heading target theta = unwrap(atan2(ydot, xdot)) and P^T theta
    bool wrap = false;
#pragma unroll
    for (int r = 0; r < NKM; ++r) {
      const int k = lane + 32 * r;
      if (r < nk && k < n) {
        double xd = 0.0, yd = 0.0;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double pd = sPd[i * npad + k];
          const double2 c = cxy[i];
          xd = fma(pd, c.x, xd);
          yd = fma(pd, c.y, yd);
        }
        ws.th[k] = atan2(yd, xd);
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NKM; ++r) {
      const int k = lane + 32 * r;
      if (r < nk && k < n && k > 0) {
        const double dd = ws.th[k] - ws.th[k - 1];
        if (!(fabs(dd) < CUDART_PI)) wrap = true;
      }
    }
    if (__any_sync(BMPC_FULL, wrap)) {
      if (lane == 0) np_unwrap_serial(ws.th, n);
      __syncwarp();
    }
    double pth;
    {
      double pt[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pt[i] = 0.0;
#pragma unroll
      for (int r = 0; r < NKM; ++r) {
        const int k = lane + 32 * r;
        if (r < nk && k < n) {
          const double th = ws.th[k];
#pragma unroll
          for (int i = 0; i < NB; ++i) pt[i] = fma(sP[i * npad + k], th, pt[i]);
        }
      }
      pth = reduce_pairs16(pt);
    }

    // (3) psi QP
    {
      if (!yax && owner) ws.bc[li] = rho * pth + lamp;
      if (yax && li < 4) ws.bc[NB + li] = bps;
      __syncwarp();
      if (lane < RP) ws.sol[lane] = kkt_row_dot<RP>(sKpf + lane * C.kps, ws.bc);
      __syncwarp();
      if (lane < RP) ws.res[lane] = ws.bc[lane] - kkt_row_dot<RP>(sKpa + lane * C.kps, ws.sol);
      __syncwarp();
      if (lane < NB) ws.cp[lane] = ws.sol[lane] + kkt_row_dot<RP>(sKpf + lane * C.kps, ws.res);
      __syncwarp();
      if (!yax && owner) cpown = ws.cp[li];
    }

    // (4) fused tail + on-the-fly contractions
    double Gx[NB], Gy[NB], Rx[NB], Ry[NB], Lp[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) { Gx[i] = Gy[i] = Rx[i] = Ry[i] = Lp[i] = 0.0; }
    double sqo = 0.0, sqa = 0.0, sqn = 0.0;
#pragma unroll
    for (int r = 0; r < NKM; ++r) {
      const int k = lane + 32 * r;
      if (r < nk && k < n) {
        double x = 0, y = 0, xd = 0, yd = 0, xdd = 0, ydd = 0, ps = 0;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double p = sP[i * npad + k], pd = sPd[i * npad + k], pdd = sPdd[i * npad + k];
          const double2 c = cxy[i];
          const double cpi = ws.cp[i];
          x = fma(p, c.x, x);
          y = fma(p, c.y, y);
          xd = fma(pd, c.x, xd);
          yd = fma(pd, c.y, yd);
          xdd = fma(pdd, c.x, xdd);
          ydd = fma(pdd, c.y, ydd);
          ps = fma(p, cpi, ps);
        }
        // obstacle block (_speedups.pyx:150-176), summed over obstacles
        double gsx = 0.0, gsy = 0.0, rsx = 0.0, rsy = 0.0, sq = 0.0;
#pragma unroll 2
        for (int j = 0; j < m; ++j) {
          const double2 q = __ldg(xi + j * n + k);
          const double wx = x - q.x, wy = y - q.y;
          const double px = b * wx, py = a * wy;
          const double r2 = fma(px, px, py * py);
          const double ri = rsqrt(r2);
          const bool pos = r2 > 0.0;
          const double ca = pos ? px * ri : 1.0;
          const double sa = pos ? py * ri : 0.0;
          const double rr = pos ? r2 * ri : 0.0;
          const double dd = fmax(1.0, rr * inv_ab);
          const double adca = (a * dd) * ca, bdsa = (b * dd) * sa;
          const double rx = wx - adca, ry = wy - bdsa;
          sq = fma(rx, rx, fma(ry, ry, sq));
          gsx += q.x + adca;
          gsy += q.y + bdsa;
          rsx += rx;
          rsy += ry;
        }
        sqo += sq;
        // acceleration block (_speedups.pyx:179-198)
        const double m2 = fma(xdd, xdd, ydd * ydd);
        const double mi = rsqrt(m2);
        const bool mpos = m2 > 0.0;
        const double caa = mpos ? xdd * mi : 1.0, saa = mpos ? ydd * mi : 0.0;
        const double mag = mpos ? m2 * mi : 0.0;
        const double da = fmin(mag, A.a_max);
        const double gax = da * caa, gay = da * saa;
        const double rax = xdd - gax, ray = ydd - gay;
        sqa = fma(rax, rax, fma(ray, ray, sqa));
        // non-holonomic block (_speedups.pyx:200-216)
        double s = sqrt(fma(xd, xd, yd * yd));
        s = fmin(fmax(s, A.v_min), A.v_max);
        double sp, cpv;
        sincos(ps, &sp, &cpv);
        const double gnx = s * cpv, gny = s * sp;
        const double rnx = xd - gnx, rny = yd - gny;
        sqn = fma(rnx, rnx, fma(rny, rny, sqn));
        if (last && (A.flags & BMPC_F_V)) A.v_out[(size_t)k * L + inst] = s;
        const double dpt = ps - ws.th[k];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double p = sP[i * npad + k], pd = sPd[i * npad + k], pdd = sPdd[i * npad + k];
          Gx[i] = fma(p, gsx, Gx[i]);
          Gx[i] = fma(pdd, gax, Gx[i]);
          Gx[i] = fma(pd, gnx, Gx[i]);
          Gy[i] = fma(p, gsy, Gy[i]);
          Gy[i] = fma(pdd, gay, Gy[i]);
          Gy[i] = fma(pd, gny, Gy[i]);
          Rx[i] = fma(p, rsx, Rx[i]);
          Rx[i] = fma(pdd, rax, Rx[i]);
          Rx[i] = fma(pd, rnx, Rx[i]);
          Ry[i] = fma(p, rsy, Ry[i]);
          Ry[i] = fma(pdd, ray, Ry[i]);
          Ry[i] = fma(pd, rny, Ry[i]);
          Lp[i] = fma(p, dpt, Lp[i]);
        }
      }
    }
    // warp contractions -> owner lanes
    double v32[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v32[i] = i < NB ? Gx[i] : 0.0;
      v32[16 + i] = i < NB ? Gy[i] : 0.0;
    }
    G = reduce_scatter32(v32);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v32[i] = i < NB ? Rx[i] : 0.0;
      v32[16 + i] = i < NB ? Ry[i] : 0.0;
    }
    const double R = reduce_scatter32(v32);
#pragma unroll
    for (int i = 0; i < 16; ++i) v32[i] = i < NB ? Lp[i] : 0.0;
    v32[16] = sqo;
    v32[17] = sqa;
    v32[18] = sqn;
#pragma unroll
    for (int i = 19; i < 32; ++i) v32[i] = 0.0;
    const double q3 = reduce_scatter32(v32);
    if (owner) lam -= rho * R;
    if (!yax && owner) lamp -= rho * q3;
    if (lane >= 16 && lane < 19) {
      const double res = sqrt(q3);
      if (A.flags & BMPC_F_HISTORY)
        A.hist[((size_t)(A.hist_offset + t) * 3 + (lane - 16)) * L + inst] = res;
      if (last && A.res_final) A.res_final[(size_t)(lane - 16) * L + inst] = res;
    }
    __syncwarp();
  }

  // ------------------------------------------------------------- outputs ----
  if (owner) {
    const size_t o = (size_t)li * L + inst;
    if (!yax) {
      if (A.c_x) A.c_x[o] = cown;
      if (A.l_x) A.l_x[o] = lam;
      if (A.c_psi) A.c_psi[o] = cpown;
      if (A.l_psi) A.l_psi[o] = lamp;
    } else {
      if (A.c_y) A.c_y[o] = cown;
      if (A.l_y) A.l_y[o] = lam;
    }
    if (A.flags & BMPC_F_CARRY) {
      double* cr = A.carry + (size_t)inst * 5 * NB;
      cr[(yax ? 1 : 0) * NB + li] = lam;
      if (!yax) cr[2 * NB + li] = lamp;
      cr[(yax ? 4 : 3) * NB + li] = G;
    }
  }
}

}  // namespace bmpc
