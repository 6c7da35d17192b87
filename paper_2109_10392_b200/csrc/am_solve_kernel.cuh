#pragma once
// am_solve_kernel.cuh -- persistent fused alternating-minimization kernel
// (sm_100a, fp64).
//
// One warp owns one trajectory instance for the whole solve; all AM sweeps run
// inside a single launch and every iterate stays on chip (registers + a few
// KB of per-warp shared memory).  Per sweep (reference
// /root/reference/pkg/src/batchmpc/solver.py:458-500):
//
//   1. xy QP     null-space form of [c; mu] = K_axis^-1 [rho*G + lambda ; b]
//                (solver.py:302-312): c = B b + Z (rho*G + lambda), the boundary
//                part B b once per solve, one refinement step against H only
//                on ill-conditioned shapes (:164-168; capi.cu reduced_qp)
//   2. pass A    x, y, xdot, ydot, xddot, yddot = [P; Pdot; Pddot] c;
//                theta = unwrap(atan2(ydot, xdot)) (:474-477); acceleration
//                block (kernels/_speedups.pyx:179-198); P^T theta, Pddot^T g_a
//   3. psi QP    the same for c_psi from rho*P^T theta + lambda_psi and b_psi
//                (:322-328); lambda_psi step via (P^T P) c_psi - P^T theta
//   4. pass B    psi = P c_psi, non-holonomic block (_speedups.pyx:200-216), Pdot^T g_n
//   5. obstacles exact form of _speedups.pyx:150-176 (outside: g_j = x, r_j = 0),
//                P^T sum_j g_j; the outside test in the ellipse frame on
//                predictions staged in shared memory (n <= 128)
//   6. G = F_axis^T g reduction; lambda_xy -= rho ((F_axis^T F_axis) c - G) (:491-494)
//
// Lanes split the horizon samples k (k = lane + 32*r); lane i owns coefficient i
// of the x axis (and of psi), lane 16+i coefficient i of the y axis.  The
// contractions over k go through a shared-memory transpose with a fixed
// summation order, so an instance's arithmetic never depends on the batch
// size, its column index or the GPU shard it lands on.
#include <cuda_runtime.h>
#include <stdio.h>

#include <type_traits>

#include "am_args.h"
#include "common.cuh"
#include "score.cuh"

namespace bmpc {

// Phase profiling build (-DBMPC_PHASE_PROF, tools/phase_prof.py): lane 0 of
// every warp adds the clock64 cycles of each kernel phase to a per-unit
// device counter.  Compiled out of the product library.
#ifdef BMPC_PHASE_PROF
static __device__ unsigned long long g_phase_cycles[20];
__shared__ unsigned long long s_prof[BMPC_MAX_WARPS][20];
__shared__ long long s_prof_t[BMPC_MAX_WARPS];
#define BMPC_PROF_DECL                                               \
  if ((threadIdx.x & 31) == 0) {                                     \
    for (int _i = 0; _i < 20; ++_i) s_prof[threadIdx.x >> 5][_i] = 0; \
    s_prof_t[threadIdx.x >> 5] = clock64();                          \
  }
#define BMPC_PROF(ph)                                                \
  do {                                                               \
    __syncwarp();                                                    \
    const long long _t = clock64();                                  \
    if ((threadIdx.x & 31) == 0) {                                   \
      s_prof[threadIdx.x >> 5][ph] += _t - s_prof_t[threadIdx.x >> 5]; \
      s_prof_t[threadIdx.x >> 5] = _t;                               \
    }                                                                \
  } while (0)
// lane-0 view without a warp sync (usable in divergent code)
#define BMPC_PROF_NS(ph)                                             \
  do {                                                               \
    const long long _t = clock64();                                  \
    if ((threadIdx.x & 31) == 0) {                                   \
      s_prof[threadIdx.x >> 5][ph] += _t - s_prof_t[threadIdx.x >> 5]; \
      s_prof_t[threadIdx.x >> 5] = _t;                               \
    }                                                                \
  } while (0)
#define BMPC_PROF_FLUSH                                               \
  if ((threadIdx.x & 31) == 0)                                        \
    for (int _i = 0; _i < 20; ++_i)                                   \
      atomicAdd(&g_phase_cycles[_i], s_prof[threadIdx.x >> 5][_i]);
#else
#define BMPC_PROF_DECL
#define BMPC_PROF(ph) do {} while (0)
#define BMPC_PROF_NS(ph) do {} while (0)
#define BMPC_PROF_FLUSH
#endif

// mbarrier + 1-D bulk asynchronous copy (TMA engine) helpers.
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes,
                                              unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

struct WarpScratch {
  double* cxy;   // 32: (c_x[i], c_y[i]) pairs
  double* cp;    // 16: c_psi
  double* res;   // 16: the last sweep's block residuals (fused scoring)
  double* th;    // npad: theta per sample (read back only by the unwrap slow path)
  double* xd;    // npad: xdot per sample (pass A -> pass B)
  double* yd;    // npad: ydot per sample
  double* x;     // npad: x per sample (pass A -> obstacle block), if stored
  double* y;     // npad: y per sample
  double* red;   // 32 x kRedStride: transpose buffer of the sample contractions
};
constexpr int kWarpScratch = 64;
constexpr int kRedStride = 33;
constexpr int kRedSize = 32 * kRedStride;

// Sum of column `col` of the 32-row transpose buffer, in a fixed order.
__device__ __forceinline__ double column_sum(const double* __restrict__ red, int col) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int r = 0; r < 32; r += 4) {
    s0 += red[(r + 0) * kRedStride + col];
    s1 += red[(r + 1) * kRedStride + col];
    s2 += red[(r + 2) * kRedStride + col];
    s3 += red[(r + 3) * kRedStride + col];
  }
  return (s0 + s1) + (s2 + s3);
}

// Work slot r of a lane.  Samples are dealt round-robin (k = lane + 32 r) for
// the F = n / 32 full rounds; the R = n % 32 leftover samples either take one
// lane each (R > 16) or, in split mode, a group of g = 2^floor(log2(32/R))
// lanes each, the group splitting that sample's obstacles (j = j0, j0+g, ...)
// so the last round is not 32-R idle lanes deep.  Only the group leader owns
// the per-sample terms.
struct SlotLayout {
  int F, R, g, lg;  // g = 2^lg lanes per leftover sample; g == 1: no split
};
struct Slot {
  int k, j0, js;
  bool valid, leader;
};
__device__ __forceinline__ SlotLayout slot_layout(int n) {
  SlotLayout s;
  s.F = n >> 5;
  s.R = n & 31;
  s.g = 1;
  s.lg = 0;
  if (s.R > 0 && s.R <= 16) {
    int g = 32 / s.R;
    while (g & (g - 1)) g &= g - 1;
    s.g = g;
    s.lg = __ffs(g) - 1;
  }
  return s;
}
__device__ __forceinline__ Slot slot(int r, int lane, const SlotLayout& sl) {
  Slot S;
  if (r < sl.F) {
    S.k = lane + 32 * r;
    S.j0 = 0;
    S.js = 1;
    S.valid = true;
    S.leader = true;
  } else if (r == sl.F && sl.R > 0) {
    const int grp = lane >> sl.lg;
    S.k = 32 * sl.F + grp;
    S.j0 = lane & (sl.g - 1);
    S.js = sl.g;
    S.valid = grp < sl.R;
    S.leader = S.j0 == 0;
  } else {
    S.k = 0;
    S.j0 = 0;
    S.js = 1;
    S.valid = false;
    S.leader = false;
  }
  return S;
}

// Exact form of the same closed forms (fp64 path): outside the ellipse
// (d = r/(ab) > 1) g_j = q + (a d cos, b d sin) = q + w = x and r_j = 0
// identically, so a term needs only the outside test; inside (d = 1)
// g_j = q + (a cos, b sin), r_j = w - (a cos, b sin).  On the BASELINE scenes
// about 1% of lane groups hold an inside term.  NaN distances test
// as inside, so they propagate like the reference's.
__device__ __forceinline__ bool obstacle_inside(double x, double y, double2 q, double a, double b,
                                                double ab2) {
  const double px = b * (x - q.x), py = a * (y - q.y);
  return !(fma(px, px, py * py) >= ab2);
}
// The sweep's form: position and prediction already in the ellipse frame
// (xs = b x, ys = a y; qs = (b qx, a qy), packed once per solve), so a term
// costs two subtractions, a multiply and an fma.  The rounding differs from
// b (x - qx) only in the last bits, which moves the d = 1 boundary by
// rounding, as the reference's own r / (a b) does.
__device__ __forceinline__ bool obstacle_inside_s(double xs, double ys, double2 qs, double ab2) {
  const double px = xs - qs.x, py = ys - qs.y;
  return !(fma(px, px, py * py) >= ab2);
}
// Inside term in the ellipse frame: w = (px / b, py / a), r_j = w - (a cos, b sin).
__device__ __forceinline__ void obstacle_inside_res_s(double xs, double ys, double2 qs, double a,
                                                      double b, double ia, double ib, double& srx,
                                                      double& sry, double& sq, double& cin) {
  const double px = xs - qs.x, py = ys - qs.y;
  const double r2 = fma(px, px, py * py);
  const double ri = rsqrt_nb(r2);
  const double ca = r2 > 0.0 ? px * ri : 1.0, sa = py * ri;  // r = 0 -> (1, 0)
  const double rx = fma(px, ib, -a * ca), ry = fma(py, ia, -b * sa);
  sq = fma(rx, rx, fma(ry, ry, sq));
  srx += rx;
  sry += ry;
  cin += 1.0;
}
__device__ __forceinline__ void obstacle_inside_term(double x, double y, double2 q, double a,
                                                     double b, double& gix, double& giy,
                                                     double& sq, double& cin) {
  const double wx = x - q.x, wy = y - q.y;
  const double px = b * wx, py = a * wy;
  const double r2 = fma(px, px, py * py);
  const double ri = rsqrt_nb(r2);
  // r = 0 -> (cos, sin) = (1, 0) (_speedups.pyx:158-166); py = 0 there
  const double ca = r2 > 0.0 ? px * ri : 1.0, sa = py * ri;
  const double ax = a * ca, by = b * sa;
  const double rx = wx - ax, ry = wy - by;
  sq = fma(rx, rx, fma(ry, ry, sq));
  gix += q.x + ax;
  giy += q.y + by;
  cin += 1.0;
}

// Obstacles in flight per sample: pair passes, single full slots, split leftover slots.
#ifndef BMPC_UPAIR
#define BMPC_UPAIR 2
#endif
#ifndef BMPC_USINGLE
#define BMPC_USINGLE 5
#endif
#ifndef BMPC_USPLIT
#define BMPC_USPLIT 1
#endif
#ifndef BMPC_USPLIT_MANY
// long horizons (n > 192): the leftover slot is split over fewer lanes per
// sample, so each lane walks many obstacles (c4: m = 50 over g = 4 lanes)
#define BMPC_USPLIT_MANY 4
#endif
// Two sample slots per obstacle pass when the accumulators leave register room.
template <int NB>
constexpr bool kPairSlots = NB <= 12;

struct TailArgs {
  const double* P;
  const double2* cxy;
  const double2* xi;  // predictions in the ellipse frame (b qx, a qy), fp64 (shared memory when staged)
  const float2* xf;   // the same rounded to fp32, for the prefilter (global)
  const double *xs, *ys;  // sampled positions (pass A) or nullptr: recompute from c
  int n, m;
  double a, b;
  double ia, ib;  // 1 / a, 1 / b
  float t32;      // prefilter threshold round_up(1.02 (ab)^2) (common.cuh prefilter_lim)
  float lim32;    // largest coordinate magnitude the prefilter may decide
  const float4* box;  // [slot][m] obstacle bounding boxes (k_obstacle_boxes) or nullptr
  float tc;           // culling threshold round_up((ab)^2 (1 + 1e-4)) on the squared box gap
  float2* sk_p0;      // clearance skipping: per sample the recorded frame position
  float* sk_m0;       //   and squared clearance (-1: never skip), or nullptr
  float ab_ru;        // a b rounded up to fp32
};

// fp32 mode inside term (the outside test runs in fp64 in both modes): with
// d = 1 the residual is r = w - (a cos, b sin) and g = x - r, evaluated in fp32
// from w rounded off the fp64 difference, so far and virtual obstacles (+1e4 m)
// never see |w| rounded in fp32.
__device__ __forceinline__ void obstacle_term_f32(double xs, double ys, double2 qs, float a, float b,
                                                  float ab2, double ia, double ib, float& srx,
                                                  float& sry, float& sq, double& cin) {
  cin += 1.0;
  const float wx = (float)((xs - qs.x) * ib), wy = (float)((ys - qs.y) * ia);
  const float px = b * wx, py = a * wy;
  const float r2 = fmaf(px, px, py * py);
  const float ri = rsqrtf(r2);
  const bool pos = r2 > 0.f;
  const float ca = pos ? px * ri : 1.f, sa = pos ? py * ri : 0.f;
  const bool inside = r2 < ab2;  // r / (ab) < 1  <=>  d = 1
  const float rx = inside ? fmaf(-a, ca, wx) : 0.f;
  const float ry = inside ? fmaf(-b, sa, wy) : 0.f;
  sq = fmaf(rx, rx, fmaf(ry, ry, sq));
  srx += rx;
  sry += ry;
}

// Obstacle block (kernels/_speedups.pyx:150-176) in exact form for NS samples
// of one lane: every term takes the outside test; the inside terms' residuals
// r_j give the correction -P^T sum_inside r_j to P^T sum_j g_j = m (P^T P) c
// (the Gram part is added once per sweep) and the squared residual.
// Obstacles j0, j0+js, ...; `group` > 1 marks a split slot whose partials are
// summed over `group` consecutive lanes (warp-uniform) before the group leader
// contributes them.  The acceleration and non-holonomic blocks run in passes
// A and B of the sweep.
// Basis rows at the slots of a chunk: with PAIRED the NS == 2 slots are an even
// slot pair (samples k and k + 32), adjacent in the paired-slot image, so one
// 16-byte load returns both; otherwise one load per slot.
// (T = double, or float for the fp32 mode's basis: the same index order)
template <class T> struct vec2_of { using type = double2; };
template <> struct vec2_of<float> { using type = float2; };
template <int NS, bool PAIRED, int NPAD, class T>
__device__ __forceinline__ void basis1(const T* B, int i, const int (&k)[NS], T (&v)[NS]) {
  if constexpr (PAIRED && NS == 2) {
    const auto w = *reinterpret_cast<const typename vec2_of<T>::type*>(B + bmpc_basis_index(i, k[0], NPAD));
    v[0] = w.x;
    v[1] = w.y;
  } else {
#pragma unroll
    for (int s = 0; s < NS; ++s) v[s] = B[bmpc_basis_index(i, k[s], NPAD)];
  }
}
template <int NS, bool PAIRED, int NPAD, class T>
__device__ __forceinline__ void basis3(const T* B0, const T* B1, const T* B2, int i,
                                       const int (&k)[NS], T (&v0)[NS], T (&v1)[NS],
                                       T (&v2)[NS]) {
  basis1<NS, PAIRED, NPAD>(B0, i, k, v0);
  basis1<NS, PAIRED, NPAD>(B1, i, k, v1);
  basis1<NS, PAIRED, NPAD>(B2, i, k, v2);
}

// Prediction loads: shared memory when the block staged its scene(s), else
// the read-only global path.
template <bool XS, class T>
__device__ __forceinline__ T ldq(const T* p) {
  if constexpr (XS)
    return *p;
  else
    return __ldg(p);
}

// BMPC_XS32: staged predictions are the fp32 ellipse-frame copies (half the
// shared-memory bytes); the obstacle test runs through the exact fp32
// prefilter on them, undecided terms take the fp64 pair from global memory.
#ifndef BMPC_XS32
#define BMPC_XS32 0
#endif
// BMPC_SKIP: clearance skipping of whole obstacle slots (staged fp64
// predictions, one warp per instance, n <= 128).  A pass over a slot records
// per sample its position P0 (ellipse frame, fp32) and a lower bound M0 of
// min_j |P0 - Q_j| - ab; while every sample of the slot has moved less than
// its M0 since then, every term of the slot is outside (triangle inequality)
// and contributes exactly nothing, so the pass is skipped.  Bit-identical to
// running it (kSkipSlack covers every fp32 rounding of the test).
#ifndef BMPC_SKIP_LATE
#define BMPC_SKIP_LATE 0  // 1: the clearance test in its own loop after pass A's chunks
#endif
constexpr float kSkipSlack = 0.02f;    // frame units, >> the test's rounding (2.5e-3 worst case)
constexpr float kSkipMaxM = 2048.f;    // clearance cap
constexpr float kSkipMaxP0 = 6000.f;   // |P0| bound: |P| <= 8192 while skipping
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Warp-wide min / max of a float (no NaN among the inputs) in one REDUX each:
// floats order like the signed integers key(f) = bits >= 0 ? bits : bits ^
// 0x7fffffff, and the map is its own inverse.  (-0 sorts below +0; the boxes it
// feeds only take differences, where the sign of a zero is immaterial.)
#ifndef BMPC_BOX_REDUX
#define BMPC_BOX_REDUX 1  // 0: xor-shuffle butterflies
#endif
__device__ __forceinline__ int f2key(float f) {
  const int b = __float_as_int(f);
  return b >= 0 ? b : b ^ 0x7fffffff;
}
__device__ __forceinline__ float warp_fmin(float v) {
#if BMPC_BOX_REDUX
  return __int_as_float(f2key(__int_as_float(__reduce_min_sync(BMPC_FULL, f2key(v)))));
#else
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fminf(v, __shfl_xor_sync(BMPC_FULL, v, o));
  return v;
#endif
}
__device__ __forceinline__ float warp_fmax(float v) {
#if BMPC_BOX_REDUX
  return __int_as_float(f2key(__int_as_float(__reduce_max_sync(BMPC_FULL, f2key(v)))));
#else
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(BMPC_FULL, v, o));
  return v;
#endif
}
#ifndef BMPC_PF_SCALE
#define BMPC_PF_SCALE 1  // obstacles in flight with the prefilter, relative to U (2, 3: slower at c4)
#endif
// TESTIN (with TRACK, whole slots): the clearance test runs here, on the
// positions this pass has just evaluated, against the records in T.sk_p0 /
// T.sk_m0 (global scratch of the long-horizon kernels, which do not sample
// x, y in pass A); a slot whose samples are all clear returns before the loop.
template <int NS, int NB, int NPAD, bool F32, int U, bool XS, bool PAIRED, bool CULL, bool TRACK = false,
          bool TESTIN = false>
__device__ __forceinline__ void obstacle_block(const TailArgs& T, const int (&k)[NS], int j0, int js,
                                               int group, bool valid, bool leader,
                                               double (&Gx)[NB], double (&Gy)[NB], double& sqo) {
  static_assert(!TRACK || (!F32 && !BMPC_XS32 && (XS || CULL)),
                "clearance tracking: the fp64 loops (staged, or the culling survivors)");
  static_assert(!TESTIN || (TRACK && NS == 1), "in-pass clearance test: tracked single-slot passes");
  float2 tp0[NS];
  float tm0[NS];
  if constexpr (TESTIN) {  // issued first: the loads fly while x, y are evaluated
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      // (no scratch, e.g. an SM id past its range: nothing recorded, never clear)
      tp0[s] = T.sk_m0 ? T.sk_p0[k[s]] : make_float2(0.f, 0.f);
      tm0[s] = T.sk_m0 ? T.sk_m0[k[s]] : -1.f;
    }
  }
  double x[NS], y[NS], gsx[NS], gsy[NS], sq[NS];  // gsx, gsy: sum of inside residuals
  double cin[NS];                                   // inside terms per sample
  // TRACK: high word of the smallest r^2 seen per sample (positive doubles order
  // like their high words; truncation rounds down), and the smallest squared box
  // gap of the culled obstacles
  int rmn[NS];
  float cmn[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    x[s] = y[s] = gsx[s] = gsy[s] = sq[s] = cin[s] = 0.0;
    rmn[s] = 0x7fefffff;
    cmn[s] = 3.0e38f;
  }
  const double abd2 = (T.a * T.b) * (T.a * T.b);
  // r^2 of one term, its outside test (obstacle_inside_s), and the running minimum
  auto inside_t = [&](int s, double2 q) {
    const double px = x[s] - q.x, py = y[s] - q.y;
    const double r2 = fma(px, px, py * py);
    if constexpr (TRACK) rmn[s] = min(rmn[s], __double2hiint(r2));
    return !(r2 >= abd2);
  };
  if (valid) {
    if (T.xs) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        x[s] = T.xs[k[s]];
        y[s] = T.ys[k[s]];
      }
    } else {
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double2 c = T.cxy[i];
        double p[NS];
        basis1<NS, PAIRED, NPAD>(T.P, i, k, p);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          x[s] = fma(p[s], c.x, x[s]);
          y[s] = fma(p[s], c.y, y[s]);
        }
      }
    }
    // into the ellipse frame, rounded here (an explicit product: left to the
    // compiler it may fuse into the outside test's subtraction in one loop
    // variant and not in another, and the variants would differ in the last bit)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#ifdef BMPC_FRAME_CONTRACT
      x[s] *= T.b;
      y[s] *= T.a;
#else
      x[s] = __dmul_rn(x[s], T.b);
      y[s] = __dmul_rn(y[s], T.a);
#endif
    }
  }
  if constexpr (TESTIN) {
    // moved less than the recorded clearance since the slot's last pass (fp32;
    // kSkipSlack covers every rounding): every term is outside, nothing to add
    bool clear = true;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float dx = __double2float_rn(x[s]) - tp0[s].x, dy = __double2float_rn(y[s]) - tp0[s].y;
      clear &= !valid || fmaf(dx, dx, dy * dy) < tm0[s];
    }
    if (__all_sync(BMPC_FULL, clear)) return;
  }
  const double ia = T.ia, ib = T.ib;
  constexpr int UF = U * BMPC_PF_SCALE;
  BMPC_PROF_NS(10);
  const int qstep = js * T.n;
  float srx[NS], sry[NS], sqf[NS];  // fp32 mode: sum_j r_j and sum_j |r_j|^2
#pragma unroll
  for (int s = 0; s < NS; ++s) srx[s] = sry[s] = sqf[s] = 0.f;
  const float af = (float)T.a, bf = (float)T.b, ab2 = (float)(T.a * T.b * T.a * T.b);
  // CULL is a separate instantiation: the culling code compiled into the other
  // kernels costs them registers even unused (c1 +13%)
  if (CULL && js == 1) {
    // Whole (or partial, unsplit) slots: cull obstacles by bounding boxes first.
    // The warp's samples of the slot span a box (fp32, rounded outward; NaN
    // samples make it unbounded); each obstacle's samples over the same slot
    // span a precomputed box (k_obstacle_boxes, rounded outward).  When the
    // gap between the two boxes is at least ab, every term of that obstacle
    // is outside (r >= gap >= ab), contributes nothing (exact form), and is
    // skipped; the survivors take the fp64 test in increasing j, so the inside
    // terms accumulate in the same order as the full loop -- same bits.
#ifndef BMPC_UC1
#define BMPC_UC1 (NPAD > 128 ? 8 : 4)  // long horizons: c4 -2.6% at 8 (c2 +0.6%)
#endif
#ifndef BMPC_UC2
#define BMPC_UC2 2
#endif
    constexpr int UC = NS == 2 ? BMPC_UC2 : BMPC_UC1;  // surviving obstacles in flight
    float bx0[NS], bx1[NS], by0[NS], by1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      float lx = INFINITY, hx = -INFINITY, ly = INFINITY, hy = -INFINITY;
      if (valid) {
        const bool nan = x[s] != x[s] || y[s] != y[s];
        lx = nan ? -INFINITY : __double2float_rd(x[s]);
        hx = nan ? INFINITY : __double2float_ru(x[s]);
        ly = nan ? -INFINITY : __double2float_rd(y[s]);
        hy = nan ? INFINITY : __double2float_ru(y[s]);
      }
      bx0[s] = warp_fmin(lx), bx1[s] = warp_fmax(hx), by0[s] = warp_fmin(ly), by1[s] = warp_fmax(hy);
    }
    const float tc = T.tc;
    const int lane = threadIdx.x & 31;
#if defined(BMPC_CULL_PF) || BMPC_XS32
    float cxf[NS], cyf[NS];  // fp32 samples for the prefilter (NaN: never decides)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool ok = fabs(x[s]) <= (double)T.lim32 && fabs(y[s]) <= (double)T.lim32;
      cxf[s] = ok ? __double2float_rn(x[s]) : __int_as_float(0x7fc00000);
      cyf[s] = __double2float_rn(y[s]);
    }
#endif
    for (int c0 = 0; c0 < T.m; c0 += 32) {
      const int jl = c0 + lane;
      bool keep = false;
      float g2[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) g2[s] = 0.f;
      if (jl < T.m) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const float4 bo = __ldg(T.box + (k[s] >> 5) * T.m + jl);
          const float gx = fmaxf(fmaxf(bo.x - bx1[s], bx0[s] - bo.y), 0.f);
          const float gy = fmaxf(fmaxf(bo.z - by1[s], by0[s] - bo.w), 0.f);
          g2[s] = fmaf(gx, gx, gy * gy);
          keep |= !(g2[s] >= tc);
        }
      }
      if constexpr (TRACK) {
        // culled obstacles: every sample of the slot is at least the box gap away
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int cg = (jl < T.m && !keep) ? __float_as_int(g2[s]) : 0x7f7fffff;
          cmn[s] = fminf(cmn[s], __int_as_float(__reduce_min_sync(BMPC_FULL, cg)));
        }
      }
      unsigned bits = __ballot_sync(BMPC_FULL, keep);
      while (bits) {
        int jj[UC];
        bool on[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          on[u] = bits != 0u;
          jj[u] = on[u] ? c0 + __ffs(bits) - 1 : 0;
          bits &= bits - 1u;
        }
#if defined(BMPC_CULL_PF) || BMPC_XS32
        // survivors through the fp32 prefilter (unstaged predictions, or the
        // staged fp32 copies): the pairs take half the registers, the fp64
        // pair only when undecided
#ifdef BMPC_CULL_PF
        constexpr bool kCullPf = !XS || BMPC_XS32;
#else
        constexpr bool kCullPf = XS;
#endif
        if constexpr (kCullPf) {
          float2 qf[NS][UC];
#pragma unroll
          for (int u = 0; u < UC; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              qf[s][u] = (on[u] && valid) ? ldq<XS>(T.xf + jj[u] * T.n + k[s]) : make_float2(0.f, 0.f);
          if (valid) {
#pragma unroll
            for (int u = 0; u < UC; ++u)
#pragma unroll
              for (int s = 0; s < NS; ++s) {
                // cxf is NaN past the prefilter bound: such samples never decide
                const float dx = cxf[s] - qf[s][u].x, dy = cyf[s] - qf[s][u].y;
                if (on[u] && !(fmaf(dx, dx, dy * dy) >= T.t32)) {
                  const double2 q = __ldg(T.xi + jj[u] * T.n + k[s]);
                  if (obstacle_inside_s(x[s], y[s], q, abd2)) {
                    if constexpr (F32)
                      obstacle_term_f32(x[s], y[s], q, af, bf, ab2, ia, ib, srx[s], sry[s], sqf[s], cin[s]);
                    else
                      obstacle_inside_res_s(x[s], y[s], q, T.a, T.b, ia, ib, gsx[s], gsy[s], sq[s], cin[s]);
                  }
                }
              }
          }
        } else
#endif
        {
        double2 q[NS][UC];
#pragma unroll
        for (int u = 0; u < UC; ++u)
#pragma unroll
          for (int s = 0; s < NS; ++s)
            q[s][u] = (on[u] && valid) ? ldq<XS>(T.xi + jj[u] * T.n + k[s]) : make_double2(0.0, 0.0);
        if (valid) {
#pragma unroll
          for (int u = 0; u < UC; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (on[u] && inside_t(s, q[s][u])) {
                if constexpr (F32)
                  obstacle_term_f32(x[s], y[s], q[s][u], af, bf, ab2, ia, ib, srx[s], sry[s], sqf[s],
                                    cin[s]);
                else
                  obstacle_inside_res_s(x[s], y[s], q[s][u], T.a, T.b, ia, ib, gsx[s], gsy[s], sq[s],
                                        cin[s]);
              }
        }
        }
      }
    }
  } else if (valid) {
#ifdef BMPC_NO_PREFILTER
    constexpr bool kFp64Loop = true;
#else
    constexpr bool kFp64Loop = XS && !BMPC_XS32;
#endif
    if constexpr (kFp64Loop) {
    // predictions staged in shared memory: the fp64 test straight away (LDS
    // latency; the prefilter measured slower here)
    const double2* qp[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) qp[s] = T.xi + j0 * T.n + k[s];
    int j = j0;
    double2 qn[NS][U];
    if (j + (U - 1) * js < T.m) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) qn[s][u] = ldq<XS>(qp[s] + u * qstep);
    }
#pragma unroll 1
    for (; j + (U - 1) * js < T.m; j += U * js) {
      double2 q[NS][U];
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) q[s][u] = qn[s][u];
      if (j + (2 * U - 1) * js < T.m) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int u = 0; u < U; ++u) qn[s][u] = ldq<XS>(qp[s] + (U + u) * qstep);
      }
      {
        // outside test in fp64 for both modes; the rare inside terms in the
        // mode's precision
        bool in[NS][U], any = false;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            in[s][u] = inside_t(s, q[s][u]);
            any |= in[s][u];
          }
        if (any) {
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (in[s][u]) {
                if constexpr (F32)
                  obstacle_term_f32(x[s], y[s], q[s][u], af, bf, ab2, ia, ib, srx[s], sry[s], sqf[s],
                                    cin[s]);
                else
                  obstacle_inside_res_s(x[s], y[s], q[s][u], T.a, T.b, ia, ib, gsx[s], gsy[s], sq[s],
                                        cin[s]);
              }
        }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) qp[s] += U * qstep;
    }
    for (; j < T.m; j += js) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double2 q = ldq<XS>(qp[s]);
        if (inside_t(s, q)) {
          if constexpr (F32)
            obstacle_term_f32(x[s], y[s], q, af, bf, ab2, ia, ib, srx[s], sry[s], sqf[s], cin[s]);
          else
            obstacle_inside_res_s(x[s], y[s], q, T.a, T.b, ia, ib, gsx[s], gsy[s], sq[s], cin[s]);
        }
        qp[s] += qstep;
      }
    }
    } else {
    // Predictions from L2 (not staged): an exact fp32 prefilter (common.cuh prefilter_lim): a term is decided
    // "outside" from the fp32 pairs when r2f >= t32 and the sample's
    // coordinates are within the bound; every other term (the boundary band,
    // the inside terms, large or non-finite coordinates) loads its fp64 pair
    // and takes the fp64 test, so the decisions -- and the order the inside
    // terms accumulate in -- are those of the fp64 loop.
    float xf[NS], yf[NS];
    const float lim = T.lim32, t32 = T.t32;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool ok = fabs(x[s]) <= (double)lim && fabs(y[s]) <= (double)lim;
      xf[s] = ok ? __double2float_rn(x[s]) : __int_as_float(0x7fc00000);  // NaN: never decides
      yf[s] = __double2float_rn(y[s]);
    }
    // UF obstacles in flight per sample (the fp32 pairs take half the registers)
    const float2* qp[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) qp[s] = T.xf + j0 * T.n + k[s];
    // the fp64 test of one undecided term (obstacle jj of sample s)
    auto slow = [&](int s, int jj) {
      const double2 q = __ldg(T.xi + jj * T.n + k[s]);
#ifdef BMPC_PF_DEBUG
      if (obstacle_inside_s(x[s], y[s], q, abd2) && blockIdx.x == 0 && threadIdx.x < 32)
        printf("PF inside blk0 lane=%d k=%d j=%d\n", threadIdx.x, k[s], jj);
#endif
      if (obstacle_inside_s(x[s], y[s], q, abd2)) {
        if constexpr (F32)
          obstacle_term_f32(x[s], y[s], q, af, bf, ab2, ia, ib, srx[s], sry[s], sqf[s], cin[s]);
        else
          obstacle_inside_res_s(x[s], y[s], q, T.a, T.b, ia, ib, gsx[s], gsy[s], sq[s], cin[s]);
      }
    };
    int j = j0;
    // software pipeline: the next group's predictions are in flight while the
    // current group computes (xi comes from L2 once it outgrows L1, e.g. c4)
    float2 qn[NS][UF];
    if (j + (UF - 1) * js < T.m) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < UF; ++u) qn[s][u] = ldq<XS>(qp[s] + u * qstep);
    }
#pragma unroll 1
    for (; j + (UF - 1) * js < T.m; j += UF * js) {
      float2 q[NS][UF];
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < UF; ++u) q[s][u] = qn[s][u];
      if (j + (2 * UF - 1) * js < T.m) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int u = 0; u < UF; ++u) qn[s][u] = ldq<XS>(qp[s] + (UF + u) * qstep);
      }
      {
        bool und[NS][UF], any = false;
#pragma unroll
        for (int u = 0; u < UF; ++u)
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const float dx = xf[s] - q[s][u].x, dy = yf[s] - q[s][u].y;
            und[s][u] = !(fmaf(dx, dx, dy * dy) >= t32);
            any |= und[s][u];
#ifdef BMPC_PF_DEBUG
            {
              const int jj = j + u * js;
              const double2 q64 = __ldg(T.xi + jj * T.n + k[s]);
              if (!und[s][u] && obstacle_inside_s(x[s], y[s], q64, abd2))
                printf("PF mismatch k=%d j=%d x=%.17g y=%.17g q=(%.17g,%.17g) qf=(%.9g,%.9g) xf=(%.9g,%.9g)\n",
                       k[s], jj, x[s], y[s], q64.x, q64.y, q[s][u].x, q[s][u].y, xf[s], yf[s]);
            }
#endif
          }
        if (any) {
#pragma unroll
          for (int u = 0; u < UF; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (und[s][u]) slow(s, j + u * js);
        }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) qp[s] += UF * qstep;
    }
    for (; j < T.m; j += js) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const float2 q = ldq<XS>(qp[s]);
        const float dx = xf[s] - q.x, dy = yf[s] - q.y;
#ifdef BMPC_PF_DEBUG
        {
          const double2 q64 = __ldg(T.xi + j * T.n + k[s]);
          if ((fmaf(dx, dx, dy * dy) >= t32) && obstacle_inside_s(x[s], y[s], q64, abd2))
            printf("PF tail mismatch k=%d j=%d\n", k[s], j);
        }
#endif
        if (!(fmaf(dx, dx, dy * dy) >= t32)) slow(s, j);
        qp[s] += qstep;
      }
    }
    }
  }
  if (valid) {
    if constexpr (F32) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        gsx[s] = (double)srx[s];
        gsy[s] = (double)sry[s];
        sq[s] = (double)sqf[s];
      }
    }
    }
  BMPC_PROF_NS(11);
  if (NS == 1 && group > 1) {  // split slot: combine the group's partial sums
    for (int o = 1; o < group; o <<= 1) {
      gsx[0] += __shfl_xor_sync(BMPC_FULL, gsx[0], o);
      gsy[0] += __shfl_xor_sync(BMPC_FULL, gsy[0], o);
      sq[0] += __shfl_xor_sync(BMPC_FULL, sq[0], o);
      cin[0] += __shfl_xor_sync(BMPC_FULL, cin[0], o);
      if constexpr (TRACK) rmn[0] = min(rmn[0], __shfl_xor_sync(BMPC_FULL, rmn[0], o));
    }
  }
  if constexpr (TRACK) {
    // record the slot's clearances: M0 <= min_j |P0 - Q_j| - ab - slack, every
    // step rounded down; a sample with an inside (or NaN) term, out of the
    // coordinate bound, or without clearance never skips (M0^2 stored as -1)
    if (valid && leader && (!TESTIN || T.sk_m0)) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const float r2f = fminf(__double2float_rd(__hiloint2double(rmn[s], 0)), cmn[s]);
        // MUFU sqrt (2 ulp) scaled below the true root
        const float r0 = fminf(__fmul_rd(sqrt_approx(r2f), 1.f - 1e-6f), kSkipMaxM);
        const float M = __fsub_rd(__fsub_rd(r0, T.ab_ru), kSkipSlack);
        const float X0 = __double2float_rn(x[s]), Y0 = __double2float_rn(y[s]);
        const bool ok = M > 0.f && !(cin[s] > 0.0) && fabsf(X0) <= kSkipMaxP0 && fabsf(Y0) <= kSkipMaxP0;
        T.sk_p0[k[s]] = make_float2(X0, Y0);
        T.sk_m0[k[s]] = ok ? __fmul_rd(M, M) : -1.f;
      }
    }
  }
  // P^T sum_j g_j = m (P^T P) c - P^T sum_inside r_j: only samples with an inside
  // term contribute here (the m (P^T P) c part is added once per sweep); the
  // contraction runs only when some lane of the warp has one
  const bool own = valid && leader;
  bool any = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sqo += own ? sq[s] : 0.0;
    any |= own && cin[s] > 0.0;
    gsx[s] = own ? -gsx[s] : 0.0;
    gsy[s] = own ? -gsy[s] : 0.0;
  }
  if (__any_sync(BMPC_FULL, any)) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      double p[NS];
      basis1<NS, PAIRED, NPAD>(T.P, i, k, p);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        Gx[i] = fma(p[s], gsx[s], Gx[i]);
        Gy[i] = fma(p[s], gsy[s], Gy[i]);
      }
    }
  }
  BMPC_PROF_NS(13);
}

// ---------------------------------------------------------------------------
// fp32 mode obstacle block (BMPC_F_F32): the exact form of the fp64 block in
// single precision.  Positions come from pass A's fp32 ellipse-frame samples,
// predictions from the fp32 ellipse-frame copy (xs32, NaN past the prefilter
// bound); a term whose fp32 r^2 is NaN (that bound, or a NaN input) takes the
// fp64 test on the fp64 pair, so non-finite values propagate as in fp64 mode
// and far predictions never decide in fp32.  The inside residuals r_j =
// w - (a cos, b sin) and their squares accumulate in fp32 per lane.
struct TailArgs32 {
  const float* P;            // fp32 basis (shared memory)
  const float *xs, *ys;      // pass A's ellipse-frame samples (b x, a y)
  const float2* xf;          // fp32 ellipse-frame predictions (global)
  const double2* xi;         // fp64 ellipse-frame predictions (NaN fallback)
  int n, m;
  float a, b, ia, ib, ab2;   // ab2 = (ab)^2 rounded to fp32
  double da, db, dia, dib, dab2;
  const float4* box;         // [slot][m] obstacle boxes (culling) or nullptr
  float tc;
  float2* sk_p0;             // clearance skipping (BMPC_SKIP), as in TailArgs
  float* sk_m0;
  float ab_ru;
};

template <int NS>
__device__ __forceinline__ void obstacle_term32(const TailArgs32& T, float px, float py, float r2,
                                                float& srx, float& sry, float& sq) {
  const float ri = rsqrtf(r2);
  const bool pos = r2 > 0.f;  // r = 0 -> (cos, sin) = (1, 0) (_speedups.pyx:158-166)
  const float ca = pos ? px * ri : 1.f, sa = pos ? py * ri : 0.f;
  const float rx = fmaf(px, T.ib, -T.a * ca), ry = fmaf(py, T.ia, -T.b * sa);
  sq = fmaf(rx, rx, fmaf(ry, ry, sq));
  srx += rx;
  sry += ry;
}

template <int NS, int NB, int NPAD, int U, bool PAIRED, bool CULL, bool TRACK = false>
__device__ __forceinline__ void obstacle_block_f32(const TailArgs32& T, const int (&k)[NS], int j0, int js,
                                                   int group, bool valid, bool leader, float (&Gx)[NB],
                                                   float (&Gy)[NB], float& sqo) {
  float x[NS], y[NS], srx[NS], sry[NS], sq[NS];
  bool hit[NS];
  float rmn[NS];  // TRACK: smallest r^2 per sample (fminf drops NaN: those terms set `hit`)
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    x[s] = valid ? T.xs[k[s]] : 0.f;
    y[s] = valid ? T.ys[k[s]] : 0.f;
    srx[s] = sry[s] = sq[s] = 0.f;
    hit[s] = false;
    rmn[s] = 3.0e38f;
  }
  // one term of obstacle jj at sample s, prediction q
  auto term = [&](int s, float2 q, int jj) {
    const float px = x[s] - q.x, py = y[s] - q.y;
    const float r2 = fmaf(px, px, py * py);
    if constexpr (TRACK) rmn[s] = fminf(rmn[s], r2);
    if (!(r2 >= T.ab2)) {  // inside, or NaN
      if (r2 == r2) {
        obstacle_term32<NS>(T, px, py, r2, srx[s], sry[s], sq[s]);
        hit[s] = true;
      } else {  // rare: the fp64 test and term on the fp64 pair
        if constexpr (TRACK) hit[s] = true;  // undecidable in fp32: the sample never skips
        const double2 q64 = __ldg(T.xi + jj * T.n + k[s]);
        const double dx = (double)x[s] - q64.x, dy = (double)y[s] - q64.y;
        const double d2 = fma(dx, dx, dy * dy);
        if (!(d2 >= T.dab2)) {
          const double ri = rsqrt_nb(d2);
          const double ca = d2 > 0.0 ? dx * ri : 1.0, sa = dy * ri;
          const double rx = fma(dx, T.dib, -T.da * ca), ry = fma(dy, T.dia, -T.db * sa);
          sq[s] = (float)fma(rx, rx, fma(ry, ry, (double)sq[s]));
          srx[s] += (float)rx;
          sry[s] += (float)ry;
          hit[s] = true;
        }
      }
    }
  };
  const int qstep = js * T.n;
  if (CULL && js == 1) {
    // whole slots: cull obstacles whose box is at least ab away from the
    // warp's sample box (the fp32 samples are exact values: no outward rounding)
    constexpr int UC = NS == 2 ? 2 : (NPAD > 128 ? 8 : 4);
    float bx0[NS], bx1[NS], by0[NS], by1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      float lx = INFINITY, hx = -INFINITY, ly = INFINITY, hy = -INFINITY;
      if (valid) {
        const bool nan = x[s] != x[s] || y[s] != y[s];
        lx = nan ? -INFINITY : x[s];
        hx = nan ? INFINITY : x[s];
        ly = nan ? -INFINITY : y[s];
        hy = nan ? INFINITY : y[s];
      }
      bx0[s] = warp_fmin(lx), bx1[s] = warp_fmax(hx), by0[s] = warp_fmin(ly), by1[s] = warp_fmax(hy);
    }
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < T.m; c0 += 32) {
      const int jl = c0 + lane;
      bool keep = false;
      float g2[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) g2[s] = 0.f;
      if (jl < T.m) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const float4 bo = __ldg(T.box + (k[s] >> 5) * T.m + jl);
          const float gx = fmaxf(fmaxf(bo.x - bx1[s], bx0[s] - bo.y), 0.f);
          const float gy = fmaxf(fmaxf(bo.z - by1[s], by0[s] - bo.w), 0.f);
          g2[s] = fmaf(gx, gx, gy * gy);
          keep |= !(g2[s] >= T.tc);
        }
      }
      if constexpr (TRACK) {  // culled obstacles: at least the box gap away
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int cg = (jl < T.m && !keep) ? __float_as_int(g2[s]) : 0x7f7fffff;
          rmn[s] = fminf(rmn[s], __int_as_float(__reduce_min_sync(BMPC_FULL, cg)));
        }
      }
      unsigned bits = __ballot_sync(BMPC_FULL, keep);
      while (bits) {
        int jj[UC];
        bool on[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          on[u] = bits != 0u;
          jj[u] = on[u] ? c0 + __ffs(bits) - 1 : 0;
          bits &= bits - 1u;
        }
        float2 q[NS][UC];
#pragma unroll
        for (int u = 0; u < UC; ++u)
#pragma unroll
          for (int s = 0; s < NS; ++s)
            q[s][u] = (on[u] && valid) ? __ldg(T.xf + jj[u] * T.n + k[s]) : make_float2(1e30f, 1e30f);
        if (valid) {
#pragma unroll
          for (int u = 0; u < UC; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (on[u]) term(s, q[s][u], jj[u]);
        }
      }
    }
  } else if (valid) {
    const float2* qp[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) qp[s] = T.xf + j0 * T.n + k[s];
    int j = j0;
    // software pipeline: the next group's predictions in flight (L2)
    float2 qn[NS][U];
    if (j + (U - 1) * js < T.m) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) qn[s][u] = __ldg(qp[s] + u * qstep);
    }
#pragma unroll 1
    for (; j + (U - 1) * js < T.m; j += U * js) {
      float2 q[NS][U];
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) q[s][u] = qn[s][u];
      if (j + (2 * U - 1) * js < T.m) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int u = 0; u < U; ++u) qn[s][u] = __ldg(qp[s] + (U + u) * qstep);
      }
      bool any = false;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const float px = x[s] - q[s][u].x, py = y[s] - q[s][u].y;
          const float r2 = fmaf(px, px, py * py);
          if constexpr (TRACK) rmn[s] = fminf(rmn[s], r2);
          any |= !(r2 >= T.ab2);
        }
      if (any) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int s = 0; s < NS; ++s) term(s, q[s][u], j + u * js);
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) qp[s] += U * qstep;
    }
    for (; j < T.m; j += js) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        term(s, __ldg(qp[s]), j);
        qp[s] += qstep;
      }
    }
  }
  if (NS == 1 && group > 1) {  // split slot: combine the group's partial sums
    for (int o = 1; o < group; o <<= 1) {
      srx[0] += __shfl_xor_sync(BMPC_FULL, srx[0], o);
      sry[0] += __shfl_xor_sync(BMPC_FULL, sry[0], o);
      sq[0] += __shfl_xor_sync(BMPC_FULL, sq[0], o);
      hit[0] |= __shfl_xor_sync(BMPC_FULL, (int)hit[0], o) != 0;
      if constexpr (TRACK) rmn[0] = fminf(rmn[0], __shfl_xor_sync(BMPC_FULL, rmn[0], o));
    }
  }
  if constexpr (TRACK) {
    // record the slot's clearances (as the fp64 block does): the fp32 test of a
    // later sweep says outside for every term while the sample stays within
    // M0 <= min_j |P0 - Q_j| (1 - 1e-5) - ab (1 + 1e-5) - slack of P0
    if (valid && leader) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const float r0 = fminf(__fmul_rd(sqrt_approx(rmn[s]), 1.f - 1e-5f), kSkipMaxM);
        const float M = __fsub_rd(__fsub_rd(r0, __fmul_ru(T.ab_ru, 1.f + 1e-5f)), kSkipSlack);
        const bool ok = M > 0.f && !hit[s] && fabsf(x[s]) <= kSkipMaxP0 && fabsf(y[s]) <= kSkipMaxP0;
        T.sk_p0[k[s]] = make_float2(x[s], y[s]);
        T.sk_m0[k[s]] = ok ? __fmul_rd(M, M) : -1.f;
      }
    }
  }
  // P^T sum_j g_j = m (P^T P) c - P^T sum_inside r_j (the Gram part in fp64, (6))
  const bool own = valid && leader;
  bool any = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sqo += own ? sq[s] : 0.f;
    any |= own && hit[s];
    srx[s] = own ? -srx[s] : 0.f;
    sry[s] = own ? -sry[s] : 0.f;
  }
  if (__any_sync(BMPC_FULL, any)) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      float p[NS];
      basis1<NS, PAIRED, NPAD>(T.P, i, k, p);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        Gx[i] = fmaf(p[s], srx[s], Gx[i]);
        Gy[i] = fmaf(p[s], sry[s], Gy[i]);
      }
    }
  }
}

template <int NB, int NKM, bool F32, bool TEAMS, bool XS, bool CULL>
#ifndef BMPC_MINB
#define BMPC_MINB 1
#endif
#ifndef BMPC_TEAM_MINB
#define BMPC_TEAM_MINB 1
#endif
#ifndef BMPC_MAXT
#define BMPC_MAXT (32 * BMPC_MAX_WARPS)
#endif
__global__ void __launch_bounds__(BMPC_MAXT, TEAMS ? BMPC_TEAM_MINB : BMPC_MINB) am_solve_kernel(const bmpc_dev_consts C,
                                                       const bmpc_solve_args A) {
  extern __shared__ __align__(16) double sm[];
  // device-decided sweep count (the early-stop re-run): 0 = nothing to do
  const int iters = A.iters_dev ? *A.iters_dev : A.iters;
  if (iters <= 0) return;
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  BMPC_PROF_DECL
  const int n = C.n;
  constexpr int npad = 32 * NKM;  // host pads the basis to exactly this
  constexpr int nk = NKM;
  const int L = A.L;
  constexpr int RX = NB + 6, RP = NB + 4;

  constexpr bool kStoreXY = bmpc_stores_xy(npad);  // else the obstacle block re-evaluates x, y
#ifndef BMPC_CH
#define BMPC_CH 2
#endif
  constexpr int CH = NKM < BMPC_CH ? NKM : BMPC_CH;  // sample slots per pass A / B chunk
#ifndef BMPC_CHUNK_UNROLL_A
// chunks stay rolled: the sweep loop must fit the 32 KB instruction cache
// (two chunks in flight overlapped one chunk's atan2 with the next one's
// sampling, -1%, but the larger loop cost 2-8% in instruction fetch stalls)
#define BMPC_CHUNK_UNROLL_A 1
#endif
#ifndef BMPC_CHUNK_UNROLL_B
#define BMPC_CHUNK_UNROLL_B 1
#endif
  constexpr int kChunkUnrollA = BMPC_CHUNK_UNROLL_A, kChunkUnrollB = BMPC_CHUNK_UNROLL_B;
  // Odd slot counts (n_b = 16 at c4: seven slots): the last chunk repeats the
  // last slot, masked, instead of a separate one-slot body in the hot loop.
#ifndef BMPC_ODD_DUP
#define BMPC_ODD_DUP 0
#endif
  constexpr bool kOddDup = BMPC_ODD_DUP && !TEAMS && !F32 && CH == 2 && (NKM & 1) && NKM > 2;
  // constant image (am_args.h, capi.cu bmpc_ctx_create)
  // basis rows in paired-slot order when npad is a whole number of slot pairs
  // (bmpc_basis_index); two-slot chunks are then even slot pairs (one warp per
  // instance)
  constexpr bool PAIRED = !TEAMS && (npad % 64) == 0;
  // fp32 mode: the basis sits in shared memory in fp32 (half the bytes); the
  // few fp64 basis reads (initial targets, fused scoring) go to the global image
  constexpr int kBasisD = bmpc_basis_doubles(NB, npad, F32);
  double* sPT = sm;                  // P^T, Pdot^T, Pddot^T (fp64 mode)
  double* sM = sPT + kBasisD;        // m P^T P + Pddot^T Pddot (+ Pdot^T Pdot in fp32 mode)
  double* sMp = sM + NB * C.kms;     // P^T P
  double* sMdd = sMp + NB * C.kms;   // Pddot^T Pddot
  double* sMd = sMdd + NB * C.kms;   // Pdot^T Pdot
  double* sZx = sMd + NB * C.kms;    // H_mm^-1 of the xy QP in full index space
  double* sHx = sZx + NB * C.kms;    // H = Q + rho F_axis^T F_axis (refinement)
  double* sZp = sHx + NB * C.kms;    // the same for the psi QP
  double* sHp = sZp + NB * C.kms;
  double* sBx = sHp + NB * C.kms;    // [NB][8]: c = Z rhs + B b (boundary map)
  double* sBp = sBx + 8 * NB;        // [NB][4]
  double* sTau = sBp + 4 * NB;       // even offset: the double2 scratch stays 16-byte aligned
  // team = the TW warps sharing one instance; each keeps private KKT vectors,
  // transpose buffer and exchange slots, the per-sample arrays are shared
  const int TW = TEAMS ? A.team : 1;  // compile-time 1 outside the team build
  const int team = warp / TW, wt = warp - team * TW;
  double* tbase = sTau + npad + team * bmpc_team_doubles(npad, TW);
  double* wbase = tbase + wt * bmpc_warp_private_doubles();
  double* arr = tbase + TW * bmpc_warp_private_doubles();
  WarpScratch ws{wbase,       wbase + 32,   wbase + 48,
                 arr,         arr + npad,   arr + 2 * npad,
                 kStoreXY ? arr + 3 * npad : nullptr, kStoreXY ? arr + 4 * npad : nullptr,
                 wbase + kWarpScratch};
  // exchange slots of team warp w: [0, 32) P^T theta, [32, 64) G, [64, 67) squared
  // residuals, [67] unwrap flag
  auto xch_of = [&](int w) { return tbase + w * bmpc_warp_private_doubles() + kWarpScratch + kRedSize; };
  double* xch = xch_of(wt);
  // named barrier 1 + team (a block holds at most 4 teams: W <= 8, TW >= 2);
  // immediate ids so ptxas reserves only barriers 0-4
  auto team_sync = [&]() {
    if (TW == 1) return;
    const int nt = TW * 32;
    switch (team) {
      case 0: asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory"); break;
      case 1: asm volatile("bar.sync 2, %0;" ::"r"(nt) : "memory"); break;
      case 2: asm volatile("bar.sync 3, %0;" ::"r"(nt) : "memory"); break;
      default: asm volatile("bar.sync 4, %0;" ::"r"(nt) : "memory"); break;
    }
  };
  const SlotLayout sl = slot_layout(n);
  const int nslots = sl.F + (sl.R > 0 ? 1 : 0);

  // The constant block (basis, KKT pairs, M, P^T P, tau) is one contiguous
  // image in global memory laid out exactly like shared memory: one thread
  // streams it in with bulk asynchronous copies (TMA, cp.async.bulk) that
  // complete on an mbarrier, instead of every warp issuing the loads.
  __shared__ __align__(8) unsigned long long s_cbar;
  // XS: this block's scene(s) of ellipse-frame predictions ride in the same
  // bulk transfer, after the scratch (instances blockIdx.x * ipb ... span at
  // most two scenes, xs_stage_bytes in am_inst.cu)
  const int ipb = W / TW;
  const int first_inst = blockIdx.x * ipb;
  const int scene0 = first_inst / A.l;
  const int img_doubles = C.const_doubles - 3 * NB * npad + kBasisD;  // in shared memory
  double* sXi = sm + img_doubles + (size_t)ipb * bmpc_team_doubles(npad, TW);
  // clearance skipping (BMPC_SKIP): per warp, behind the staged predictions,
  // npad (P0.x, P0.y) fp32 pairs and npad squared clearances (am_inst.cu
  // xs_stage_bytes sizes both)
  // fp32 mode: every shape (no staging; am_solve_smem_bytes sizes the arrays)
  constexpr bool SKIP = BMPC_SKIP && !TEAMS && !BMPC_XS32 && (F32 || (XS && kStoreXY));
  // Long horizons in fp64 (unstaged predictions, culling; shared memory is
  // full): the same records in a global scratch indexed by SM and warp (one
  // block per SM), the test inside the obstacle pass (x, y are evaluated there).
#ifndef BMPC_SKIPG
#define BMPC_SKIPG 1
#endif
  constexpr bool SKIPG = BMPC_SKIP && BMPC_SKIPG && !SKIP && !TEAMS && !BMPC_XS32 && !F32 && !XS && CULL && !kStoreXY;
  float2* sk_p0 = nullptr;
  float* sk_m0 = nullptr;
  if constexpr (SKIPG) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    if (A.skipg && smid < BMPC_SKIPG_SMS) {
      char* base = reinterpret_cast<char*>(A.skipg) + ((size_t)smid * BMPC_MAX_WARPS + warp) * npad * 12;
      sk_p0 = reinterpret_cast<float2*>(base);
      sk_m0 = reinterpret_cast<float*>(base + (size_t)npad * 8);
    }
  }
  if constexpr (SKIP) {
    const int last_inst = min(A.L, first_inst + ipb) - 1;
    const size_t xb = XS ? (size_t)(last_inst / A.l - scene0 + 1) * A.m * n * 16 : 0;
    char* base = reinterpret_cast<char*>(sXi) + xb + (size_t)warp * npad * 12;
    sk_p0 = reinterpret_cast<float2*>(base);
    sk_m0 = reinterpret_cast<float*>(base + (size_t)npad * 8);
  }
  if (threadIdx.x == 0) {
    // fp32 mode: the fp32 basis, then the image past its fp64 basis
    const unsigned bbytes = (unsigned)kBasisD * 8u;
    const unsigned bytes = (unsigned)img_doubles * 8u;
    unsigned xbytes = 0;
    if constexpr (XS) {
      const int last_inst = min(A.L, first_inst + ipb) - 1;
      xbytes = (unsigned)((last_inst / A.l - scene0 + 1) * A.m * n * (BMPC_XS32 ? 8 : 16));
    }
    mbar_init(&s_cbar, 1);
    mbar_arrive_expect_tx(&s_cbar, bytes + xbytes);
    constexpr unsigned kChunk = 16384;
    const char* src0 = F32 ? reinterpret_cast<const char*>(C.IMGF) : reinterpret_cast<const char*>(C.IMG);
    const char* src1 = reinterpret_cast<const char*>(C.IMG + 3 * NB * npad);
    for (unsigned o = 0; o < bbytes; o += kChunk)
      bulk_copy_g2s(reinterpret_cast<char*>(sm) + o, src0 + o, min(kChunk, bbytes - o), &s_cbar);
    for (unsigned o = bbytes; o < bytes; o += kChunk)
      bulk_copy_g2s(reinterpret_cast<char*>(sm) + o, src1 + (o - bbytes), min(kChunk, bytes - o), &s_cbar);
    if constexpr (XS) {
      const char* src = BMPC_XS32 ? reinterpret_cast<const char*>(A.xs32) + (size_t)scene0 * A.m * n * 8
                                  : reinterpret_cast<const char*>(A.xis) + (size_t)scene0 * A.m * n * 16;
      for (unsigned o = 0; o < xbytes; o += kChunk)
        bulk_copy_g2s(reinterpret_cast<char*>(sXi) + o, src + o, xbytes - o < kChunk ? xbytes - o : kChunk,
                      &s_cbar);
    }
  }
  __syncthreads();  // the initialised barrier is visible to every thread
  mbar_wait_parity(&s_cbar, 0);
  {
    // the G Gram block of this launch's obstacle count: m P^T P + Pddot^T Pddot
    // (overwrites the image's F_axis^T F_axis block, which the sweep never reads)
    const double md = (double)A.m;
    double* g = sm + kBasisD;
    // fp32 mode: + Pdot^T Pdot, the whole F_axis^T F_axis (its sweep adds only
    // the small residual contractions to it, see (6))
    for (int q = threadIdx.x; q < NB * C.kms; q += blockDim.x)
      g[q] = F32 ? fma(md, g[NB * C.kms + q], g[2 * NB * C.kms + q]) + g[3 * NB * C.kms + q]
                 : fma(md, g[NB * C.kms + q], g[2 * NB * C.kms + q]);
    __syncthreads();
  }

  const int inst = blockIdx.x * (W / TW) + team;
  if (inst >= L) return;  // team-uniform; no block-wide barriers below this point
  // Lockstep: on long horizons (n > 128) the sweep loop outgrows the 32 KB
  // instruction cache (c4: ~47 KB hot, 35-55% of the stall samples waiting for
  // instructions), so the block's live warps meet at phase boundaries of each
  // sweep (named barrier 5): they run the same code at the same time and share
  // the lines they fetch (c4 fp32 -3.5%, fp64 -1.5%).  Shorter horizons fit the
  // cache and lose latency hiding instead (c1 +3%, c3 +7%): off there.
  // Level 1: one meeting per sweep; 2: also around the obstacle block.
#ifndef BMPC_LOCKSTEP
#define BMPC_LOCKSTEP -1  // auto
#endif
  constexpr int kLockstep = TEAMS ? 0 : BMPC_LOCKSTEP >= 0 ? BMPC_LOCKSTEP : npad > 128 ? (F32 ? 2 : 1) : 0;
  const int live_threads = 32 * min(W, (L - blockIdx.x * (W / TW)) * TW);
  auto lockstep = [&](int level) {
    if (kLockstep >= level) asm volatile("bar.sync 5, %0;" ::"r"(live_threads) : "memory");
  };

  // fp64 basis: shared memory, or the global image in the fp32 mode (read only
  // by the initial targets and the fused scoring there)
  const double* __restrict__ sP = F32 ? C.IMG : sPT;
  const double* __restrict__ sPd = sP + NB * npad;
  const double* __restrict__ sPdd = sP + 2 * NB * npad;
  // fp32 mode: the shared-memory basis, per-sample arrays and coefficient copies
  const float* __restrict__ fP = reinterpret_cast<const float*>(sm);
  const float* __restrict__ fPd = fP + NB * npad;
  const float* __restrict__ fPdd = fP + 2 * NB * npad;
  float* const fth = reinterpret_cast<float*>(arr);  // theta
  float* const fxd = fth + npad;                      // xdot, ydot
  float* const fyd = fxd + npad;
  float* const fxs = fyd + npad;                      // ellipse-frame b x, a y
  float* const fys = fxs + npad;
  float* const fcxy = fys + npad;                     // 32: (c_x[i], c_y[i]) pairs
  float* const fcp = fcxy + 32;                       // 16: c_psi
  using R = std::conditional_t<F32, float, double>;   // sample-pass arithmetic
  // basis value (row i of sP / sPd / sPdd) at sample k
  auto bi = [](int i, int k) { return bmpc_basis_index(i, k, npad); };
  const double2* __restrict__ xi =
      reinterpret_cast<const double2*>(A.xi) + (size_t)(inst / A.l) * A.m * n;
  const double2* __restrict__ xis =
      (XS && !BMPC_XS32) ? reinterpret_cast<const double2*>(sXi) + (size_t)(inst / A.l - scene0) * A.m * n
                         : reinterpret_cast<const double2*>(A.xis) + (size_t)(inst / A.l) * A.m * n;
  const float2* __restrict__ xf =
      (XS && BMPC_XS32) ? reinterpret_cast<const float2*>(sXi) + (size_t)(inst / A.l - scene0) * A.m * n
                        : reinterpret_cast<const float2*>(A.xs32) + (size_t)(inst / A.l) * A.m * n;
  const int m = A.m;
  const double a = A.a, b = A.b, rho = C.rho;
  const double inv_a = 1.0 / a, inv_b = 1.0 / b;

  const int li = lane & 15;
  const bool yax = lane >= 16;
  const bool owner = li < NB;
  // lanes holding the three block residuals after each sweep's reduction
  constexpr bool kSqCols = NB + 3 <= 16;
  constexpr int sq_lane0 = kSqCols ? NB : 16;
  const bool is_sq_lane = lane >= sq_lane0 && lane < sq_lane0 + 3;

  // persistent per-lane state (owner lanes)
  double lam = 0.0, G = 0.0;   // lane i: lambda_x[i], G_x[i]; lane 16+i: lambda_y[i], G_y[i]
  double lamp = 0.0;           // lane i: lambda_psi[i]
  double bnd = 0.0, bps = 0.0;
  double cown = 0.0, cpown = 0.0;
  if (li < 6) bnd = A.b_xy[(size_t)(yax ? 6 + li : li) * L + inst];
  if (yax && li < 4) bps = A.b_psi[(size_t)li * L + inst];

  // Null-space QP steps (capi.cu reduced_qp): the boundary rows pin the first
  // and last XM0 (xy) / PM0 (psi) coefficients, c_f = T^-1 b, and the free
  // ones solve H_mm c_m = rhs_m - H_mf c_f:  c = cb + Z rhs, with the
  // per-instance boundary part cb = B b computed once here.
  constexpr int XM0 = 3, XM1 = NB - 3, PM0 = 2, PM1 = NB - 2;
  const int lrow = owner ? li : 0;
  const int hbase = lane & 16;  // first lane of this lane's axis
  const bool xfree = li >= XM0 && li < XM1;
  const bool pfree = !yax && li >= PM0 && li < PM1;
  const bool refine_xy = (C.refine & 1) != 0, refine_psi = (C.refine & 2) != 0;
  double cbx, cbp;
  {
    const double* br = sBx + lrow * 8;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      const double v = __shfl_sync(BMPC_FULL, bnd, hbase + r);
      if (r & 1) s1 = fma(br[r], v, s1); else s0 = fma(br[r], v, s0);
    }
    cbx = s0 + s1;
    const double* bq = sBp + lrow * 4;
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double v = __shfl_sync(BMPC_FULL, bps, 16 + r);
      if (r & 1) t1 = fma(bq[r], v, t1); else t0 = fma(bq[r], v, t0);
    }
    cbp = t0 + t1;
  }
  // c = c + Z (rhs - H c) over the free rows (one refinement step,
  // solver.py:164-168); `sh` is the lane's axis base for the shuffles
  auto qp_refine = [&](const double* Zr, const double* Hr, double rhs, double c, int sh, int m0,
                       int m1, bool free_row) {
    double h[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < NB; ++j) h[j & 3] = fma(Hr[j], __shfl_sync(BMPC_FULL, c, sh + j), h[j & 3]);
    const double r = rhs - ((h[0] + h[1]) + (h[2] + h[3]));
    double s[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j >= m0 && j < m1) s[j & 1] = fma(Zr[j], __shfl_sync(BMPC_FULL, r, sh + j), s[j & 1]);
    return free_row ? c + (s[0] + s[1]) : c;
  };
  // plain apply c = cb + Z rhs
  auto qp_apply = [&](const double* Zr, double rhs, double cb, int sh, int m0, int m1,
                      bool free_row) {
    double s[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j >= m0 && j < m1) s[j & 1] = fma(Zr[j], __shfl_sync(BMPC_FULL, rhs, sh + j), s[j & 1]);
    return free_row ? cb + (s[0] + s[1]) : cb;
  };

  // ---------------------------------------------------------------- init ----
  bool have_sol = false;  // [c; mu] of the previous sweep available for refinement
  if (A.init_mode == BMPC_INIT_RESUME) {
    const double* cr = A.carry + (size_t)inst * carry_doubles(NB);
    if (owner) {
      lam = cr[(yax ? 1 : 0) * NB + li];
      lamp = cr[2 * NB + li];
      G = cr[(yax ? 4 : 3) * NB + li];
    }
    // the previous sweep's coefficients: the refinement base
    if (owner) cown = cr[5 * NB + (yax ? RX : 0) + li];
    if (owner && !yax) cpown = cr[5 * NB + 2 * RX + li];
    have_sol = true;
  } else {
    // Initial targets g = assemble_g(alpha, d, alpha_a, d_a, v, psi) contracted
    // to G = F_axis^T g (solver.py:431, :281-286; kernels/_speedups.pyx:81-111).
    double ax[16], ay[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { ax[i] = 0.0; ay[i] = 0.0; }
    // warm starts may cover only some instances (the planner's eligible
    // columns, planner.py:362-410); the rest start cold
    const bool cold = A.init_mode == BMPC_INIT_COLD || (A.w_mask && !A.w_mask[inst]);
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
          // obstacle_update (_speedups.pyx:12-39) on the straight line, in the
          // exact form of the sweep's obstacle block: outside terms give
          // g_j = x, inside ones q + (a cos, b sin)
          const double abd2 = (a * b) * (a * b);
          double cin = 0.0, sq0 = 0.0;
#pragma unroll 4
          for (int j = 0; j < m; ++j) {
            const double2 q = __ldg(xi + j * n + k);
            if (obstacle_inside(xl, yl, q, a, b, abd2))
              obstacle_inside_term(xl, yl, q, a, b, gsx, gsy, sq0, cin);
          }
          gsx = fma((double)m - cin, xl, gsx);
          gsy = fma((double)m - cin, yl, gsy);
          gnx = speed0;  // v cos(psi) with psi = P c_psi = 0, alpha_a = d_a = 0
        } else {
          double ps = 0.0;
#pragma unroll
          for (int i = 0; i < NB; ++i) ps = fma(sP[bi(i, k)], A.w_cpsi[(size_t)i * L + inst], ps);
          for (int j = 0; j < m; ++j) {
            const double2 q = __ldg(xi + j * n + k);
            const size_t row = (size_t)(j * n + k) * L + inst;
            const double al = A.w_alpha[row], d = A.w_d[row];
            double sa, ca;
            sincos_nb(al, &sa, &ca);  // alpha in [-pi, pi]; full range only if needed
            if (!(fabs(al) < 1.0e5)) sincos(al, &sa, &ca);
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
          const double p = sP[bi(i, k)], pd = sPd[bi(i, k)], pdd = sPdd[bi(i, k)];
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
  BMPC_PROF(0);

  // ----------------------------------------------------------- AM sweeps ----
  // Early exit (tol > 0, first launch of a solve): the team leader's lane 0
  // reads the word of the earliest sweep it has not yet seen decided at the
  // top of each sweep and evaluates it near the end (the L2 round trip hides
  // under the sweep): flag set -> that sweep is not converged, look at the
  // next one; flag clear with all L instances counted -> that sweep is
  // globally converged, so every later sweep is wasted work (the host-side
  // re-run redoes exactly that many sweeps, solver.py:437-439).
  // The word travels by an asynchronous 16-byte copy (cp.async.cg: L2, no L1
  // staleness) into a shared slot, so no register is held across the sweep.
  // Nothing of it stays in registers across the sweep (the kernel sits at the
  // register cap): the flag is re-read from the launch parameters, the sweep
  // index to look at lives in a shared slot next to the word.  Only the team
  // instantiation carries it (the host routes polling solves there, with one
  // warp per instance when no team is asked for): compiled into the
  // throughput kernels even unused it costs them ~1.5%.
  __shared__ __align__(16) unsigned long long s_poll[BMPC_MAX_WARPS][2];
  __shared__ int s_poll_next[BMPC_MAX_WARPS];
#define BMPC_POLL (TEAMS && (A.flags & BMPC_F_POLL) != 0)  // the host sets it only with notconv
  if (BMPC_POLL && lane == 0) s_poll_next[warp] = 0;
  if constexpr (SKIP) {
    for (int k = lane; k < npad; k += 32) {  // nothing recorded yet
      sk_m0[k] = -1.f;
      sk_p0[k] = make_float2(0.f, 0.f);
    }
    __syncwarp();
  }
  if constexpr (SKIPG) {
    if (sk_m0) {
      for (int k = lane; k < npad; k += 32) {
        sk_m0[k] = -1.f;
        sk_p0[k] = make_float2(0.f, 0.f);
      }
    }
    __syncwarp();
  }
  for (int t = 0; t < iters; ++t) {
    const bool last = t == iters - 1;
    unsigned skipmask = 0;   // slots whose obstacle pass is provably all outside (warp-uniform)
    unsigned clearbits = 0;  // this lane's samples that passed the clearance test, per slot
    if (BMPC_POLL && wt == 0 && lane == 0 && t > 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&s_poll[warp][0]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;"
                   ::"r"(sa), "l"(A.notconv + (s_poll_next[warp] & ~1)) : "memory");
    }
    // (1) xy QP (solver.py:302-312) in null-space form: c = cb + Z (rho G +
    //     lambda), lane i / 16+i coefficient i of x / y.  Ill-conditioned
    //     shapes add one refinement step; it starts from the previous sweep's
    //     c once there is one (the same accuracy, one matrix pass less).
#ifndef BMPC_LOCKSTEP_EVERY
#define BMPC_LOCKSTEP_EVERY 1  // meet every k-th sweep
#endif
    if (BMPC_LOCKSTEP_EVERY == 1 || t % BMPC_LOCKSTEP_EVERY == 0) lockstep(1);
    {
      const double rhs = rho * G + lam;  // owner lanes (G = lam = 0 elsewhere)
      const double* zr = sZx + lrow * C.kms;
      double c = (refine_xy && have_sol) ? cown : qp_apply(zr, rhs, cbx, hbase, XM0, XM1, xfree);
      if (refine_xy) c = qp_refine(zr, sHx + lrow * C.kms, rhs, c, hbase, XM0, XM1, xfree);
      cown = c;
      if (owner) ws.cxy[2 * li + (yax ? 1 : 0)] = c;
      if (F32 && owner) fcxy[2 * li + (yax ? 1 : 0)] = (float)c;
      __syncwarp();
    }
    BMPC_PROF(1);
    const double2* __restrict__ cxy = reinterpret_cast<const double2*>(ws.cxy);

    // (2) pass A over every sample (lane + 32 r), CH slots at a time: x, y,
    //     xdot, ydot, xddot, yddot from c; theta = atan2(ydot, xdot) with the
    //     unwrap test against the previous sample done in registers; P^T theta.
    //     Acceleration block (_speedups.pyx:179-198) in exact form: unclipped
    //     samples give g_acc = (xddot, yddot) and r = 0, so Pddot^T g_acc =
    //     (Pddot^T Pddot) c plus a sparse correction from the clipped samples.
    double pth;                // owner lanes: P^T theta
    R Gx[NB], Gy[NB], pt[NB];  // Gx, Gy: lane partials of F_axis^T g beyond the Gram terms
#pragma unroll
    for (int i = 0; i < NB; ++i) Gx[i] = Gy[i] = pt[i] = 0;
    R sqo = 0, sqa = 0, sqn = 0;
    {
      bool wrap = false;
      R prev_last = 0;  // theta of sample 32 r - 1: lane 31 of the previous slot
      const double amax2 = A.a_max * A.a_max;
      // this warp's slots r = wt, wt + TW, ... in chunks of CH (every slot of a
      // chunk valid at compile time); chunks stay rolled for the instruction cache
      auto chunk_a = [&](auto nsc, const int r0) {
        constexpr int NSC = decltype(nsc)::value;
        int k[NSC];
        bool v[NSC];
        double xx[NSC], yy[NSC], xd[NSC], yd[NSC], xdd[NSC], ydd[NSC];
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          if constexpr (kOddDup) {  // a slot past the last one repeats it, masked
            const int r = min(r0 + s * TW, NKM - 1);
            k[s] = lane + 32 * r;
            v[s] = k[s] < n && r0 + s * TW < NKM;
          } else {
            k[s] = lane + 32 * (r0 + s * TW);
            v[s] = k[s] < n;
          }
          xx[s] = yy[s] = xd[s] = yd[s] = xdd[s] = ydd[s] = 0.0;
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double2 c = cxy[i];
          double p[NSC], pd[NSC], pdd[NSC];
          basis3<NSC, PAIRED, npad>(sP, sPd, sPdd, i, k, p, pd, pdd);
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            xx[s] = fma(p[s], c.x, xx[s]);
            yy[s] = fma(p[s], c.y, yy[s]);
            xd[s] = fma(pd[s], c.x, xd[s]);
            yd[s] = fma(pd[s], c.y, yd[s]);
            xdd[s] = fma(pdd[s], c.x, xdd[s]);
            ydd[s] = fma(pdd[s], c.y, ydd[s]);
          }
        }
        if constexpr (SKIP && !BMPC_SKIP_LATE) {
          // clearance test: moved less than the recorded clearance since the
          // slot's last obstacle pass (fp32; the slack covers every rounding)
          const float bf = (float)b, af = (float)a;
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            // padding samples hold P0 = 0, clearance -1 and never pass; their
            // lanes are masked after the vote (one vote for all slots, below)
            const float2 p0 = sk_p0[k[s]];
            const float dx = fmaf(bf, __double2float_rn(xx[s]), -p0.x);
            const float dy = fmaf(af, __double2float_rn(yy[s]), -p0.y);
            if (fmaf(dx, dx, dy * dy) < sk_m0[k[s]] || !v[s]) clearbits |= 1u << (r0 + s);
          }
        }
        double th[NSC];
        bool clip[NSC], anyclip = false;
        // headings within +-22.5 deg on every valid sample (the common case):
        // the octant-0 atan2, bit-identical to the full one there
        bool o0 = true;
#pragma unroll
        for (int s = 0; s < NSC; ++s) o0 &= !v[s] || atan2_is_o0(yd[s], xd[s]);
        if (__all_sync(BMPC_FULL, o0)) {
#pragma unroll
          for (int s = 0; s < NSC; ++s) th[s] = atan2_o0(yd[s], xd[s]);
        } else {
#pragma unroll
          for (int s = 0; s < NSC; ++s) th[s] = atan2_nb(yd[s], xd[s]);
        }
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          clip[s] = false;
          double prev = __shfl_up_sync(BMPC_FULL, th[s], 1);
          const double last = __shfl_sync(BMPC_FULL, th[s], 31);
          if (lane == 0) prev = prev_last;
          prev_last = last;
          // lane 0's predecessor belongs to another warp of a team: checked
          // after the team barrier
          if (v[s] && k[s] > 0 && (lane > 0 || TW == 1) && !(fabs(th[s] - prev) < CUDART_PI))
            wrap = true;
          if (v[s]) {
            ws.th[k[s]] = th[s];
            ws.xd[k[s]] = xd[s];
            ws.yd[k[s]] = yd[s];
            if constexpr (kStoreXY) {
              ws.x[k[s]] = xx[s];
              ws.y[k[s]] = yy[s];
            }
          } else {
            th[s] = 0.0;
          }
          // |acc| > a_max (NaN tests unclipped: g = acc propagates it)
          clip[s] = v[s] && fma(xdd[s], xdd[s], ydd[s] * ydd[s]) > amax2;
          anyclip |= clip[s];
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          double p[NSC];
          basis1<NSC, PAIRED, npad>(sP, i, k, p);
#pragma unroll
          for (int s = 0; s < NSC; ++s) pt[i] = fma(p[s], th[s], pt[i]);
        }
        if (__any_sync(BMPC_FULL, anyclip)) {  // clipped samples: g = a_max (cos, sin)
          double ex[NSC], ey[NSC];  // g_acc - acc
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            ex[s] = ey[s] = 0.0;
            const double m2 = fma(xdd[s], xdd[s], ydd[s] * ydd[s]);
            const double mi = rsqrt_nb(m2);
            const double dx = A.a_max * (xdd[s] * mi) - xdd[s], dy = A.a_max * (ydd[s] * mi) - ydd[s];
            ex[s] = clip[s] ? dx : 0.0;
            ey[s] = clip[s] ? dy : 0.0;
            sqa = fma(ex[s], ex[s], fma(ey[s], ey[s], sqa));
          }
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            double pdd[NSC];
            basis1<NSC, PAIRED, npad>(sPdd, i, k, pdd);
#pragma unroll
            for (int s = 0; s < NSC; ++s) {
              Gx[i] = fma(pdd[s], ex[s], Gx[i]);
              Gy[i] = fma(pdd[s], ey[s], Gy[i]);
            }
          }
        }
      };
      // fp32 mode pass A: the same chunk in single precision (no teams); the
      // samples for pass B and the obstacle block are stored in fp32, the
      // positions already in the ellipse frame
      const float amax2f = (float)(A.a_max * A.a_max), amaxf = (float)A.a_max;
      const float af = (float)a, bf = (float)b;
      auto chunk_a32 = [&](auto nsc, const int r0) {
        constexpr int NSC = decltype(nsc)::value;
        int k[NSC];
        bool v[NSC];
        float xx[NSC], yy[NSC], xd[NSC], yd[NSC], xdd[NSC], ydd[NSC];
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          k[s] = lane + 32 * (r0 + s);
          v[s] = k[s] < n;
          xx[s] = yy[s] = xd[s] = yd[s] = xdd[s] = ydd[s] = 0.f;
        }
        const float2* __restrict__ cf = reinterpret_cast<const float2*>(fcxy);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const float2 c = cf[i];
          float p[NSC], pd[NSC], pdd[NSC];
          basis3<NSC, PAIRED, npad>(fP, fPd, fPdd, i, k, p, pd, pdd);
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            xx[s] = fmaf(p[s], c.x, xx[s]);
            yy[s] = fmaf(p[s], c.y, yy[s]);
            xd[s] = fmaf(pd[s], c.x, xd[s]);
            yd[s] = fmaf(pd[s], c.y, yd[s]);
            xdd[s] = fmaf(pdd[s], c.x, xdd[s]);
            ydd[s] = fmaf(pdd[s], c.y, ydd[s]);
          }
        }
        if constexpr (SKIP) {  // clearance test on the fp32 frame positions (see chunk_a)
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            const float2 p0 = sk_p0[k[s]];
            const float dx = fmaf(xx[s], bf, -p0.x), dy = fmaf(yy[s], af, -p0.y);
            if (fmaf(dx, dx, dy * dy) < sk_m0[k[s]] || !v[s]) clearbits |= 1u << (r0 + s);
          }
        }
        float th[NSC];
        bool clip[NSC], anyclip = false;
#pragma unroll
        for (int s = 0; s < NSC; ++s) th[s] = atan2_f32_nb(yd[s], xd[s]);
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          float prev = __shfl_up_sync(BMPC_FULL, th[s], 1);
          const float lst = __shfl_sync(BMPC_FULL, th[s], 31);
          if (lane == 0) prev = prev_last;
          prev_last = lst;
          if (v[s] && k[s] > 0 && !(fabsf(th[s] - prev) < 3.14159265f)) wrap = true;
          if (v[s]) {
            fth[k[s]] = th[s];
            fxd[k[s]] = xd[s];
            fyd[k[s]] = yd[s];
            fxs[k[s]] = xx[s] * bf;
            fys[k[s]] = yy[s] * af;
          } else {
            th[s] = 0.f;
          }
          clip[s] = v[s] && fmaf(xdd[s], xdd[s], ydd[s] * ydd[s]) > amax2f;
          anyclip |= clip[s];
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          float p[NSC];
          basis1<NSC, PAIRED, npad>(fP, i, k, p);
#pragma unroll
          for (int s = 0; s < NSC; ++s) pt[i] = fmaf(p[s], th[s], pt[i]);
        }
        if (__any_sync(BMPC_FULL, anyclip)) {  // clipped samples: g = a_max (cos, sin)
          float ex[NSC], ey[NSC];
#pragma unroll
          for (int s = 0; s < NSC; ++s) {
            const float m2 = fmaf(xdd[s], xdd[s], ydd[s] * ydd[s]);
            const float mi = rsqrtf(m2);
            ex[s] = clip[s] ? amaxf * (xdd[s] * mi) - xdd[s] : 0.f;
            ey[s] = clip[s] ? amaxf * (ydd[s] * mi) - ydd[s] : 0.f;
            sqa = fmaf(ex[s], ex[s], fmaf(ey[s], ey[s], sqa));
          }
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            float pdd[NSC];
            basis1<NSC, PAIRED, npad>(fPdd, i, k, pdd);
#pragma unroll
            for (int s = 0; s < NSC; ++s) {
              Gx[i] = fmaf(pdd[s], ex[s], Gx[i]);
              Gy[i] = fmaf(pdd[s], ey[s], Gy[i]);
            }
          }
        }
      };
      int r0 = wt;
      if constexpr (F32) {
#pragma unroll kChunkUnrollA
        for (; r0 + (CH - 1) < NKM; r0 += CH) chunk_a32(std::integral_constant<int, CH>{}, r0);
#pragma unroll 1
        for (; CH > 1 && r0 < NKM; r0 += 1) chunk_a32(std::integral_constant<int, 1>{}, r0);
      } else {
        if constexpr (kOddDup) {
#pragma unroll 1
          for (; r0 < NKM; r0 += CH * TW) chunk_a(std::integral_constant<int, CH>{}, r0);
        } else {
#pragma unroll kChunkUnrollA
        for (; r0 + (CH - 1) * TW < NKM; r0 += CH * TW) chunk_a(std::integral_constant<int, CH>{}, r0);
#pragma unroll 1
        for (; CH > 1 && r0 < NKM; r0 += TW) chunk_a(std::integral_constant<int, 1>{}, r0);  // remainder
        }
      }
      if constexpr (SKIP && BMPC_SKIP_LATE) {
        // clearance test after the chunks, on the stored samples (keeps the
        // chunks' register footprint)
        const float bf = (float)b, af = (float)a;
#pragma unroll
        for (int r = 0; r < NKM; ++r) {
          const int k = lane + 32 * r;
          const float2 p0 = sk_p0[k];
          const float dx = fmaf(bf, __double2float_rn(ws.x[k]), -p0.x);
          const float dy = fmaf(af, __double2float_rn(ws.y[k]), -p0.y);
          if (fmaf(dx, dx, dy * dy) < sk_m0[k] || k >= n) clearbits |= 1u << r;
        }
      }
      if constexpr (SKIP) {
        skipmask = __reduce_and_sync(BMPC_FULL, clearbits);
#ifdef BMPC_PHASE_PROF
        {
          // slots tested / skipped; failed slots holding a sample that never
          // skips (inside or touching an obstacle); failing samples
          unsigned never = 0;
          int nfail = 0;
          for (int r = 0; r < nslots; ++r) {
            const int k = lane + 32 * r;
            if (k < n && sk_m0[k] < 0.f) never |= 1u << r;
            if (k < n && !((clearbits >> r) & 1u)) ++nfail;
          }
          never = __reduce_or_sync(BMPC_FULL, never);
          nfail = __reduce_add_sync(BMPC_FULL, nfail);
          if (lane == 0) {
            s_prof[warp][14] += nslots;
            s_prof[warp][15] += __popc(skipmask & ((1u << nslots) - 1u));
            s_prof[warp][16] += __popc(never & ~skipmask & ((1u << nslots) - 1u));
            s_prof[warp][17] += nfail;
          }
        }
#endif
      }
      BMPC_PROF(2);
      // P^T theta of this warp's slots (again after an unwrap)
      auto pt_slots = [&]() {
#pragma unroll
        for (int i = 0; i < NB; ++i) pt[i] = 0;
#pragma unroll 1
        for (int r = wt; r < NKM; r += TW) {
          const int k = lane + 32 * r;
          if (k < n) {
            if constexpr (F32) {
              const float t = fth[k];
#pragma unroll
              for (int i = 0; i < NB; ++i) pt[i] = fmaf(fP[bi(i, k)], t, pt[i]);
            } else {
              const double t = ws.th[k];
#pragma unroll
              for (int i = 0; i < NB; ++i) pt[i] = fma(sP[bi(i, k)], t, pt[i]);
            }
          }
        }
      };
      auto pt_colsum = [&]() {
#pragma unroll
        for (int i = 0; i < NB; ++i) ws.red[lane * kRedStride + i] = pt[i];
        __syncwarp();
        const double c = owner ? column_sum(ws.red, li) : 0.0;  // lanes i and 16+i: sum_k P_ki theta_k
        __syncwarp();
        return c;
      };
      if (TW == 1) {
        if (__any_sync(BMPC_FULL, wrap)) {  // rare: exact numpy unwrap, then P^T theta again
          __syncwarp();
          if (lane == 0) {
            if constexpr (F32) np_unwrap_serial_f(fth, n);
            else np_unwrap_serial(ws.th, n);
          }
          __syncwarp();
          pt_slots();
        }
        pth = pt_colsum();
      } else {
        // team: partial sums and unwrap flags through the exchange slots; the
        // slot-boundary tests (sample 32 r against 32 r - 1) by every warp
        const double part = pt_colsum();
        if (owner) xch[li] = part;
        const bool wf = __any_sync(BMPC_FULL, wrap);
        if (lane == 0) xch[67] = wf ? 1.0 : 0.0;
        team_sync();
        bool gw = false;
        for (int w = 0; w < TW; ++w) gw |= xch_of(w)[67] != 0.0;
        for (int r = 1 + lane; r < NKM; r += 32) {
          const int k = 32 * r;
          if (k < n && !(fabs(ws.th[k] - ws.th[k - 1]) < CUDART_PI)) gw = true;
        }
        if (__any_sync(BMPC_FULL, gw)) {  // rare: serial numpy unwrap by one warp
          team_sync();
          if (wt == 0 && lane == 0) np_unwrap_serial(ws.th, n);
          team_sync();
          pt_slots();
          const double p2 = pt_colsum();
          if (owner) xch[li] = p2;
          team_sync();
        }
        double acc = 0.0;
        for (int w = 0; w < TW; ++w) acc += owner ? xch_of(w)[li] : 0.0;
        pth = acc;
      }
    }
    BMPC_PROF(3);
    lockstep(2);

    // (3) obstacle block (exact form, independent of psi), samples dealt as in
    //     slot(): full slots two at a time, the n % 32 leftover samples split
    //     over lane groups.
    if constexpr (F32) {
      const double abd = a * b;
      TailArgs32 T{fP, fxs, fys, xf, xis, n, m, (float)a, (float)b, (float)inv_a, (float)inv_b,
                   (float)(abd * abd), a, b, inv_a, inv_b, abd * abd,
                   CULL ? reinterpret_cast<const float4*>(A.boxes) + (size_t)(inst / A.l) * ((n + 31) >> 5) * m
                        : nullptr,
                   __double2float_ru(abd * abd * (1.0 + 1e-4)), sk_p0, sk_m0, __double2float_ru(abd)};
      if constexpr (SKIP) {
        // only the slots that failed the clearance test, one at a time
        const unsigned todo = ~skipmask & ((1u << nslots) - 1u);
        unsigned full = todo & ((1u << sl.F) - 1u);
#pragma unroll 1
        while (full) {
          const int r = __ffs(full) - 1;
          full &= full - 1u;
          const int ks[1] = {lane + 32 * r};
          obstacle_block_f32<1, NB, npad, BMPC_USINGLE, false, CULL, true>(T, ks, 0, 1, 1, true, true, Gx, Gy, sqo);
        }
        if (todo >> sl.F) {
          const Slot S = slot(sl.F, lane, sl);
          const int ks[1] = {S.k};
          obstacle_block_f32<1, NB, npad, (NKM >= 7 ? BMPC_USPLIT_MANY : BMPC_USPLIT), false, false, true>(
              T, ks, S.j0, S.js, sl.g, S.valid, S.leader, Gx, Gy, sqo);
        }
        __syncwarp();
      } else {
      int r = 0;
      if (kPairSlots<NB>) {
#pragma unroll 1
        for (; r + 1 < sl.F; r += 2) {
          const int ks[2] = {lane + 32 * r, lane + 32 * (r + 1)};
          obstacle_block_f32<2, NB, npad, BMPC_UPAIR, PAIRED, CULL>(T, ks, 0, 1, 0, true, true, Gx, Gy, sqo);
        }
      }
#pragma unroll 1
      for (; r < nslots; ++r) {
        const Slot S = slot(r, lane, sl);
        const int ks[1] = {S.k};
        if (r < sl.F)
          obstacle_block_f32<1, NB, npad, BMPC_USINGLE, false, CULL>(T, ks, S.j0, S.js, 1, S.valid, S.leader,
                                                                      Gx, Gy, sqo);
        else
          obstacle_block_f32<1, NB, npad, (NKM >= 7 ? BMPC_USPLIT_MANY : BMPC_USPLIT), false, false>(
              T, ks, S.j0, S.js, sl.g, S.valid, S.leader, Gx, Gy, sqo);
      }
      }
    } else {
      TailArgs T{sP, cxy, xis, xf, kStoreXY ? ws.x : nullptr, kStoreXY ? ws.y : nullptr, n, m, a, b,
                 inv_a, inv_b, __double2float_ru((a * b) * (a * b) * 1.02),
                 __double2float_rd(prefilter_lim(a, b)),
                 CULL ? reinterpret_cast<const float4*>(A.boxes) + (size_t)(inst / A.l) * ((n + 31) >> 5) * m
                      : nullptr,
                 __double2float_ru((a * b) * (a * b) * (1.0 + 1e-4)), sk_p0, sk_m0, __double2float_ru(a * b)};
      if constexpr (SKIP) {
        // only the slots that failed the clearance test (pass A): full slots in
        // pairs as they come, a leftover one alone; each pass records the
        // slot's new clearances
        const unsigned todo = ~skipmask & ((1u << nslots) - 1u);
        unsigned full = todo & ((1u << sl.F) - 1u);
#ifndef BMPC_SKIP_NOPAIR
#define BMPC_SKIP_NOPAIR 1  // no two-slot passes: most slots are skipped, and the sweep code stays small
#endif
        if (kPairSlots<NB> && !BMPC_SKIP_NOPAIR) {
#pragma unroll 1
          while (full & (full - 1u)) {  // at least two
            const int ra = __ffs(full) - 1;
            full &= full - 1u;
            const int rb = __ffs(full) - 1;
            full &= full - 1u;
            const int ks[2] = {lane + 32 * ra, lane + 32 * rb};
            obstacle_block<2, NB, npad, F32, BMPC_UPAIR, XS, false, CULL, true>(T, ks, 0, 1, 0, true, true, Gx, Gy,
                                                                                  sqo);
          }
        }
#pragma unroll 1
        while (full) {
          const int r = __ffs(full) - 1;
          full &= full - 1u;
          const int ks[1] = {lane + 32 * r};
          obstacle_block<1, NB, npad, F32, BMPC_USINGLE, XS, false, CULL, true>(T, ks, 0, 1, 1, true, true, Gx, Gy,
                                                                                  sqo);
        }
        if (todo >> sl.F) {  // the leftover samples, obstacles split over lane groups (js = g)
          const Slot S = slot(sl.F, lane, sl);
          const int ks[1] = {S.k};
          obstacle_block<1, NB, npad, F32, (NKM >= 7 ? BMPC_USPLIT_MANY : BMPC_USPLIT), XS, false, false, true>(
              T, ks, S.j0, S.js, sl.g, S.valid, S.leader, Gx, Gy, sqo);
        }
        __syncwarp();  // the recorded clearances are read by other lanes in the next sweep's pass A
      } else if constexpr (SKIPG) {
        // every whole slot takes its pass; the pass tests the slot's recorded
        // clearances itself and returns early when they all hold
#ifndef BMPC_SKIPG_LEFTOVER_CULL
// 1: the leftover samples through the culling path too (tracked, unsplit): c4
// 208.2 vs 212.1 ms per 128 scenes, but the unsplit pass sums a sample's
// inside terms in another order (coefficients move by 1e-7 absolute): off
#define BMPC_SKIPG_LEFTOVER_CULL 0
#endif
#pragma unroll 1
        for (int r = 0; r < (BMPC_SKIPG_LEFTOVER_CULL ? nslots : sl.F); ++r) {
          const int ks[1] = {lane + 32 * r};
          obstacle_block<1, NB, npad, F32, BMPC_USINGLE, XS, false, CULL, SKIPG, SKIPG>(
              T, ks, 0, 1, 1, BMPC_SKIPG_LEFTOVER_CULL ? ks[0] < n : true, true, Gx, Gy, sqo);
        }
        if (!BMPC_SKIPG_LEFTOVER_CULL && sl.R > 0) {  // the leftover samples: split over lane groups, untracked, every sweep
          const Slot S = slot(sl.F, lane, sl);
          const int ks[1] = {S.k};
          obstacle_block<1, NB, npad, F32, (NKM >= 7 ? BMPC_USPLIT_MANY : BMPC_USPLIT), XS, false, false>(
              T, ks, S.j0, S.js, sl.g, S.valid, S.leader, Gx, Gy, sqo);
        }
      } else {
      int r = wt;  // this warp's slots r = wt, wt + TW, ...
      if (kPairSlots<NB>) {
#pragma unroll 1
        for (; r + TW < sl.F; r += 2 * TW) {
          const int ks[2] = {lane + 32 * r, lane + 32 * (r + TW)};
          obstacle_block<2, NB, npad, F32, BMPC_UPAIR, XS, PAIRED, CULL>(T, ks, 0, 1, 0, true, true, Gx, Gy, sqo);
        }
      }
#pragma unroll 1
      for (; r < nslots; r += TW) {
        const Slot S = slot(r, lane, sl);
        const int ks[1] = {S.k};
        if (r < sl.F)  // a full slot on its own
          obstacle_block<1, NB, npad, F32, BMPC_USINGLE, XS, false, CULL>(T, ks, S.j0, S.js, 1, S.valid, S.leader,
                                                             Gx, Gy, sqo);
        else  // the leftover samples, obstacles split over lane groups (js = g)
          obstacle_block<1, NB, npad, F32, (NKM >= 7 ? BMPC_USPLIT_MANY : BMPC_USPLIT), XS, false, false>(
              T, ks, S.j0, S.js, sl.g, S.valid, S.leader, Gx, Gy, sqo);
      }
      }
    }
    BMPC_PROF(5);
#ifndef BMPC_LS_AFTER_OBST
#define BMPC_LS_AFTER_OBST 0  // 1: fp64 long horizons also meet after the obstacle block
#endif
    lockstep(BMPC_LS_AFTER_OBST && !F32 ? 1 : 2);

    // (4) psi QP (solver.py:322-328), null-space form on lanes 0..NB-1
    {
      const double rhs = rho * pth + lamp;  // x owner lanes
      const double* zr = sZp + lrow * C.kms;
      double c = (refine_psi && have_sol) ? cpown : qp_apply(zr, rhs, cbp, 0, PM0, PM1, pfree);
      if (refine_psi) c = qp_refine(zr, sHp + lrow * C.kms, rhs, c, 0, PM0, PM1, pfree);
      cpown = c;
      if (!yax && owner) ws.cp[li] = c;
      if (F32 && !yax && owner) fcp[li] = (float)c;
      __syncwarp();
    }
    BMPC_PROF(4);

    // (5) pass B: psi = P c_psi and the non-holonomic block (_speedups.pyx:200-216),
    //     contracted onto Pdot.
    // full chunks of CH slots (every slot valid at compile time), then the
    // NKM % CH remainder; chunks stay rolled for the instruction cache
    R cps_reg[NB];  // c_psi, held in registers for every chunk
#pragma unroll
    for (int i = 0; i < NB; ++i) cps_reg[i] = F32 ? (R)fcp[i] : (R)ws.cp[i];
    auto chunk_b = [&](auto nsc, const int r0) {
      constexpr int NSC = decltype(nsc)::value;
      int k[NSC];
      bool v[NSC];
      double ps[NSC];
#pragma unroll
      for (int s = 0; s < NSC; ++s) {
        if constexpr (kOddDup) {
          const int r = min(r0 + s * TW, NKM - 1);
          k[s] = lane + 32 * r;
          v[s] = k[s] < n && r0 + s * TW < NKM;
        } else {
          k[s] = lane + 32 * (r0 + s * TW);
          v[s] = k[s] < n;
        }
        ps[s] = 0.0;
      }
      // two partial sums per slot: half the dependent chain
      double ps1[NSC];
#pragma unroll
      for (int s = 0; s < NSC; ++s) ps1[s] = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        double p[NSC];
        basis1<NSC, PAIRED, npad>(sP, i, k, p);
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          if (i & 1) ps1[s] = fma(p[s], cps_reg[i], ps1[s]);
          else ps[s] = fma(p[s], cps_reg[i], ps[s]);
        }
      }
#pragma unroll
      for (int s = 0; s < NSC; ++s) ps[s] += ps1[s];
      // branch-free sin/cos for every slot first, so the slots interleave; the
      // full-range fallback (huge / non-finite headings) is one rare branch
      double sps[NSC], cps[NSC];
      bool q0 = true;
#pragma unroll
      for (int s = 0; s < NSC; ++s) q0 &= fabs(ps[s]) <= 0.78;
      if (__all_sync(BMPC_FULL, q0)) {  // headings within +-45 deg (the common case)
#pragma unroll
        for (int s = 0; s < NSC; ++s) sincos_q0(ps[s], &sps[s], &cps[s]);
      } else {
        bool big = false;
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          sps[s] = 0.0;
          cps[s] = 1.0;
          sincos_nb(ps[s], &sps[s], &cps[s]);
          big |= !(fabs(ps[s]) < 1.0e5);
        }
        if (big) {
#pragma unroll
          for (int s = 0; s < NSC; ++s)
            if (!(fabs(ps[s]) < 1.0e5)) sincos(ps[s], &sps[s], &cps[s]);
        }
      }
      double gnx[NSC], gny[NSC], vv[NSC];
#pragma unroll
      for (int s = 0; s < NSC; ++s) {
        gnx[s] = gny[s] = vv[s] = 0.0;
        const double xd = v[s] ? ws.xd[k[s]] : 0.0, yd = v[s] ? ws.yd[k[s]] : 0.0;
        const double s2 = fma(xd, xd, yd * yd);
        double u = s2 * rsqrt_nb(s2);
        u = u < A.v_min ? A.v_min : (u > A.v_max ? A.v_max : u);
        vv[s] = u;
        gnx[s] = v[s] ? u * cps[s] : 0.0;
        gny[s] = v[s] ? u * sps[s] : 0.0;
        const double rnx = xd - gnx[s], rny = yd - gny[s];
        const double q = fma(rnx, rnx, fma(rny, rny, (double)sqn));
        sqn = v[s] ? (R)q : sqn;
      }
      if (last && (A.flags & BMPC_F_V)) {
#pragma unroll
        for (int s = 0; s < NSC; ++s)
          if (v[s]) A.v_out[(size_t)k[s] * L + inst] = vv[s];
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        double pd[NSC];
        basis1<NSC, PAIRED, npad>(sPd, i, k, pd);
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          Gx[i] = fma(pd[s], gnx[s], Gx[i]);
          Gy[i] = fma(pd[s], gny[s], Gy[i]);
        }
      }
    };
    // fp32 mode pass B: psi, sin/cos, the clipped speed and the non-holonomic
    // residual in single precision; contracted as Pdot^T (g_nh - xdot), the
    // small part of Pdot^T g_nh (the Gram part Pdot^T Pdot c is added in fp64)
    auto chunk_b32 = [&](auto nsc, const int r0) {
      constexpr int NSC = decltype(nsc)::value;
      int k[NSC];
      bool v[NSC];
      float ps[NSC], ps1[NSC];
#pragma unroll
      for (int s = 0; s < NSC; ++s) {
        k[s] = lane + 32 * (r0 + s);
        v[s] = k[s] < n;
        ps[s] = ps1[s] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        float p[NSC];
        basis1<NSC, PAIRED, npad>(fP, i, k, p);
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          if (i & 1) ps1[s] = fmaf(p[s], cps_reg[i], ps1[s]);
          else ps[s] = fmaf(p[s], cps_reg[i], ps[s]);
        }
      }
      float sps[NSC], cps[NSC];
      bool big = false;
#pragma unroll
      for (int s = 0; s < NSC; ++s) {
        ps[s] += ps1[s];
        sincos_f32_nb(ps[s], &sps[s], &cps[s]);
        big |= !(fabsf(ps[s]) < 1.0e4f);
      }
      if (big) {
#pragma unroll
        for (int s = 0; s < NSC; ++s)
          if (!(fabsf(ps[s]) < 1.0e4f)) sincosf(ps[s], &sps[s], &cps[s]);
      }
      const float vminf = (float)A.v_min, vmaxf = (float)A.v_max;
      float rnx[NSC], rny[NSC];
#pragma unroll
      for (int s = 0; s < NSC; ++s) {
        const float xd = v[s] ? fxd[k[s]] : 0.f, yd = v[s] ? fyd[k[s]] : 0.f;
        float u = sqrt_f32_nb(fmaf(xd, xd, yd * yd));
        u = u < vminf ? vminf : (u > vmaxf ? vmaxf : u);
        rnx[s] = v[s] ? fmaf(u, cps[s], -xd) : 0.f;  // g_nh - xdot
        rny[s] = v[s] ? fmaf(u, sps[s], -yd) : 0.f;
        sqn = fmaf(rnx[s], rnx[s], fmaf(rny[s], rny[s], sqn));
        if (last && (A.flags & BMPC_F_V) && v[s]) A.v_out[(size_t)k[s] * L + inst] = (double)u;
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        float pd[NSC];
        basis1<NSC, PAIRED, npad>(fPd, i, k, pd);
#pragma unroll
        for (int s = 0; s < NSC; ++s) {
          Gx[i] = fmaf(pd[s], rnx[s], Gx[i]);
          Gy[i] = fmaf(pd[s], rny[s], Gy[i]);
        }
      }
    };
    {
      int r0 = wt;
      if constexpr (F32) {
#pragma unroll kChunkUnrollB
        for (; r0 + (CH - 1) < NKM; r0 += CH) chunk_b32(std::integral_constant<int, CH>{}, r0);
#pragma unroll 1
        for (; CH > 1 && r0 < NKM; r0 += 1) chunk_b32(std::integral_constant<int, 1>{}, r0);
      } else {
        if constexpr (kOddDup) {
#pragma unroll 1
          for (; r0 < NKM; r0 += CH * TW) chunk_b(std::integral_constant<int, CH>{}, r0);
        } else {
#pragma unroll kChunkUnrollB
        for (; r0 + (CH - 1) * TW < NKM; r0 += CH * TW) chunk_b(std::integral_constant<int, CH>{}, r0);
#pragma unroll 1
        for (; CH > 1 && r0 < NKM; r0 += TW) chunk_b(std::integral_constant<int, 1>{}, r0);
        }
      }
    }
    BMPC_PROF(12);
    lockstep(3);

    // (6) G = F_axis^T g = m (P^T P) c + (Pddot^T Pddot) c + the lane partials
    //     (Pdot^T g_nh and the exact-form corrections):
    //     the dense sample part through the shared-memory transpose (fixed
    //     summation order), residual sums by xor butterflies (identical on all
    //     lanes).  lambda step F_axis^T (F_axis c - g) = (F_axis^T F_axis) c - G
    //     = (Pdot^T Pdot) c - lane partials.
    // For n_b <= 13 the three squared-residual partials ride in the free
    // x-half columns n_b, n_b+1, n_b+2 of the same transpose (lanes n_b..n_b+2
    // end with the block totals); wider bases use xor butterflies (lanes 16..18).
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      ws.red[lane * kRedStride + i] = Gx[i];
      ws.red[lane * kRedStride + 16 + i] = Gy[i];
    }
    if constexpr (kSqCols) {
      ws.red[lane * kRedStride + NB] = sqo;
      ws.red[lane * kRedStride + NB + 1] = sqa;
      ws.red[lane * kRedStride + NB + 2] = sqn;
    }
    __syncwarp();
    double gn = (owner || is_sq_lane) ? column_sum(ws.red, lane) : 0.0;
    if constexpr (!kSqCols) {
      sqo = warp_sum(sqo);
      sqa = warp_sum(sqa);
      sqn = warp_sum(sqn);
    }
    __syncwarp();
    bool stop = false;
    if (BMPC_POLL) {
      int dec = 0;  // 1: sweep s_poll_next not converged, 2: converged -> exit
      if (wt == 0 && lane == 0) {
        if (t > 0) {
          asm volatile("cp.async.wait_all;" ::: "memory");
          const int nx = s_poll_next[warp];
          const unsigned long long w = s_poll[warp][nx & 1];
          if ((w >> 32) != 0ull) {
            dec = 1;
            s_poll_next[warp] = nx + 1;
          } else if ((unsigned)w == (unsigned)L) {
            dec = 2;
          }
        }
        if (TW > 1) xch[68] = dec == 2 ? 1.0 : 0.0;  // every sweep; read after the team barrier
      }
      stop = __shfl_sync(BMPC_FULL, dec, 0) == 2;
    }
    if (TW > 1) {  // team: sum the warps' partials in a fixed order
      if (owner) xch[32 + lane] = gn;
      if constexpr (kSqCols) {
        if (is_sq_lane) xch[64 + lane - NB] = gn;
      } else if (lane == 0) {
        xch[64] = sqo;
        xch[65] = sqa;
        xch[66] = sqn;
      }
      team_sync();
      if (BMPC_POLL) stop = xch_of(0)[68] != 0.0;  // the leader's decision, team-uniform
      gn = 0.0;
      sqo = sqa = sqn = 0.0;
      for (int w = 0; w < TW; ++w) {
        const double* xw = xch_of(w);
        gn += owner ? xw[32 + lane] : (kSqCols && is_sq_lane ? xw[64 + lane - NB] : 0.0);
        sqo += xw[64];
        sqa += xw[65];
        sqn += xw[66];
      }
    }
    BMPC_PROF(6);
    if (owner) {
      const double* m1 = sM + li * C.kms;   // m P^T P + Pddot^T Pddot
      const double* m3 = sMd + li * C.kms;  // Pdot^T Pdot
      double a1[2] = {0.0, 0.0}, a3[2] = {0.0, 0.0};
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double cj = ws.cxy[2 * j + (yax ? 1 : 0)];
        a1[j & 1] = fma(m1[j], cj, a1[j & 1]);
        a3[j & 1] = fma(m3[j], cj, a3[j & 1]);
      }
      const double rest = gn;
      if constexpr (F32) {
        // m1 = F_axis^T F_axis here, gn = F_axis^T (g - F c): G = F_axis^T g and
        // lambda -= rho F_axis^T (F c - g) from the residual contractions alone
        G = (a1[0] + a1[1]) + rest;
        lam += rho * rest;
      } else {
        G = (a1[0] + a1[1]) + rest;
        lam -= rho * ((a3[0] + a3[1]) - rest);
      }
    }
    // lambda_psi step P^T (psi - theta) = (P^T P) c_psi - P^T theta (solver.py:494),
    // evaluated here where its latency overlaps the residual bookkeeping
    if (!yax && owner) {
      const double* mr = sMp + li * C.kms;
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < NB; ++j) s4[j & 3] = fma(mr[j], ws.cp[j], s4[j & 3]);
      lamp -= rho * (((s4[0] + s4[1]) + (s4[2] + s4[3])) - pth);
    }
    const double sqv = kSqCols ? gn : (lane == 16 ? sqo : (lane == 17 ? sqa : sqn));  // sq lanes
    if (A.notconv && wt == 0) {  // global early stop: flag this sweep unless every residual <= tol
      // res = sqrt(sqv) <= tol; for tol = 0 (the fixed-sweep benchmarks) that is
      // exactly sqv <= 0 (sqrt is exact at +-0 and keeps NaN), so the square
      // root stays off the sweep's critical path
      const bool ok = A.tol > 0.0 ? sqrt(sqv) <= A.tol : (A.tol == 0.0 && sqv <= 0.0);
      const bool nc = __any_sync(BMPC_FULL, is_sq_lane && !ok);
      // a plain store into the high half: the flag only ever goes 0 -> 1, and a
      // read-before-write would stall the warp on a coherent L2 round trip every
      // sweep; polling solves count instead (a reduction, nothing waits on it)
      unsigned long long* w = A.notconv + A.hist_offset + t;
      if (lane == 0) {
        if (BMPC_POLL) atomicAdd(w, nc ? 0x100000001ull : 1ull);
        else if (nc) reinterpret_cast<int*>(w)[1] = 1;
      }
    }
    if (is_sq_lane && wt == 0 && ((A.flags & BMPC_F_HISTORY) || last)) {
      const double res = sqrt(sqv);
      const int blk = lane - sq_lane0;  // 0 obstacle, 1 acceleration, 2 non-holonomic
      if (A.flags & BMPC_F_HISTORY)
        A.hist[((size_t)(A.hist_offset + t) * 3 + blk) * L + inst] = res;
      if (last && A.res_final) A.res_final[(size_t)blk * L + inst] = res;
      if (last) ws.res[blk] = res;  // for the fused scoring below
    }
    have_sol = true;
    BMPC_PROF(7);
    if (stop) return;  // an earlier sweep converged everywhere: the re-run takes over
  }

  // The global clearance scratch slot of this warp is reused by the next block
  // scheduled on this SM, which starts by clearing it: make this warp's last
  // records land first (they are thousands of cycles old by the time the block
  // exits; the fence makes it certain).
  if constexpr (SKIPG) __threadfence();

  // ------------------------------------------------- fused planner scoring ----
  // sample_plan + filter_candidates + meta_cost of this instance straight from
  // the on-chip coefficients (planner.py:210-245, :412-423; csrc/score.cuh).
  if ((A.flags & BMPC_F_SCORE) && wt == 0) {
    const bmpc_fused_score& F = A.score;
    const ScoreParams sp{n, m, F.kind, a, b, F.v_cruise, F.v_max, F.y_rl, F.w1, F.w2,
                         F.heading_limit, F.residual_tol, F.ratio_min};
    const double2* __restrict__ cxy2 = reinterpret_cast<const double2*>(ws.cxy);
    // x, y, xdot, ydot of the final coefficients were stored by the last
    // sweep's pass A (the same sequential fma chains as k_score's sampling, so
    // the fused and stand-alone scores agree bit for bit); psi is sampled here
    auto sample = [&](int k, double& x, double& y, double& xd, double& yd, double& ps) {
      if constexpr (F32) {  // fp64 samples of the final coefficients (global basis)
        x = y = xd = yd = ps = 0.0;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double p = sP[bi(i, k)], pd = sPd[bi(i, k)];
          const double2 c = cxy2[i];
          x = __fma_rn(p, c.x, x);
          y = __fma_rn(p, c.y, y);
          xd = __fma_rn(pd, c.x, xd);
          yd = __fma_rn(pd, c.y, yd);
          ps = __fma_rn(p, ws.cp[i], ps);
        }
        return;
      }
      xd = ws.xd[k];
      yd = ws.yd[k];
      ps = 0.0;
      if constexpr (kStoreXY) {
        x = ws.x[k];
        y = ws.y[k];
#pragma unroll
        for (int i = 0; i < NB; ++i) ps = __fma_rn(sP[bi(i, k)], ws.cp[i], ps);
      } else {
        x = y = 0.0;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const double p = sP[bi(i, k)];
          const double2 c = cxy2[i];
          x = __fma_rn(p, c.x, x);
          y = __fma_rn(p, c.y, y);
          ps = __fma_rn(p, ws.cp[i], ps);
        }
      }
    };
    double cost, rmin, hmax;
    unsigned char f;
    score_instance(sp, xi, sample, ws.res[0], ws.res[1], ws.res[2], cost, rmin, hmax, f);
    if (lane == 0) {
      F.meta[inst] = cost;
      F.min_ratio[inst] = rmin;
      F.heading_max[inst] = hmax;
      F.flags[inst] = f;
    }
  }
  BMPC_PROF(8);

  // ------------------------------------------------------------- outputs ----
  if (wt != 0) return;  // the team's warp 0 holds the same state and writes it
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
      double* cr = A.carry + (size_t)inst * carry_doubles(NB);
      cr[(yax ? 1 : 0) * NB + li] = lam;
      if (!yax) cr[2 * NB + li] = lamp;
      cr[(yax ? 4 : 3) * NB + li] = G;
    }
  }
  if ((A.flags & BMPC_F_CARRY) && owner) {  // the refinement base of the next sweep
    double* cr = A.carry + (size_t)inst * carry_doubles(NB);
    cr[5 * NB + (yax ? RX : 0) + li] = cown;
    if (!yax) cr[5 * NB + 2 * RX + li] = cpown;
  }
  BMPC_PROF(9);
  BMPC_PROF_FLUSH
}

}  // namespace bmpc
