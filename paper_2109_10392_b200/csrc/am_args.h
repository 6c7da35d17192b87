// am_args.h -- argument blocks shared by the C-ABI and the sm_100a kernels.
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

// Device-side constants of one problem shape (uploaded once per context).
typedef struct {
  int n;          // horizon samples
  int npad;       // n rounded up to a multiple of 32
  int nb;         // Bernstein coefficients per axis (degree + 1)
  int kxs, kps;   // padded (odd) row strides of the (nb+6)^2 and (nb+4)^2 KKT blocks
  int kms;        // padded (odd) row stride of M
  double rho;
  const double* PT;   // [3][nb][npad]: P^T, Pdot^T, Pddot^T, zero padded past n
  const double* IMG;  // the persistent kernel's constant image (shared-memory layout):
                      // the basis in bmpc_basis_index order, then M, the QP blocks, tau
  const double* tau;  // [npad] (t_k - t0)/(tf - t0), cold-start line parameter
  const double* Kxf;  // [nb+6][kxs] inverse of the per-axis KKT matrix
  const double* Kxa;  // [nb+6][kxs] the per-axis KKT matrix (refinement residual)
  const double* Kpf;  // [nb+4][kps] inverse of the heading KKT matrix
  const double* Kpa;  // [nb+4][kps] the heading KKT matrix
  const double* M;    // [4][nb][kms] F_axis^T F_axis, P^T P, Pddot^T Pddot, Pdot^T Pdot,
                      // then the null-space QP blocks Z_xy, H_xy, Z_psi, H_psi [nb][kms],
                      // B_xy [nb][8], B_psi [nb][4] (capi.cu: reduced_qp)
  int const_doubles;  // size of the whole constant image starting at PT (even; the
                      // kernel's shared-memory layout, copied in one bulk transfer)
  const float* IMGF;  // fp32 copy of the image's basis part (same bmpc_basis_index
                      // order): the fp32 mode's shared-memory basis
  int refine;         // QP refinement step: bit 0 xy, bit 1 psi
} bmpc_dev_consts;

// Doubles of the constant image (shared-memory layout): basis, the four Gram
// blocks, the four null-space QP blocks, the two boundary maps and tau.
#ifdef __CUDACC__
__host__ __device__
#endif
static inline size_t bmpc_const_image_doubles(int nb, int npad) {
  return (size_t)3 * nb * npad + (size_t)8 * nb * (nb | 1) + (size_t)12 * nb + (size_t)npad;
}

// Basis order of the constant image.  When npad is a whole number of slot
// pairs (64, 128, 256), row `row` (q * nb + i for basis q in {P, Pdot, Pddot})
// at sample k sits at
//   (row * npad / 64 + k / 64) * 64 + 2 * (k % 32) + (k / 32) % 2,
// so samples k and k + 32 of an even slot pair are adjacent and one 16-byte
// shared load feeds both slots of a pass chunk; otherwise (npad = 224) rows
// are plain, row * npad + k.
#ifdef __CUDACC__
__host__ __device__
#endif
static inline int bmpc_basis_index(int row, int k, int npad) {
  return (npad & 63) ? row * npad + k
                     : (row * (npad >> 6) + (k >> 6)) * 64 + ((k & 31) << 1) + ((k >> 5) & 1);
}

enum { BMPC_INIT_COLD = 0, BMPC_INIT_WARM = 1, BMPC_INIT_RESUME = 2 };
enum {
  BMPC_F_HISTORY = 1,   // write residual history rows
  BMPC_F_V = 2,         // write the last tail's clipped speed v (n, L)
  BMPC_F_CARRY = 4,     // write the carried state (for chunked / resumed solves)
  BMPC_F_F32 = 8,       // mixed precision: fp32 sample passes and obstacle block, fp64
                        // QP steps, Gram terms, G and multipliers
  BMPC_F_SCORE = 16,    // fused planner scoring after the last sweep
  BMPC_F_POLL = 32,     // tol > 0: count finished instances per sweep and exit once an
                        // earlier sweep is known to be globally converged
  BMPC_F_TEAM_BUILD = 64,  // run the team instantiation (the one that carries the
                           // early-exit poll) even with one warp per instance
};

// Planner scoring parameters and outputs for the fused epilogue.
typedef struct {
  int kind;  // 0 cruise, 1 highspeed
  double v_cruise, v_max, y_rl, w1, w2;
  double heading_limit, residual_tol, ratio_min;
  double *meta, *min_ratio, *heading_max;  // (L)
  unsigned char* flags;                    // (L)
} bmpc_fused_score;

typedef struct {
  int m, l, L, S;       // obstacles, goals per scene, instances, scenes (L = S*l)
  int iters;            // AM sweeps in this launch
  int init_mode;        // BMPC_INIT_*
  int flags;            // BMPC_F_*
  int hist_offset;      // first history row written by this launch
  double a, b, v_min, v_max, a_max;
  const double* xi;     // [S][m][n] interleaved (xi_x, xi_y) pairs
  const double* xis;    // the same pairs in the ellipse frame: (b xi_x, a xi_y)
  const float* xs32;    // those pairs rounded to fp32 (NaN beyond the prefilter bound)
  const float* boxes;   // [S][ceil(n/32)][m] float4 obstacle boxes per sample slot, or NULL
  float* skipg;         // clearance-skipping scratch in global memory (long horizons, fp64):
                        // [BMPC_SKIPG_SMS][BMPC_MAX_WARPS][npad] (float2 P0, then float M0^2), or NULL
  const double* b_xy;   // [12][L]
  const double* b_psi;  // [4][L]
  // warm start (BMPC_INIT_WARM), reference AmState layouts (rows, L)
  const double *w_alpha, *w_d, *w_alpha_a, *w_d_a, *w_v, *w_cpsi;
  const double *w_lx, *w_ly, *w_lp;   // may be NULL (zero multipliers)
  const unsigned char* w_mask;        // may be NULL (every instance warm); 0 = cold
  double* carry;        // [L][5*nb]: lambda_x, lambda_y, lambda_psi, G_x, G_y
  double *c_x, *c_y, *c_psi, *l_x, *l_y, *l_psi;  // (nb, L)
  double* v_out;        // (n, L)
  double* hist;         // [rows][3][L]
  double* res_final;    // [3][L]
  bmpc_fused_score score;  // used with BMPC_F_SCORE
  // global early stop (solver.py:437-439), one 64-bit word per sweep: its high
  // half is non-zero once an instance's worst residual after sweep hist_offset
  // + t is not <= tol; with BMPC_F_POLL its low half counts the instances that
  // finished that sweep (so a sweep is decided converged at count L, flag 0)
  double tol;
  unsigned long long* notconv;
  const int* iters_dev;  // non-NULL: sweep count read on the device (0 = nothing to do)
  int team;              // warps per instance (1, 2 or 4)
} bmpc_solve_args;

// Doubles of carried state per instance: lambda_x, lambda_y, lambda_psi, G_x,
// G_y (5 nb), then the xy and psi KKT solutions [c; mu] (2 (nb+6) + nb+4).
#ifdef __CUDACC__
__host__ __device__
#endif
static inline int carry_doubles(int nb) { return 5 * nb + 2 * (nb + 6) + (nb + 4); }

// Fused scoring (sample_plan + filter_candidates + meta_cost), warp per instance.
typedef struct {
  int n, npad, nb, m, l, L;
  double a, b;
  int kind;  // 0 cruise, 1 highspeed
  double v_cruise, v_max, y_rl, w1, w2;
  double heading_limit, residual_tol, ratio_min;
  const double* PT;
  const double* xi;  // packed (S, m, n) (xi_x, xi_y) pairs
  const double *c_x, *c_y, *c_psi, *res_final;
  double *meta, *min_ratio, *heading_max;
  unsigned char* flags;  // bit0 heading ok, bit1 residual ok, bit2 collision ok
} bmpc_score_args;

#ifdef __cplusplus
}
#endif

#ifdef __cplusplus
#ifdef __CUDACC__
#define BMPC_HD __host__ __device__
#else
#define BMPC_HD
#endif
// Per-warp shared scratch of the persistent kernel (csrc/am_solve_kernel.cuh):
// 64 doubles of QP vectors (c_xy pairs, c_psi, residuals), the per-sample arrays (theta, xdot, ydot and,
// for npad <= 128, x and y), and the 32 x 33 transpose buffer.
#ifndef BMPC_XY_NPAD_MAX
#define BMPC_XY_NPAD_MAX 128
#endif
#ifndef BMPC_MAX_WARPS
#define BMPC_MAX_WARPS 8  // warps (instances) per CTA; the kernel's launch bound is 32x this
#endif
#define BMPC_SKIPG_SMS 256  // SM ids covered by the global clearance scratch (a block on a higher id never skips)
// Clearance skipping of obstacle slots (am_solve_kernel.cuh): 12 bytes per
// sample and warp of recorded positions and clearances.
#ifndef BMPC_SKIP
#define BMPC_SKIP 1
#endif
BMPC_HD constexpr size_t bmpc_skip_bytes(int npad, int warps) { return BMPC_SKIP ? (size_t)warps * npad * 12 : 0; }
BMPC_HD constexpr bool bmpc_stores_xy(int npad) { return npad <= BMPC_XY_NPAD_MAX; }
// Doubles of the image's basis part in shared memory: P^T, Pdot^T, Pddot^T in
// fp64, or in fp32 (the fp32 mode; npad is a multiple of 32, so this is whole).
BMPC_HD constexpr int bmpc_basis_doubles(int nb, int npad, bool f32) {
  return f32 ? 3 * nb * npad / 2 : 3 * nb * npad;
}
// fp32 mode per-sample arrays (floats, in the team's sample-array region):
// theta, xdot, ydot, and the ellipse-frame positions (b x, a y), then the fp32
// copies of the coefficients (32 c_xy pair slots, 16 c_psi).  They fit the
// fp64 region for every npad (224: 584 of 672 doubles).
BMPC_HD constexpr int bmpc_f32_sample_doubles(int npad) { return (5 * npad + 48) / 2; }
BMPC_HD constexpr int bmpc_sample_arrays(int npad) { return bmpc_stores_xy(npad) ? 5 : 3; }
// Team layout (team = the TW warps sharing one instance): per warp 64 QP
// doubles + the 32 x 33 transpose buffer + 72 exchange doubles; per team the
// per-sample arrays once.
BMPC_HD constexpr int bmpc_warp_private_doubles() { return 64 + 32 * 33 + 72; }
BMPC_HD constexpr int bmpc_team_doubles(int npad, int tw) {
  return tw * bmpc_warp_private_doubles() + bmpc_sample_arrays(npad) * npad;
}
#endif
