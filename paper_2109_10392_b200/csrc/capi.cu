// capi.cu -- extern "C" boundary (include/batchmpc_b200.h) over the sm_100a kernels.
#include <cuda_runtime.h>
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/batchmpc_b200.h"
#include "am_args.h"
#include "score.cuh"

namespace bmpc {
cudaError_t launch_am_solve(const bmpc_dev_consts& C, const bmpc_solve_args& A, int warps,
                            cudaStream_t st);
size_t am_solve_smem_bytes(int nb, int npad, int kxs, int kps, int warps, int team, bool f32);
cudaError_t op_obstacle_update(int n, int l, long long mn, const double* x, const double* y,
                               const double* xi_x, const double* xi_y, double a, double b,
                               double* alpha, double* d, cudaStream_t st);
cudaError_t op_accel_update(long long nl, const double* xdd, const double* ydd, double a_max,
                            double* alpha_a, double* d_a, cudaStream_t st);
cudaError_t op_v_update(long long nl, const double* xd, const double* yd, double v_min,
                        double v_max, double* v, cudaStream_t st);
cudaError_t op_assemble_g(int n, int l, long long mn, const double* xi_x, const double* xi_y,
                          const double* alpha, const double* d, const double* alpha_a,
                          const double* d_a, const double* v, const double* psi, double a,
                          double b, double* g_x, double* g_y, cudaStream_t st);
cudaError_t op_residual_vectors(int n, int l, long long mn, const double* x, const double* y,
                                const double* xd, const double* yd, const double* xdd,
                                const double* ydd, const double* psi, const double* xi_x,
                                const double* xi_y, const double* alpha, const double* d,
                                const double* alpha_a, const double* d_a, const double* v,
                                double a, double b, double* r_x, double* r_y, cudaStream_t st);
cudaError_t op_tail(bool with_angles, int n, int l, long long mn, const double* x, const double* y,
                    const double* xd, const double* yd, const double* xdd, const double* ydd,
                    const double* psi, const double* xi_x, const double* xi_y, double v_min,
                    double v_max, double a_max, double a, double b, double* alpha, double* d,
                    double* alpha_a, double* d_a, double* v, double* r_x, double* r_y,
                    double* g_x, double* g_y, double* sq_obs, double* sq_acc, double* sq_nonhol,
                    cudaStream_t st);
cudaError_t op_sample(int n, int npad, int nb, int L, const double* PT, const double* c_x,
                      const double* c_y, const double* c_psi, double* x, double* y, double* xd,
                      double* yd, double* xdd, double* ydd, double* psi, double* psid, double* v,
                      cudaStream_t st);
using ScoreArgs = bmpc_score_args;
cudaError_t op_score(const ScoreArgs& S, cudaStream_t st);
cudaError_t op_score_samples(const ScoreParams& sp, int l, int L, const double* xi2, const double* x,
                             const double* y, const double* psi, const double* v, const double* res,
                             double* meta, double* min_ratio, double* heading_max, uint8_t* flags,
                             cudaStream_t st);
cudaError_t op_argmin(int S, int l, const double* meta, const uint8_t* flags, long long* best,
                      long long* best_all, long long* best_hc, long long* nfeas, cudaStream_t st);
cudaError_t op_obstacle_boxes(int S, int m, int n, const double* xis, float* boxes, cudaStream_t st);
cudaError_t op_pack_xi(long long total, const double* xi_x, const double* xi_y, double* out,
                       cudaStream_t st, double* scaled = nullptr, double a = 1.0, double b = 1.0,
                       int* zero = nullptr, int nzero = 0);
cudaError_t op_early_stop(int max_iter, const unsigned long long* notconv, int* rerun, int* status, int* status2,
                          cudaStream_t st);
cudaError_t op_assemble(int S, int V, int m, int n, int l, const double* veh, const int* nveh,
                        const double* ego, const double* goals, const double* rel, double* xi_x,
                        double* xi_y, double* b_xy, double* b_psi, cudaStream_t st);
cudaError_t dfma_peak_tflops(int reps, double* tflops, cudaStream_t st);
cudaError_t op_math_check(int fn, long long n, const double* a, const double* b, double* out,
                          double* out2, cudaStream_t st);
cudaError_t latency_probe(int which, double* cyc_per_op, cudaStream_t st);
cudaError_t op_project(const bmpc_dev_consts& C, int mode, int m, long long L, const double* g,
                       double* out, cudaStream_t st);
cudaError_t op_kkt_apply(const bmpc_dev_consts& C, int which, long long L, const double* rhs,
                         double* out_x, double* out_y, cudaStream_t st);
cudaError_t op_heading(const bmpc_dev_consts& C, long long L, const double* c_x, const double* c_y,
                       double* theta, cudaStream_t st);
cudaError_t op_d_obs(int n, long long l, long long mn, const double* x, const double* y,
                     const double* xi_x, const double* xi_y, const double* alpha, double a,
                     double b, double* d, cudaStream_t st);
cudaError_t op_collision_ratios(int n, long long l, long long mn, const double* x, const double* y,
                                const double* xi_x, const double* xi_y, double a, double b,
                                double* out, cudaStream_t st);
cudaError_t op_block_norms(int n, long long l, long long mn, const double* r_x, const double* r_y,
                           double* out, cudaStream_t st);
}  // namespace bmpc

struct bmpc_ctx {
  bmpc_dev_consts C;
  double* dmem = nullptr;  // one allocation for every constant
  double cond_xy = 0.0, cond_psi = 0.0;  // 1-norm condition numbers of the reduced Hessians
  int sms = 148;
  int smem_optin = 227 * 1024;
  // private stream-ordered pool for the per-call workspaces: freed blocks stay
  // cached (release threshold = max) without touching the device's default pool
  cudaMemPool_t pool = nullptr;
  // pinned staging for bmpc_plan_host's results (grown on demand)
  std::mutex stage_mu;
  void* stage = nullptr;
  size_t stage_bytes = 0;
};

static thread_local std::string g_err;
// reduced-Hessian condition number above which the QP steps refine
static constexpr double kRefineCond = 1.0e4;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  return fail(BMPC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(expr, where)                              \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------ host e2e ----
// Stream-ordered workspace from the context's private pool.
static inline cudaError_t ws_alloc(const bmpc_ctx* c, void** p, size_t bytes, cudaStream_t st) {
  return c->pool ? cudaMallocFromPoolAsync(p, bytes, c->pool, st) : cudaMallocAsync(p, bytes, st);
}

struct DevBuf {
  std::vector<void*> ptrs;
  const bmpc_ctx* ctx;
  cudaStream_t st;
  DevBuf(const bmpc_ctx* c, cudaStream_t s) : ctx(c), st(s) {}
  ~DevBuf() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (ws_alloc(ctx, &p, count * sizeof(T), st) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

extern "C" {

const char* bmpc_last_error(void) { return g_err.c_str(); }
int bmpc_abi_version(void) { return 2; }

int bmpc_abi_layout(long long* out, int n) {
  // sizes and last-field offsets of the ABI structs, for binding checks
  const long long v[] = {
      (long long)sizeof(bmpc_problem),    (long long)offsetof(bmpc_problem, a_max),
      (long long)sizeof(bmpc_solve_opts), (long long)offsetof(bmpc_solve_opts, team_warps),
      (long long)sizeof(bmpc_solve_out),  (long long)offsetof(bmpc_solve_out, converged),
      (long long)sizeof(bmpc_score_spec), (long long)offsetof(bmpc_score_spec, collision_margin),
      (long long)sizeof(bmpc_score_out),  (long long)offsetof(bmpc_score_out, n_feasible)};
  const int count = (int)(sizeof(v) / sizeof(v[0]));
  if (!out) return count;
  for (int i = 0; i < n && i < count; ++i) out[i] = v[i];
  return count;
}

int bmpc_carry_doubles(const bmpc_ctx* ctx) { return ctx ? carry_doubles(ctx->C.nb) : -1; }

}  // extern "C"

// Gauss-Jordan inverse with partial pivoting in extended precision (the
// reduced QP blocks are at most 12 x 12); false if singular.
static bool inverse_ld(int k, std::vector<long double>& a, std::vector<long double>& inv) {
  inv.assign((size_t)k * k, 0.0L);
  for (int i = 0; i < k; ++i) inv[(size_t)i * k + i] = 1.0L;
  for (int col = 0; col < k; ++col) {
    int piv = col;
    for (int r = col + 1; r < k; ++r)
      if (fabsl(a[(size_t)r * k + col]) > fabsl(a[(size_t)piv * k + col])) piv = r;
    if (a[(size_t)piv * k + col] == 0.0L) return false;
    if (piv != col)
      for (int j = 0; j < k; ++j) {
        std::swap(a[(size_t)piv * k + j], a[(size_t)col * k + j]);
        std::swap(inv[(size_t)piv * k + j], inv[(size_t)col * k + j]);
      }
    const long double d = a[(size_t)col * k + col];
    for (int j = 0; j < k; ++j) {
      a[(size_t)col * k + j] /= d;
      inv[(size_t)col * k + j] /= d;
    }
    for (int r = 0; r < k; ++r) {
      if (r == col) continue;
      const long double f = a[(size_t)r * k + col];
      if (f == 0.0L) continue;
      for (int j = 0; j < k; ++j) {
        a[(size_t)r * k + j] -= f * a[(size_t)col * k + j];
        inv[(size_t)r * k + j] -= f * inv[(size_t)col * k + j];
      }
    }
  }
  return true;
}

// Null-space form of one KKT block K = [[H, A^T], [A, 0]] (solver.py:120-176).
// The default BoundarySpec pins orders 0..rows/2-1 at both ends, and the
// Bernstein endpoint rows are supported on the first / last rows/2
// coefficients only (basis.py:45-49), so A fixes those coefficients c_f
// through a triangular system and leaves the middle ones free:
//   c_f = T^-1 b,  c_m = H_mm^-1 (rhs_m - H_mf c_f).
// Outputs in the full coefficient index space: Z = H_mm^-1 placed in the
// middle block (zero rows/columns for fixed coefficients), B (nb x rows) with
// c = Z rhs + B b, and the 1-norm condition number of H_mm.
static int reduced_qp(int nb, int rows, const double* K, std::vector<double>& Z,
                      std::vector<double>& B, double* cond1) {
  const int kd = nb + rows, h = rows / 2, nm = nb - rows;
  if (nm < 0) return fail(BMPC_EINVAL, "boundary rows exceed the basis size");
  auto fixed_col = [&](int q) { return q < h ? q : nb - rows + q; };  // q-th fixed coefficient
  auto mid_col = [&](int q) { return h + q; };
  for (int r = 0; r < rows; ++r)
    for (int q = 0; q < nm; ++q)
      if (K[(size_t)(nb + r) * kd + mid_col(q)] != 0.0)
        return fail(BMPC_EINVAL, "boundary rows are not supported on the end coefficients");
  std::vector<long double> T((size_t)rows * rows), Ti, Hm((size_t)nm * nm), Hi;
  for (int r = 0; r < rows; ++r)
    for (int q = 0; q < rows; ++q) T[(size_t)r * rows + q] = K[(size_t)(nb + r) * kd + fixed_col(q)];
  if (!inverse_ld(rows, T, Ti)) return fail(BMPC_ESINGULAR, "KKT factorization failed: singular boundary block");
  for (int i = 0; i < nm; ++i)
    for (int j = 0; j < nm; ++j) Hm[(size_t)i * nm + j] = K[(size_t)mid_col(i) * kd + mid_col(j)];
  std::vector<long double> Hm0 = Hm;
  if (nm > 0 && !inverse_ld(nm, Hm, Hi)) return fail(BMPC_ESINGULAR, "KKT factorization failed: singular reduced Hessian");
  Z.assign((size_t)nb * nb, 0.0);
  B.assign((size_t)nb * rows, 0.0);
  for (int i = 0; i < nm; ++i)
    for (int j = 0; j < nm; ++j) Z[(size_t)mid_col(i) * nb + mid_col(j)] = (double)Hi[(size_t)i * nm + j];
  for (int q = 0; q < rows; ++q)
    for (int r = 0; r < rows; ++r) B[(size_t)fixed_col(q) * rows + r] = (double)Ti[(size_t)q * rows + r];
  for (int i = 0; i < nm; ++i)
    for (int r = 0; r < rows; ++r) {
      long double s = 0.0L;  // -(H_mm^-1 H_mf T^-1)[i][r]
      for (int j = 0; j < nm; ++j) {
        long double hf = 0.0L;
        for (int q = 0; q < rows; ++q)
          hf += (long double)K[(size_t)mid_col(j) * kd + fixed_col(q)] * Ti[(size_t)q * rows + r];
        s += Hi[(size_t)i * nm + j] * hf;
      }
      B[(size_t)mid_col(i) * rows + r] = (double)(-s);
    }
  long double n1 = 0.0L, n2 = 0.0L;
  for (int j = 0; j < nm; ++j) {
    long double s1 = 0.0L, s2 = 0.0L;
    for (int i = 0; i < nm; ++i) {
      s1 += fabsl(Hm0[(size_t)i * nm + j]);
      s2 += fabsl(Hi[(size_t)i * nm + j]);
    }
    n1 = s1 > n1 ? s1 : n1;
    n2 = s2 > n2 ? s2 : n2;
  }
  *cond1 = (double)(n1 * n2);
  for (double v : Z)
    if (!isfinite(v)) return fail(BMPC_ESINGULAR, "KKT factorization failed: non-finite reduced inverse");
  for (double v : B)
    if (!isfinite(v)) return fail(BMPC_ESINGULAR, "KKT factorization failed: non-finite boundary map");
  return BMPC_OK;
}

extern "C" {

int bmpc_ctx_create(int n, int nb, double rho, const double* P, const double* Pdot,
                    const double* Pddot, const double* tau, const double* kinv_axis,
                    const double* k_axis, const double* kinv_psi, const double* k_psi,
                    const double* ftf_axis, bmpc_ctx** out) {
  if (!out || !P || !Pdot || !Pddot || !tau || !kinv_axis || !k_axis || !kinv_psi || !k_psi ||
      !ftf_axis)
    return fail(BMPC_EINVAL, "bmpc_ctx_create: null argument");
  if (nb < 6 || nb > 16) return fail(BMPC_EINVAL, "bmpc_ctx_create: need 6 <= n_b <= 16");
  if (n < 2 || n > 256) return fail(BMPC_EINVAL, "bmpc_ctx_create: need 2 <= n <= 256");
  if (!(rho > 0.0)) return fail(BMPC_EINVAL, "bmpc_ctx_create: rho must be positive");
  const int rx = nb + 6, rp = nb + 4;
  for (int i = 0; i < rx * rx; ++i)
    if (!isfinite(kinv_axis[i])) return fail(BMPC_ESINGULAR, "KKT xy inverse is not finite");
  for (int i = 0; i < rp * rp; ++i)
    if (!isfinite(kinv_psi[i])) return fail(BMPC_ESINGULAR, "KKT psi inverse is not finite");
  // null-space form of both QP blocks (the persistent kernel's QP steps)
  std::vector<double> Zx, Bx, Zp, Bp;
  double cond_x = 0.0, cond_p = 0.0;
  int rc = reduced_qp(nb, 6, k_axis, Zx, Bx, &cond_x);
  if (rc != BMPC_OK) return rc;
  rc = reduced_qp(nb, 4, k_psi, Zp, Bp, &cond_p);
  if (rc != BMPC_OK) return rc;
  // = 32 * NKM of the kernel instantiations (csrc/am_inst.cu)
  const int npad = n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 224 ? 224 : 256));
  const int kxs = rx | 1, kps = rp | 1, kms = nb | 1;
  const size_t nPT = (size_t)3 * nb * npad, nKx = (size_t)rx * kxs, nKp = (size_t)rp * kps;
  // The kernel's shared-memory image (every block an even number of doubles,
  // so tau and the total stay 16-byte aligned for the bulk copy):
  //   P^T, Pdot^T, Pddot^T | F_axis^T F_axis, P^T P, Pddot^T Pddot, Pdot^T Pdot |
  //   Z_xy, H_xy, Z_psi, H_psi | B_xy [nb][8], B_psi [nb][4] | tau
  // followed in global memory only by the full KKT inverse / matrix pairs
  // (the step API's refined solves, csrc/steps.cu).
  // Layout of the one allocation: the plain transposed basis PT (the ABI's
  // bmpc_ctx_info, the stand-alone kernels), then the image, then the KKT pairs.
  const size_t nimg = bmpc_const_image_doubles(nb, npad);
  const size_t oI = nPT;  // image start (nPT is even: 16-byte aligned)
  // ... and last the fp32 copy of the image's basis part (the fp32 mode's
  // shared-memory basis; nPT floats = nPT / 2 doubles, nPT even)
  const size_t oF = nPT + nimg + 2 * nKx + 2 * nKp;
  std::vector<double> h(oF + nPT / 2, 0.0);
  const double* mats[3] = {P, Pdot, Pddot};
  for (int q = 0; q < 3; ++q)
    for (int i = 0; i < nb; ++i)
      for (int k = 0; k < n; ++k) {
        const double v = mats[q][(size_t)k * nb + i];
        h[((size_t)q * nb + i) * npad + k] = v;
        h[oI + bmpc_basis_index(q * nb + i, k, npad)] = v;
        reinterpret_cast<float*>(h.data() + oF)[bmpc_basis_index(q * nb + i, k, npad)] = (float)v;
      }
  const size_t oM = oI + (size_t)3 * nb * npad;
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j < nb; ++j) h[oM + (size_t)i * kms + j] = ftf_axis[(size_t)i * nb + j];
  // P^T P, Pddot^T Pddot, Pdot^T Pdot right after F_axis^T F_axis (the
  // exact-form sweep and multiplier identities), in extended precision
  const double* grams[3] = {P, Pddot, Pdot};
  for (int q = 0; q < 3; ++q)
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) {
        long double acc = 0.0L;
        for (int k = 0; k < n; ++k)
          acc += (long double)grams[q][(size_t)k * nb + i] * grams[q][(size_t)k * nb + j];
        h[oM + ((size_t)(q + 1) * nb + i) * kms + j] = (double)acc;
      }
  size_t o = oM + (size_t)4 * nb * kms;
  const double* qp[4] = {Zx.data(), k_axis, Zp.data(), k_psi};
  const int qps[4] = {nb, rx, nb, rp};  // source row strides (H = top-left nb x nb of K)
  for (int q = 0; q < 4; ++q, o += (size_t)nb * kms)
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) h[o + (size_t)i * kms + j] = qp[q][(size_t)i * qps[q] + j];
  for (int i = 0; i < nb; ++i)
    for (int r = 0; r < 6; ++r) h[o + (size_t)i * 8 + r] = Bx[(size_t)i * 6 + r];
  o += (size_t)8 * nb;
  for (int i = 0; i < nb; ++i)
    for (int r = 0; r < 4; ++r) h[o + (size_t)i * 4 + r] = Bp[(size_t)i * 4 + r];
  o += (size_t)4 * nb;
  const size_t otau = o;
  for (int k = 0; k < n; ++k) h[otau + k] = tau[k];
  size_t offs[4];
  o = oI + nimg;
  const double* blocks[4] = {kinv_axis, k_axis, kinv_psi, k_psi};
  const int dims[4] = {rx, rx, rp, rp}, strides[4] = {kxs, kxs, kps, kps};
  for (int q = 0; q < 4; ++q) {
    offs[q] = o;
    for (int i = 0; i < dims[q]; ++i)
      for (int j = 0; j < dims[q]; ++j) h[o + (size_t)i * strides[q] + j] = blocks[q][(size_t)i * dims[q] + j];
    o += (size_t)dims[q] * strides[q];
  }
  // One refinement step (solver.py:164-168) per QP only where the reduced
  // Hessian is ill-conditioned: the explicit inverse loses about cond * eps.
  // BMPC_QP_REFINE=0/1/2/3 (bit 0 xy, bit 1 psi) overrides, for experiments.
  int refine = (cond_x > kRefineCond ? 1 : 0) | (cond_p > kRefineCond ? 2 : 0);
  if (const char* env = getenv("BMPC_QP_REFINE")) refine = atoi(env) & 3;
  bmpc_ctx* c = new bmpc_ctx();
  cudaError_t e = cudaMalloc(&c->dmem, h.size() * sizeof(double));
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "bmpc_ctx_create/cudaMalloc"); }
  e = cudaMemcpy(c->dmem, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(c->dmem); delete c; return cuda_fail(e, "bmpc_ctx_create/memcpy"); }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // Per-call workspaces come from a private stream-ordered pool that keeps
  // freed blocks cached instead of trimming them back to the OS at every
  // synchronisation (the device's default pool is left as the caller set it).
  cudaMemPoolProps props;
  memset(&props, 0, sizeof(props));
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  if (cudaMemPoolCreate(&c->pool, &props) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  } else {
    c->pool = nullptr;
    cudaGetLastError();
  }
  c->C.n = n;
  c->C.npad = npad;
  c->C.nb = nb;
  c->C.kxs = kxs;
  c->C.kps = kps;
  c->C.kms = kms;
  c->C.rho = rho;
  c->C.PT = c->dmem;
  c->C.IMG = c->dmem + oI;
  c->C.Kxf = c->dmem + offs[0];
  c->C.Kxa = c->dmem + offs[1];
  c->C.Kpf = c->dmem + offs[2];
  c->C.Kpa = c->dmem + offs[3];
  c->C.M = c->dmem + oM;
  c->C.tau = c->dmem + otau;
  c->C.const_doubles = (int)nimg;
  c->C.IMGF = reinterpret_cast<const float*>(c->dmem + oF);
  c->C.refine = refine;
  c->cond_xy = cond_x;
  c->cond_psi = cond_p;
  *out = c;
  return BMPC_OK;
}

int bmpc_ctx_destroy(bmpc_ctx* ctx) {
  if (!ctx) return BMPC_OK;
  cudaFree(ctx->dmem);
  if (ctx->stage) cudaFreeHost(ctx->stage);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);  // released once outstanding blocks are freed
  delete ctx;
  return BMPC_OK;
}

int bmpc_reduced_qp(int nb, int rows, const double* k, double* z, double* bmap, double* cond1) {
  if (!k || !z || !bmap || !cond1 || (rows != 4 && rows != 6) || nb < rows || nb > 16)
    return fail(BMPC_EINVAL, "bmpc_reduced_qp: bad arguments");
  std::vector<double> Z, B;
  const int rc = reduced_qp(nb, rows, k, Z, B, cond1);
  if (rc != BMPC_OK) return rc;
  memcpy(z, Z.data(), Z.size() * sizeof(double));
  memcpy(bmap, B.data(), B.size() * sizeof(double));
  return BMPC_OK;
}

int bmpc_ctx_qp_info(const bmpc_ctx* ctx, double* cond_xy, double* cond_psi, int* refine) {
  if (!ctx) return fail(BMPC_EINVAL, "null ctx");
  if (cond_xy) *cond_xy = ctx->cond_xy;
  if (cond_psi) *cond_psi = ctx->cond_psi;
  if (refine) *refine = ctx->C.refine;
  return BMPC_OK;
}

int bmpc_ctx_info(const bmpc_ctx* ctx, int* n, int* npad, int* nb, const double** PT) {
  if (!ctx) return fail(BMPC_EINVAL, "null ctx");
  if (n) *n = ctx->C.n;
  if (npad) *npad = ctx->C.npad;
  if (nb) *nb = ctx->C.nb;
  if (PT) *PT = ctx->C.PT;
  return BMPC_OK;
}

static int check_problem(const bmpc_ctx* ctx, const bmpc_problem* p) {
  if (!ctx || !p) return fail(BMPC_EINVAL, "null ctx/problem");
  if (p->m < 0 || p->l < 0 || p->S < 1) return fail(BMPC_EINVAL, "invalid m/l/S");
  if (!(0.0 < p->v_min && p->v_min < p->v_max))
    return fail(BMPC_EINVAL, "need 0 < v_min < v_max");
  if (!(p->a_max > 0.0)) return fail(BMPC_EINVAL, "a_max must be positive");
  if (!(p->a >= p->b && p->b > 0.0)) return fail(BMPC_EINVAL, "ellipse axes must satisfy a >= b > 0");
  if (p->l > 0 && (!p->b_xy || !p->b_psi)) return fail(BMPC_EINVAL, "null boundary vectors");
  if (p->m > 0 && (!p->xi_x || !p->xi_y)) return fail(BMPC_EINVAL, "null obstacle predictions");
  return BMPC_OK;
}

// Warps (= instances) per CTA: about one CTA per SM for small batches, at most
// 8 (the register file holds 8 warps of this kernel), and never more than the
// opt-in shared memory per block allows.
static int auto_warps(const bmpc_ctx* ctx, int L, int req, int team, bool f32) {
  // warps per block: a multiple of the team size, about one block per SM
  int ipb = req > 0 ? req / team : (L + ctx->sms - 1) / ctx->sms;
  if (ipb < 1) ipb = 1;
  if (ipb * team > BMPC_MAX_WARPS) ipb = BMPC_MAX_WARPS / team;
  while (ipb > 1 && bmpc::am_solve_smem_bytes(ctx->C.nb, ctx->C.npad, ctx->C.kxs, ctx->C.kps,
                                              ipb * team, team, f32) > (size_t)ctx->smem_optin)
    --ipb;
  return ipb * team;
}

// Offset (doubles) of the boxes: after the fp32 pairs, 16-byte aligned.
static inline size_t box_offset(size_t tot) { return (5 * tot + 1) & ~(size_t)1; }
// Bytes of the packed predictions: raw pairs (2 tot doubles), ellipse-frame
// pairs (2 tot), their fp32 copy (tot), the per-slot obstacle boxes.
// ... and, for long horizons (n > 128), the clearance-skipping scratch of the
// unstaged fp64 culling kernels: 12 bytes per sample for every resident warp,
// indexed by SM and warp (one block per SM there: shared memory is full).
static inline size_t skip_scratch_offset(const bmpc_problem* p, int n) {  // doubles
  const size_t tot = (size_t)p->S * p->m * n;
  return (box_offset(tot) + 2 * (size_t)p->S * ((n + 31) / 32) * p->m + 1) & ~(size_t)1;
}
static inline size_t skip_scratch_doubles(int n) {
  const size_t npad = n <= 224 ? 224 : 256;
  return n > 128 ? (size_t)BMPC_SKIPG_SMS * BMPC_MAX_WARPS * npad * 12 / 8 : 0;
}
static size_t xi_work_bytes(const bmpc_problem* p, int n) {
  const size_t tot = (size_t)p->S * p->m * n;
  return tot == 0 ? 0 : (skip_scratch_offset(p, n) + skip_scratch_doubles(n)) * sizeof(double);
}

// Obstacle culling by bounding boxes pays from about two dozen obstacles (c2
// m = 30: -5%, c4 m = 50: -18%; c1 m = 10 / c3 m = 20: +7% / +3%); not in teams.
static bool use_cull(const bmpc_problem* p, const bmpc_solve_opts* o, int extra_flags) {
  static const int cull_min_m = getenv("BMPC_CULL_MIN_M") ? atoi(getenv("BMPC_CULL_MIN_M")) : 24;
  return p->m >= cull_min_m && o->team_warps <= 1 && !(extra_flags & BMPC_F_TEAM_BUILD);
}

// Launch `iters` sweeps; xi2 is the packed (S, m, n) double2 buffer.
static int launch_sweeps(bmpc_ctx* ctx, const bmpc_problem* p, const double* xi2,
                         const bmpc_solve_opts* o, int iters, int init_mode, int hist_offset,
                         double* carry, int write_carry, bmpc_solve_out* out, cudaStream_t st,
                         const bmpc_fused_score* fsc = nullptr,
                         unsigned long long* notconv = nullptr, const int* iters_dev = nullptr,
                         int extra_flags = 0) {
  const int L = p->S * p->l;
  bmpc_solve_args A;
  memset(&A, 0, sizeof(A));
  A.m = p->m;
  A.l = p->l;
  A.L = L;
  A.S = p->S;
  A.iters = iters;
  A.init_mode = init_mode;
  A.flags = (out->history ? BMPC_F_HISTORY : 0) | ((o->want_v && out->v) ? BMPC_F_V : 0) |
            (write_carry ? BMPC_F_CARRY : 0) | (o->precision == 1 ? BMPC_F_F32 : 0) | extra_flags;
  A.hist_offset = hist_offset;
  A.a = p->a;
  A.b = p->b;
  A.v_min = p->v_min;
  A.v_max = p->v_max;
  A.a_max = p->a_max;
  A.xi = xi2;
  A.xis = xi2 ? xi2 + 2 * (size_t)p->S * p->m * ctx->C.n : nullptr;
  A.xs32 = xi2 ? reinterpret_cast<const float*>(xi2 + 4 * (size_t)p->S * p->m * ctx->C.n) : nullptr;
  A.boxes = (xi2 && use_cull(p, o, extra_flags))
                ? reinterpret_cast<const float*>(xi2 + box_offset((size_t)p->S * p->m * ctx->C.n))
                : nullptr;
  // (only the fp64 culling kernels of long horizons use it)
  A.skipg = (A.boxes && ctx->C.n > 128 && o->precision == 0)
                ? reinterpret_cast<float*>(const_cast<double*>(xi2) + skip_scratch_offset(p, ctx->C.n))
                : nullptr;
  A.b_xy = p->b_xy;
  A.b_psi = p->b_psi;
  A.w_alpha = o->w_alpha;
  A.w_d = o->w_d;
  A.w_alpha_a = o->w_alpha_a;
  A.w_d_a = o->w_d_a;
  A.w_v = o->w_v;
  A.w_cpsi = o->w_c_psi;
  A.w_mask = o->w_mask;
  A.team = o->team_warps > 1 ? o->team_warps : 1;
  const bool keep = o->keep_multipliers != 0;
  A.w_lx = keep ? o->w_l_x : nullptr;
  A.w_ly = keep ? o->w_l_y : nullptr;
  A.w_lp = keep ? o->w_l_psi : nullptr;
  A.carry = carry;
  A.c_x = out->c_x;
  A.c_y = out->c_y;
  A.c_psi = out->c_psi;
  A.l_x = out->l_x;
  A.l_y = out->l_y;
  A.l_psi = out->l_psi;
  A.v_out = out->v;
  A.hist = out->history;
  A.res_final = out->res_final;
  A.tol = o->tol;
  A.notconv = notconv;
  A.iters_dev = iters_dev;
  if (fsc) {
    A.flags |= BMPC_F_SCORE;
    A.score = *fsc;
  }
  if (L == 0 || iters <= 0) return BMPC_OK;
  CK(bmpc::launch_am_solve(ctx->C, A, auto_warps(ctx, L, o->warps_per_block, A.team, o->precision == 1), st),
     "am_solve launch");
  return BMPC_OK;
}

static bool is_warm(const bmpc_solve_opts* o) {
  return o->w_alpha || o->w_d || o->w_alpha_a || o->w_d_a || o->w_v || o->w_c_psi;
}

static int check_warm(const bmpc_solve_opts* o, const bmpc_problem* p) {
  if (!is_warm(o)) return BMPC_OK;
  if (!o->w_alpha || !o->w_d || !o->w_alpha_a || !o->w_d_a || !o->w_v || !o->w_c_psi)
    return fail(BMPC_EINVAL, "warm start needs alpha, d, alpha_a, d_a, v and c_psi");
  if (o->keep_multipliers && (!o->w_l_x || !o->w_l_y || !o->w_l_psi))
    return fail(BMPC_EINVAL, "keep_multipliers needs the warm multipliers");
  (void)p;
  return BMPC_OK;
}

int bmpc_sweeps(bmpc_ctx* ctx, const bmpc_problem* p, const bmpc_solve_opts* o, int iters,
                int resume, int hist_offset, double* carry, int write_carry, bmpc_solve_out* out,
                void* stream) {
  int rc = check_problem(ctx, p);
  if (rc) return rc;
  if (!o || !out) return fail(BMPC_EINVAL, "null opts/out");
  if ((resume || write_carry) && !carry) return fail(BMPC_EINVAL, "carry buffer required");
  if ((rc = check_warm(o, p))) return rc;
  cudaStream_t st = S_(stream);
  const long long tot = (long long)p->S * p->m * ctx->C.n;
  double* xi2 = nullptr;
  if (tot > 0) {
    // raw pairs, then the ellipse-frame pairs for the sweeps' outside test (fp64
    // and the fp32 prefilter copy), then the obstacle boxes of the culling
    CK(ws_alloc(ctx, (void**)&xi2, xi_work_bytes(p, ctx->C.n), st), "workspace allocation");
    CK(bmpc::op_pack_xi(tot, p->xi_x, p->xi_y, xi2, st, xi2 + 2 * tot, p->a, p->b), "pack_xi");
    if (use_cull(p, o, 0))
      CK(bmpc::op_obstacle_boxes(p->S, p->m, ctx->C.n, xi2 + 2 * tot, (float*)(xi2 + box_offset(tot)), st),
         "boxes");
  }
  const int mode = resume ? BMPC_INIT_RESUME : (is_warm(o) ? BMPC_INIT_WARM : BMPC_INIT_COLD);
  rc = launch_sweeps(ctx, p, xi2, o, iters, mode, hist_offset, carry, write_carry, out, st);
  if (xi2) cudaFreeAsync(xi2, st);
  return rc;
}

// Work enqueued right after the sweeps (the per-scene argmin of bmpc_plan):
// issued before the early-stop check synchronises, and again after a re-run.
struct PostSolve {
  const bmpc_problem* p;
  const bmpc_score_out* so;
};
static int post_solve(const PostSolve* ps, cudaStream_t st);

static int solve_impl(bmpc_ctx* ctx, const bmpc_problem* p, const bmpc_solve_opts* o,
                      bmpc_solve_out* out, const bmpc_fused_score* fsc, void* stream,
                      const PostSolve* post = nullptr);

int bmpc_solve(bmpc_ctx* ctx, const bmpc_problem* p, const bmpc_solve_opts* o,
               bmpc_solve_out* out, void* stream) {
  return solve_impl(ctx, p, o, out, nullptr, stream);
}

static int check_spec(const bmpc_score_spec* spec) {
  if (!spec) return fail(BMPC_EINVAL, "null score spec");
  if (spec->kind != 0 && spec->kind != 1) return fail(BMPC_EINVAL, "unknown meta-cost kind");
  if (spec->w1 < 0 || spec->w2 < 0) return fail(BMPC_EINVAL, "meta-cost weights must be nonnegative");
  return BMPC_OK;
}

static bmpc_fused_score fused_from(const bmpc_score_spec* spec, const bmpc_score_out* so) {
  bmpc_fused_score f;
  f.kind = spec->kind;
  f.v_cruise = spec->v_cruise;
  f.v_max = spec->v_max;
  f.y_rl = spec->y_rl;
  f.w1 = spec->w1;
  f.w2 = spec->w2;
  f.heading_limit = spec->heading_limit;
  f.residual_tol = spec->residual_tol;
  f.ratio_min = 1.0 - spec->collision_margin;  // planner.py:244
  f.meta = so->meta_cost;
  f.min_ratio = so->min_ratio;
  f.heading_max = so->heading_max;
  f.flags = so->flags;
  return f;
}

int bmpc_plan(bmpc_ctx* ctx, const bmpc_problem* p, const bmpc_solve_opts* o, bmpc_solve_out* out,
              const bmpc_score_spec* spec, bmpc_score_out* so, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (!so || !so->meta_cost || !so->min_ratio || !so->heading_max || !so->flags)
    return fail(BMPC_EINVAL, "bmpc_plan: per-instance score outputs required");
  const bmpc_fused_score f = fused_from(spec, so);
  const PostSolve post{p, so};
  return solve_impl(ctx, p, o, out, &f, stream, &post);
}

static int post_solve(const PostSolve* ps, cudaStream_t st) {
  const bmpc_score_out* so = ps->so;
  if (so->best_index && so->argmin_all && so->argmin_hc && so->n_feasible)
    CK(bmpc::op_argmin(ps->p->S, ps->p->l, so->meta_cost, so->flags, so->best_index, so->argmin_all,
                       so->argmin_hc, so->n_feasible, st),
       "argmin");
  return BMPC_OK;
}

static int solve_impl(bmpc_ctx* ctx, const bmpc_problem* p, const bmpc_solve_opts* o,
                      bmpc_solve_out* out, const bmpc_fused_score* fsc, void* stream,
                      const PostSolve* post) {
  int rc = check_problem(ctx, p);
  if (rc) return rc;
  if (!o || !out) return fail(BMPC_EINVAL, "null opts/out");
  if (o->precision != 0 && o->precision != 1) return fail(BMPC_EINVAL, "precision must be 0 (fp64) or 1 (fp32 sample passes)");
  if (o->max_iter < 1) return fail(BMPC_EINVAL, "max_iter must be >= 1");
  if (o->team_warps != 0 && o->team_warps != 1 && o->team_warps != 2 && o->team_warps != 4)
    return fail(BMPC_EINVAL, "team_warps must be 0, 1, 2 or 4");
  if (o->team_warps > 1 && (o->precision != 0 || ctx->C.npad > 128))
    return fail(BMPC_EINVAL, "team_warps > 1 needs fp64 and n <= 128");
  if (!out->res_final) return fail(BMPC_EINVAL, "the res_final output is required");
  if ((rc = check_warm(o, p))) return rc;
  cudaStream_t st = S_(stream);
  const int L = p->S * p->l;
  const long long tot = (long long)p->S * p->m * ctx->C.n;
  const int mode = is_warm(o) ? BMPC_INIT_WARM : BMPC_INIT_COLD;
  const int M = o->max_iter;
  int status[2] = {M, 0};
  // One workspace: the packed predictions (raw pairs, then the ellipse-frame
  // pairs of the sweeps' outside test, fp64 and fp32) and the scratch -- M 64-bit per-sweep
  // early-stop words (not-converged flag | finished-instance count), then
  // ints: [0] the re-run sweep count, [1, 2] {iterations, converged}.
  // k_pack_xi zeroes the words (no memset call).
  const size_t xi_bytes = (xi_work_bytes(p, ctx->C.n) + 15) & ~(size_t)15;
  char* wsp = nullptr;
  CK(ws_alloc(ctx, (void**)&wsp, xi_bytes + (size_t)M * 8 + 4 * sizeof(int), st), "workspace allocation");
  double* xi2 = tot > 0 ? reinterpret_cast<double*>(wsp) : nullptr;
  unsigned long long* words = L > 0 ? reinterpret_cast<unsigned long long*>(wsp + xi_bytes) : nullptr;
  int* scr = L > 0 ? reinterpret_cast<int*>(wsp + xi_bytes + (size_t)M * 8) : nullptr;
  if (tot > 0 || L > 0)
    CK(bmpc::op_pack_xi(tot, p->xi_x, p->xi_y, xi2, st, xi2 ? xi2 + 2 * tot : nullptr, p->a, p->b,
                        reinterpret_cast<int*>(words), words ? 2 * M : 0),
       "pack_xi");
  // tol > 0 (fp64, n <= 128) runs on the team instantiation (see below)
  const int tb = (o->tol > 0.0 && o->precision == 0 && ctx->C.npad <= 128) ? BMPC_F_TEAM_BUILD : 0;
  if (tot > 0 && use_cull(p, o, tb))
    CK(bmpc::op_obstacle_boxes(p->S, p->m, ctx->C.n, xi2 + 2 * tot, (float*)(xi2 + box_offset(tot)), st),
       "boxes");
  // tol > 0 (fp64, n <= 128: the team instantiation's shapes): the first launch
  // exits once some sweep is known to be globally converged (BMPC_F_POLL), so
  // a solve that converges at sweep t costs about t + (t + 1) sweeps instead of
  // max_iter + (t + 1).  The re-run uses the same instantiation, without polling.
  const int poll = tb ? BMPC_F_POLL : 0;
  rc = launch_sweeps(ctx, p, xi2, o, M, mode, 0, nullptr, 0, out, st, fsc, words, nullptr, tb | poll);
  if (!rc && L > 0) {
    // Global early stop (solver.py:437-439): the first sweep whose worst
    // residual over every instance is <= tol.  When it is not the last one the
    // solve re-runs exactly that many sweeps (instances are independent and
    // deterministic, so the re-run reproduces the same iterates).  The decision
    // and the re-run launch stay on the device -- the second launch exits at
    // once when there is nothing to redo -- so nothing waits on the host.
    CK(bmpc::op_early_stop(M, words, scr, scr + 1, o->status_dev, st), "early_stop");
    rc = launch_sweeps(ctx, p, xi2, o, M, mode, 0, nullptr, 0, out, st, fsc, words, scr, tb);
  }
  if (!rc && post) rc = post_solve(post, st);
  if (!rc && L > 0 && !o->status_dev)
    CK(cudaMemcpyAsync(status, scr + 1, sizeof(status), cudaMemcpyDeviceToHost, st), "memcpy");
  cudaFreeAsync(wsp, st);
  if (rc) return rc;
  CK(cudaGetLastError(), "bmpc_solve");
  if (o->status_dev) {
    if (L == 0) {  // nothing ran: report max_iter sweeps, not converged
      const int h[2] = {M, 0};
      CK(cudaMemcpyAsync(o->status_dev, h, sizeof(h), cudaMemcpyHostToDevice, st), "memcpy");
      CK(cudaStreamSynchronize(st), "sync");
    }
    out->iterations = -1;
    out->converged = -1;
    return BMPC_OK;
  }
  CK(cudaStreamSynchronize(st), "sync");
  const int iters = status[0], converged = status[1];
  out->iterations = iters;
  out->converged = converged;
  return BMPC_OK;
}

int bmpc_score(bmpc_ctx* ctx, const bmpc_problem* p, const double* c_x, const double* c_y,
               const double* c_psi, const double* res_final, const bmpc_score_spec* spec,
               bmpc_score_out* out, void* stream) {
  int rc = check_problem(ctx, p);
  if (rc) return rc;
  if (!spec || !out || !c_x || !c_y || !c_psi || !res_final)
    return fail(BMPC_EINVAL, "bmpc_score: null argument");
  if (spec->kind != 0 && spec->kind != 1) return fail(BMPC_EINVAL, "unknown meta-cost kind");
  cudaStream_t st = S_(stream);
  const int L = p->S * p->l;
  const long long tot = (long long)p->S * p->m * ctx->C.n;
  double* xi2 = nullptr;
  if (tot > 0) {
    CK(ws_alloc(ctx, (void**)&xi2, tot * 2 * sizeof(double), st), "workspace allocation");
    CK(bmpc::op_pack_xi(tot, p->xi_x, p->xi_y, xi2, st), "pack_xi");
  }
  bmpc::ScoreArgs S;
  memset(&S, 0, sizeof(S));
  S.n = ctx->C.n;
  S.npad = ctx->C.npad;
  S.nb = ctx->C.nb;
  S.m = p->m;
  S.l = p->l;
  S.L = L;
  S.a = p->a;
  S.b = p->b;
  S.kind = spec->kind;
  S.v_cruise = spec->v_cruise;
  S.v_max = spec->v_max;
  S.y_rl = spec->y_rl;
  S.w1 = spec->w1;
  S.w2 = spec->w2;
  S.heading_limit = spec->heading_limit;
  S.residual_tol = spec->residual_tol;
  S.ratio_min = 1.0 - spec->collision_margin;
  S.PT = ctx->C.PT;
  S.xi = xi2;
  S.c_x = c_x;
  S.c_y = c_y;
  S.c_psi = c_psi;
  S.res_final = res_final;
  S.meta = out->meta_cost;
  S.min_ratio = out->min_ratio;
  S.heading_max = out->heading_max;
  S.flags = out->flags;
  if (!S.meta || !S.min_ratio || !S.heading_max || !S.flags)
    return fail(BMPC_EINVAL, "bmpc_score: per-instance outputs required");
  CK(bmpc::op_score(S, st), "score");
  if (out->best_index && out->argmin_all && out->argmin_hc && out->n_feasible)
    CK(bmpc::op_argmin(p->S, p->l, out->meta_cost, out->flags, out->best_index, out->argmin_all,
                       out->argmin_hc, out->n_feasible, st),
       "argmin");
  if (xi2) cudaFreeAsync(xi2, st);
  return BMPC_OK;
}

int bmpc_score_samples(const bmpc_problem* p, int n, const double* x, const double* y,
                       const double* psi, const double* v, const double* res,
                       const bmpc_score_spec* spec, bmpc_score_out* out, void* stream) {
  if (!p || !spec || !out || n < 1 || p->S < 0 || p->l < 0 || p->m < 0)
    return fail(BMPC_EINVAL, "bmpc_score_samples: bad argument");
  if (spec->kind != 0 && spec->kind != 1) return fail(BMPC_EINVAL, "unknown meta-cost kind");
  const int L = p->S * p->l;
  if (L > 0 && (!x || !y || !psi || !v)) return fail(BMPC_EINVAL, "bmpc_score_samples: null samples");
  if (L > 0 && (!out->meta_cost || !out->min_ratio || !out->heading_max || !out->flags))
    return fail(BMPC_EINVAL, "bmpc_score_samples: per-instance outputs required");
  cudaStream_t st = S_(stream);
  const long long tot = (long long)p->S * p->m * n;
  if (tot > 0 && (!p->xi_x || !p->xi_y)) return fail(BMPC_EINVAL, "bmpc_score_samples: null predictions");
  double* xi2 = nullptr;
  if (tot > 0) {
    CK(cudaMallocAsync(&xi2, tot * 2 * sizeof(double), st), "cudaMallocAsync");
    CK(bmpc::op_pack_xi(tot, p->xi_x, p->xi_y, xi2, st), "pack_xi");
  }
  const bmpc::ScoreParams sp{n, p->m, spec->kind, p->a, p->b, spec->v_cruise, spec->v_max,
                             spec->y_rl, spec->w1, spec->w2, spec->heading_limit,
                             spec->residual_tol, 1.0 - spec->collision_margin};
  CK(bmpc::op_score_samples(sp, p->l, L, xi2, x, y, psi, v, res, out->meta_cost, out->min_ratio,
                            out->heading_max, out->flags, st),
     "score_samples");
  if (out->best_index && out->argmin_all && out->argmin_hc && out->n_feasible)
    CK(bmpc::op_argmin(p->S, p->l, out->meta_cost, out->flags, out->best_index, out->argmin_all,
                       out->argmin_hc, out->n_feasible, st),
       "argmin");
  if (xi2) cudaFreeAsync(xi2, st);
  return BMPC_OK;
}

int bmpc_assemble(bmpc_ctx* ctx, int S, int V, int m, int l, const double* veh, const int* nveh,
                  const double* ego, const double* goals, const double* rel, double* xi_x,
                  double* xi_y, double* b_xy, double* b_psi, void* stream) {
  if (!ctx || S < 0 || V < 0 || m < 0 || l < 0) return fail(BMPC_EINVAL, "bmpc_assemble: bad size");
  if ((S > 0 && (!ego || !nveh || (V > 0 && !veh))) || (m > 0 && (!rel || !xi_x || !xi_y)) ||
      (l > 0 && (!goals || !b_xy || !b_psi)))
    return fail(BMPC_EINVAL, "bmpc_assemble: null argument");
  if ((size_t)(V + 4 * m) * sizeof(double) > 48 * 1024)
    return fail(BMPC_EINVAL, "bmpc_assemble: V + 4m too large (shared-memory staging)");
  CK(bmpc::op_assemble(S, V, m, ctx->C.n, l, veh, nveh, ego, goals, rel, xi_x, xi_y, b_xy, b_psi,
                       S_(stream)),
     "assemble");
  return BMPC_OK;
}

int bmpc_sample(bmpc_ctx* ctx, int L, const double* c_x, const double* c_y, const double* c_psi,
                double* x, double* y, double* xd, double* yd, double* xdd, double* ydd,
                double* psi, double* psid, double* v, void* stream) {
  if (!ctx || L < 0) return fail(BMPC_EINVAL, "bmpc_sample: bad argument");
  CK(bmpc::op_sample(ctx->C.n, ctx->C.npad, ctx->C.nb, L, ctx->C.PT, c_x, c_y, c_psi, x, y, xd, yd,
                     xdd, ydd, psi, psid, v, S_(stream)),
     "sample");
  return BMPC_OK;
}

// Results block of bmpc_plan_host (arena order): coefficients (c_x, c_y,
// c_psi), res_final, then with scoring meta_cost, min_ratio, heading_max, the
// four per-scene index rows, flags, and the {iterations, converged} status.
struct ResultsLayout {
  size_t coef, rf, meta, mr, hm, best, fl, stat, bytes;
};
static ResultsLayout results_layout(int nb, size_t L, size_t S, bool score) {
  ResultsLayout r;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t at = off; off += (bytes + 15) & ~(size_t)15; return at; };
  r.coef = take(3 * nb * L * 8);
  r.rf = take(3 * L * 8);
  r.meta = take(score ? L * 8 : 0);
  r.mr = take(score ? L * 8 : 0);
  r.hm = take(score ? L * 8 : 0);
  r.best = take(score ? 4 * S * 8 : 0);
  r.fl = take(score ? L : 0);
  r.stat = take(2 * sizeof(int));
  r.bytes = off;
  return r;
}

int bmpc_plan_host_layout(const bmpc_ctx* ctx, int S, int l, int score, long long* out, int n) {
  if (!ctx || S < 1 || l < 0) return fail(BMPC_EINVAL, "bmpc_plan_host_layout: bad arguments");
  const ResultsLayout r = results_layout(ctx->C.nb, (size_t)S * l, (size_t)S, score != 0);
  const long long v[] = {(long long)r.coef, (long long)r.rf,   (long long)r.meta,
                         (long long)r.mr,   (long long)r.hm,   (long long)r.best,
                         (long long)r.fl,   (long long)r.stat, (long long)r.bytes};
  for (int i = 0; i < n && i < 9; ++i) out[i] = v[i];
  return BMPC_OK;
}

// BMPC_TRACE=1: bmpc_plan_host prints its host / device phase times to stderr
// (tools/e2e_breakdown.py); off by default.
struct PlanTrace {
  bool on = false;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point h[8];
  cudaEvent_t e[8];
  int nh = 0, ne = 0;
  explicit PlanTrace(cudaStream_t s) : st(s) {
    static const bool env = getenv("BMPC_TRACE") != nullptr;
    on = env;
    if (on)
      for (auto& ev : e) cudaEventCreate(&ev);
  }
  void host() { if (on && nh < 8) h[nh++] = std::chrono::steady_clock::now(); }
  void dev() { if (on && ne < 8) cudaEventRecord(e[ne++], st); }
  ~PlanTrace() {
    if (!on) return;
    fprintf(stderr, "[bmpc_trace] host us:");
    for (int i = 1; i < nh; ++i)
      fprintf(stderr, " %.1f", std::chrono::duration<double, std::micro>(h[i] - h[i - 1]).count());
    fprintf(stderr, " | device us:");
    for (int i = 1; i < ne; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[i - 1], e[i]);
      fprintf(stderr, " %.1f", ms * 1e3);
    }
    fprintf(stderr, "\n");
    for (auto& ev : e) cudaEventDestroy(ev);
  }
};

int bmpc_plan_host(bmpc_ctx* ctx, const bmpc_problem* hp, const bmpc_solve_opts* o,
                   bmpc_solve_out* ho, const bmpc_score_spec* spec, bmpc_score_out* hs,
                   void* stream) {
  int rc = check_problem(ctx, hp);
  if (rc) return rc;
  if (!o || !ho) return fail(BMPC_EINVAL, "null opts/out");
  if (is_warm(o)) return fail(BMPC_EINVAL, "bmpc_plan_host: warm starts use the device API");
  cudaStream_t st = S_(stream);
  PlanTrace tr(st);
  tr.host();
  const int n = ctx->C.n, nb = ctx->C.nb;
  const size_t L = (size_t)hp->S * hp->l, mn = (size_t)hp->m * n, S = (size_t)hp->S;
  const bool score = spec && hs;
  // One device arena: inputs, then the results in the order they come back.
  // Results are contiguous so one copy brings them to the pinned staging
  // buffer; every region is a multiple of 8 bytes.
  const size_t hist = (size_t)o->max_iter * 3 * L;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t at = off; off += (bytes + 15) & ~(size_t)15; return at; };
  const size_t o_xix = take(S * mn * 8), o_xiy = take(S * mn * 8), o_bxy = take(12 * L * 8),
               o_bps = take(4 * L * 8), o_hist = take(ho->history ? hist * 8 : 0),
               o_lam = take(3 * nb * L * 8),
               o_v = take(o->want_v && ho->v ? n * L * 8 : 0);
  const size_t o_res0 = off;  // results block
  const ResultsLayout R = results_layout(nb, L, S, score);
  off += R.bytes;
  const size_t o_coef = o_res0 + R.coef, o_rf = o_res0 + R.rf, o_meta = o_res0 + R.meta,
               o_mr = o_res0 + R.mr, o_hm = o_res0 + R.hm, o_best = o_res0 + R.best,
               o_fl = o_res0 + R.fl, o_stat = o_res0 + R.stat;
  const size_t res_bytes = R.bytes;
  // Zero-copy return: when the caller's outputs already sit in one pinned
  // block laid out like the results block (bmpc_plan_host_layout), the block
  // comes back with one copy straight into place -- no staging buffer, no
  // host memcpy.
  char* direct = nullptr;
  if (ho->c_x) {
    char* base = (char*)ho->c_x - R.coef;
    bool ok = (char*)ho->c_y == base + R.coef + nb * L * 8 &&
              (char*)ho->c_psi == base + R.coef + 2 * nb * L * 8 && (char*)ho->res_final == base + R.rf;
    if (ok && score)
      ok = (char*)hs->meta_cost == base + R.meta && (char*)hs->min_ratio == base + R.mr &&
           (char*)hs->heading_max == base + R.hm && (char*)hs->flags == base + R.fl &&
           (char*)hs->best_index == base + R.best && (char*)hs->argmin_all == base + R.best + S * 8 &&
           (char*)hs->argmin_hc == base + R.best + 2 * S * 8 &&
           (char*)hs->n_feasible == base + R.best + 3 * S * 8;
    if (ok) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, base) == cudaSuccess && at.type == cudaMemoryTypeHost)
        direct = base;
      else
        cudaGetLastError();  // clear a sticky "invalid value" from pageable memory
    }
  }
  DevBuf B(ctx, st);
  char* arena = B.alloc<char>(off);
  if (!arena) return fail(BMPC_ECUDA, "device allocation failed");
  double* xix = (double*)(arena + o_xix);
  double* xiy = (double*)(arena + o_xiy);
  double* bxy = (double*)(arena + o_bxy);
  double* bps = (double*)(arena + o_bps);
  tr.host();
  tr.dev();
  // Inputs in page-locked host memory are read in place over the host link
  // (unified addressing: k_pack_xi reads the predictions once, the solve reads
  // each instance's 16 boundary values once at its start), which saves four
  // copy launches on the critical path; pageable inputs are copied in.
  auto pinned = [](const void* ptr, const void** dev) {
    cudaPointerAttributes at;
    if (!ptr || cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return false;
    *dev = at.devicePointer;
    return true;
  };
  const void *dxix = nullptr, *dxiy = nullptr, *dbxy = nullptr, *dbps = nullptr;
  const bool in_place = getenv("BMPC_NO_ZERO_COPY_IN") == nullptr && pinned(hp->b_xy, &dbxy) &&
                        pinned(hp->b_psi, &dbps) &&
                        (S * mn == 0 || (pinned(hp->xi_x, &dxix) && pinned(hp->xi_y, &dxiy)));
  bmpc_problem dp = *hp;
  if (in_place) {
    dp.xi_x = (const double*)dxix;
    dp.xi_y = (const double*)dxiy;
    dp.b_xy = (const double*)dbxy;
    dp.b_psi = (const double*)dbps;
  } else {
    CK(cudaMemcpyAsync(xix, hp->xi_x, S * mn * 8, cudaMemcpyHostToDevice, st), "h2d");
    CK(cudaMemcpyAsync(xiy, hp->xi_y, S * mn * 8, cudaMemcpyHostToDevice, st), "h2d");
    CK(cudaMemcpyAsync(bxy, hp->b_xy, 12 * L * 8, cudaMemcpyHostToDevice, st), "h2d");
    CK(cudaMemcpyAsync(bps, hp->b_psi, 4 * L * 8, cudaMemcpyHostToDevice, st), "h2d");
    dp.xi_x = xix;
    dp.xi_y = xiy;
    dp.b_xy = bxy;
    dp.b_psi = bps;
  }
  tr.host();
  tr.dev();
  bmpc_solve_out dout;
  memset(&dout, 0, sizeof(dout));
  double* coef = (double*)(arena + o_coef);
  double* lam = (double*)(arena + o_lam);
  dout.c_x = coef;
  dout.c_y = coef + nb * L;
  dout.c_psi = coef + 2 * nb * L;
  dout.l_x = lam;
  dout.l_y = lam + nb * L;
  dout.l_psi = lam + 2 * nb * L;
  dout.history = ho->history ? (double*)(arena + o_hist) : nullptr;  // written only on request
  dout.res_final = (double*)(arena + o_rf);
  dout.v = (o->want_v && ho->v) ? (double*)(arena + o_v) : nullptr;
  // no synchronisation inside the solve: its {iterations, converged} come back
  // with the results block
  bmpc_solve_opts o2 = *o;
  o2.status_dev = (int*)(arena + o_stat);
  o = &o2;
  bmpc_score_out ds;
  memset(&ds, 0, sizeof(ds));
  if (score) {  // solve with the fused scoring epilogue, then the per-scene argmin
    ds.meta_cost = (double*)(arena + o_meta);
    ds.min_ratio = (double*)(arena + o_mr);
    ds.heading_max = (double*)(arena + o_hm);
    ds.flags = (unsigned char*)(arena + o_fl);
    long long* idx = (long long*)(arena + o_best);
    ds.best_index = idx;
    ds.argmin_all = idx + S;
    ds.argmin_hc = idx + 2 * S;
    ds.n_feasible = idx + 3 * S;
    rc = bmpc_plan(ctx, &dp, o, &dout, spec, &ds, stream);
  } else {
    rc = bmpc_solve(ctx, &dp, o, &dout, stream);
  }
  if (rc) return rc;
  tr.host();
  tr.dev();
  // rarely requested extras straight to the caller's memory
  struct Cp { void* h; const void* d; size_t bytes; };
  const Cp extra[] = {
      {ho->l_x, dout.l_x, nb * L * 8}, {ho->l_y, dout.l_y, nb * L * 8},
      {ho->l_psi, dout.l_psi, nb * L * 8}, {ho->v, dout.v, n * L * 8},
      {ho->history, dout.history, (size_t)o->max_iter * 3 * L * 8},  // rows past iterations: stale
  };
  for (const Cp& c : extra)
    if (c.h && c.d && c.bytes) CK(cudaMemcpyAsync(c.h, c.d, c.bytes, cudaMemcpyDeviceToHost, st), "d2h");
  if (direct) {
    CK(cudaMemcpyAsync(direct, arena + o_res0, res_bytes, cudaMemcpyDeviceToHost, st), "d2h");
    tr.dev();
    tr.host();
    CK(cudaStreamSynchronize(st), "sync");
    tr.host();
    const int* stat = (const int*)(direct + R.stat);
    ho->iterations = stat[0];
    ho->converged = stat[1];
    return BMPC_OK;
  }
  // the results block in one copy through the pinned staging buffer
  std::lock_guard<std::mutex> lk(ctx->stage_mu);
  if (ctx->stage_bytes < res_bytes) {
    if (ctx->stage) cudaFreeHost(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    CK(cudaHostAlloc(&ctx->stage, res_bytes, cudaHostAllocDefault), "pinned staging");
    ctx->stage_bytes = res_bytes;
  }
  CK(cudaMemcpyAsync(ctx->stage, arena + o_res0, res_bytes, cudaMemcpyDeviceToHost, st), "d2h");
  CK(cudaStreamSynchronize(st), "sync");
  const char* hb = (const char*)ctx->stage - o_res0;  // arena offset -> staging
  const int* stat = (const int*)(hb + o_stat);
  ho->iterations = stat[0];
  ho->converged = stat[1];
  const Cp res[] = {
      {ho->c_x, hb + o_coef, nb * L * 8}, {ho->c_y, hb + o_coef + nb * L * 8, nb * L * 8},
      {ho->c_psi, hb + o_coef + 2 * nb * L * 8, nb * L * 8}, {ho->res_final, hb + o_rf, 3 * L * 8},
      {score ? hs->meta_cost : nullptr, hb + o_meta, L * 8},
      {score ? hs->min_ratio : nullptr, hb + o_mr, L * 8},
      {score ? hs->heading_max : nullptr, hb + o_hm, L * 8},
      {score ? hs->flags : nullptr, hb + o_fl, L},
      {score ? hs->best_index : nullptr, hb + o_best, S * 8},
      {score ? hs->argmin_all : nullptr, hb + o_best + S * 8, S * 8},
      {score ? hs->argmin_hc : nullptr, hb + o_best + 2 * S * 8, S * 8},
      {score ? hs->n_feasible : nullptr, hb + o_best + 3 * S * 8, S * 8},
  };
  for (const Cp& c : res)
    if (c.h && c.bytes) memcpy(c.h, c.d, c.bytes);
  return BMPC_OK;
}

// ------------------------------------------------------------ op-level ----
int bmpc_op_obstacle_update(int n, int l, int mn, const double* x, const double* y,
                            const double* xi_x, const double* xi_y, double a, double b,
                            double* alpha, double* d, void* s) {
  if (n < 1 || l < 0 || mn < 0 || mn % n) return fail(BMPC_EINVAL, "obstacle_update: bad shape");
  CK(bmpc::op_obstacle_update(n, l, mn, x, y, xi_x, xi_y, a, b, alpha, d, S_(s)), "obstacle_update");
  return BMPC_OK;
}
int bmpc_op_accel_update(int n, int l, const double* xdd, const double* ydd, double a_max,
                         double* alpha_a, double* d_a, void* s) {
  CK(bmpc::op_accel_update((long long)n * l, xdd, ydd, a_max, alpha_a, d_a, S_(s)), "accel_update");
  return BMPC_OK;
}
int bmpc_op_v_update(int n, int l, const double* xd, const double* yd, double v_min, double v_max,
                     double* v, void* s) {
  CK(bmpc::op_v_update((long long)n * l, xd, yd, v_min, v_max, v, S_(s)), "v_update");
  return BMPC_OK;
}
int bmpc_op_assemble_g(int n, int l, int mn, const double* xi_x, const double* xi_y,
                       const double* alpha, const double* d, const double* alpha_a,
                       const double* d_a, const double* v, const double* psi, double a, double b,
                       double* g_x, double* g_y, void* s) {
  CK(bmpc::op_assemble_g(n, l, mn, xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi, a, b, g_x, g_y, S_(s)),
     "assemble_g");
  return BMPC_OK;
}
int bmpc_op_residual_vectors(int n, int l, int mn, const double* x, const double* y,
                             const double* xd, const double* yd, const double* xdd,
                             const double* ydd, const double* psi, const double* xi_x,
                             const double* xi_y, const double* alpha, const double* d,
                             const double* alpha_a, const double* d_a, const double* v, double a,
                             double b, double* r_x, double* r_y, void* s) {
  CK(bmpc::op_residual_vectors(n, l, mn, x, y, xd, yd, xdd, ydd, psi, xi_x, xi_y, alpha, d, alpha_a,
                               d_a, v, a, b, r_x, r_y, S_(s)),
     "residual_vectors");
  return BMPC_OK;
}
int bmpc_op_tail(int n, int l, int mn, const double* x, const double* y, const double* xd,
                 const double* yd, const double* xdd, const double* ydd, const double* psi,
                 const double* xi_x, const double* xi_y, double v_min, double v_max, double a_max,
                 double a, double b, double* alpha, double* d, double* alpha_a, double* d_a,
                 double* v, double* r_x, double* r_y, double* g_x, double* g_y, double* sq_obs,
                 double* sq_acc, double* sq_nonhol, void* s) {
  const bool with_angles = alpha != nullptr && alpha_a != nullptr;
  if (!with_angles && (!sq_obs || !sq_acc || !sq_nonhol))
    return fail(BMPC_EINVAL, "tail_core needs the squared-sum outputs");
  CK(bmpc::op_tail(with_angles, n, l, mn, x, y, xd, yd, xdd, ydd, psi, xi_x, xi_y, v_min, v_max, a_max,
                   a, b, alpha, d, alpha_a, d_a, v, r_x, r_y, g_x, g_y, sq_obs, sq_acc, sq_nonhol, S_(s)),
     "tail");
  return BMPC_OK;
}

int bmpc_math_check(int fn, long long n, const double* a, const double* b, double* out,
                    double* out2, void* s) {
  if (fn < 0 || fn > 7 || !a || !out || (fn == 3 || fn == 4 || fn == 7) && !out2)
    return fail(BMPC_EINVAL, "bmpc_math_check: bad argument");
  CK(bmpc::op_math_check(fn, n, a, b, out, out2, S_(s)), "math_check");
  return BMPC_OK;
}

int bmpc_dfma_peak(int reps, double* tflops, void* s) {
  if (!tflops) return fail(BMPC_EINVAL, "null output");
  CK(bmpc::dfma_peak_tflops(reps < 1 ? 1 : reps, tflops, S_(s)), "dfma_peak");
  return BMPC_OK;
}

int bmpc_latency_probe(int which, double* cycles_per_op, void* s) {
  if (!cycles_per_op || which < 0 || which > 7) return fail(BMPC_EINVAL, "latency_probe: bad argument");
  CK(bmpc::latency_probe(which, cycles_per_op, S_(s)), "latency_probe");
  return BMPC_OK;
}

// ------------------------------------------------------- step-wise API ----
int bmpc_project(bmpc_ctx* ctx, int mode, int m, int L, const double* g, double* out, void* s) {
  if (!ctx || (mode != 0 && mode != 1) || m < 0 || L < 0 || !g || !out)
    return fail(BMPC_EINVAL, "bmpc_project: bad argument");
  CK(bmpc::op_project(ctx->C, mode, m, L, g, out, S_(s)), "project");
  return BMPC_OK;
}
int bmpc_kkt_apply(bmpc_ctx* ctx, int which, int L, const double* rhs, double* out_a,
                   double* out_b, void* s) {
  if (!ctx || (which != 0 && which != 1) || L < 0 || !rhs || !out_a || (which == 0 && !out_b))
    return fail(BMPC_EINVAL, "bmpc_kkt_apply: bad argument");
  CK(bmpc::op_kkt_apply(ctx->C, which, L, rhs, out_a, out_b, S_(s)), "kkt_apply");
  return BMPC_OK;
}
int bmpc_heading(bmpc_ctx* ctx, int L, const double* c_x, const double* c_y, double* theta, void* s) {
  if (!ctx || L < 0 || !c_x || !c_y || !theta) return fail(BMPC_EINVAL, "bmpc_heading: bad argument");
  CK(bmpc::op_heading(ctx->C, L, c_x, c_y, theta, S_(s)), "heading");
  return BMPC_OK;
}
int bmpc_op_d_obs(int n, int l, int mn, const double* x, const double* y, const double* xi_x,
                  const double* xi_y, const double* alpha, double a, double b, double* d, void* s) {
  if (n < 1 || l < 0 || mn < 0 || mn % n) return fail(BMPC_EINVAL, "d_obs: bad shape");
  CK(bmpc::op_d_obs(n, l, mn, x, y, xi_x, xi_y, alpha, a, b, d, S_(s)), "d_obs");
  return BMPC_OK;
}
int bmpc_op_collision_ratios(int n, int l, int mn, const double* x, const double* y,
                             const double* xi_x, const double* xi_y, double a, double b, double* out,
                             void* s) {
  if (n < 1 || l < 0 || mn < 0 || mn % n) return fail(BMPC_EINVAL, "collision_ratios: bad shape");
  if ((long long)mn * l > 0 && (!x || !y || !xi_x || !xi_y || !out))
    return fail(BMPC_EINVAL, "collision_ratios: null pointer");
  CK(bmpc::op_collision_ratios(n, l, mn, x, y, xi_x, xi_y, a, b, out, S_(s)), "collision_ratios");
  return BMPC_OK;
}
int bmpc_block_norms(int n, int l, int mn, const double* r_x, const double* r_y, double* out,
                     void* s) {
  CK(bmpc::op_block_norms(n, l, mn, r_x, r_y, out, S_(s)), "block_norms");
  return BMPC_OK;
}

}  // extern "C"
