// am_inst.cu -- one n_b instantiation of the persistent AM kernel (compiled
// once per n_b with -DBMPC_INST_NB=<n_b> so the builds run in parallel).
#include <atomic>

#include "am_solve_kernel.cuh"

namespace bmpc {

size_t am_solve_smem_bytes(int nb, int npad, int kxs, int kps, int warps, int team, bool f32);

template <int NB, int NKM, bool F32, bool TEAMS = false, bool XS = false, bool CULL = false>
static cudaError_t launch_t(const bmpc_dev_consts& C, const bmpc_solve_args& A, int warps,
                            cudaStream_t st, size_t xs_bytes = 0) {
  const size_t smem = am_solve_smem_bytes(NB, C.npad, C.kxs, C.kps, warps, A.team, F32) + xs_bytes;
  auto kfn = am_solve_kernel<NB, NKM, F32, TEAMS, XS, CULL>;
  // raise the dynamic shared-memory limit once per device and size (a driver
  // call per launch costs microseconds of host time on the critical path)
  static std::atomic<int> granted[16];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& g = granted[dev & 15];
  if ((int)smem > g.load(std::memory_order_relaxed)) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int cur = g.load();
    while ((int)smem > cur && !g.compare_exchange_weak(cur, (int)smem)) {
    }
  }
  const int ipb = warps / A.team;  // instances per block
  const int grid = (A.L + ipb - 1) / ipb;
  if (A.skipg) {
    // The global clearance scratch is indexed by SM id and warp: valid only
    // while an SM holds one block of this launch.  Two blocks fit when their
    // shared memory (+1 KB reserved each) does: then no scratch, no skipping.
    int per_sm = 0;
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (2 * (smem + 1024) <= (size_t)per_sm) {
      bmpc_solve_args A2 = A;
      A2.skipg = nullptr;
      kfn<<<grid, warps * 32, smem, st>>>(C, A2);
      return cudaGetLastError();
    }
  }
  kfn<<<grid, warps * 32, smem, st>>>(C, A);
  return cudaGetLastError();
}

// Bytes of staged predictions for one block (0: stage none).
static size_t xs_stage_bytes(const bmpc_dev_consts& C, const bmpc_solve_args& A, int warps) {
#ifdef BMPC_NO_XI_STAGE
  return 0;
#endif
  if (A.team != 1 || C.npad > 128 || A.m <= 0 || !A.xis || (BMPC_XS32 && !A.xs32) || A.l < warps) return 0;
  const int scenes = (A.S > 1 && A.l % warps != 0) ? 2 : 1;
  // + the clearance-skipping arrays behind them (BMPC_SKIP: 12 bytes per sample and warp)
  const size_t xs = (size_t)scenes * A.m * C.n * (BMPC_XS32 ? 8 : 16) +
                    ((!BMPC_XS32 && bmpc_stores_xy(C.npad)) ? bmpc_skip_bytes(C.npad, warps) : 0);
  static int optin[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!optin[dev & 15]) cudaDeviceGetAttribute(&optin[dev & 15], cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t base = am_solve_smem_bytes(C.nb, C.npad, C.kxs, C.kps, warps, 1, false);
  return base + xs <= (size_t)optin[dev & 15] ? xs : 0;
}

#define BMPC_CAT2(a, b) a##b
#define BMPC_CAT(a, b) BMPC_CAT2(a, b)

cudaError_t BMPC_CAT(launch_am_nb_, BMPC_INST_NB)(const bmpc_dev_consts& C,
                                                   const bmpc_solve_args& A, int warps,
                                                   cudaStream_t st) {
  const bool f32 = (A.flags & BMPC_F_F32) != 0;
  // teams: the small-batch latency mode, fp64, n <= 128; also every polling
  // (tol > 0) solve of that shape, with teams of one warp if none was asked for
  if (A.team > 1 || (A.flags & BMPC_F_TEAM_BUILD)) {
    if (f32) return cudaErrorNotSupported;
    switch (C.npad) {
      case 64: return launch_t<BMPC_INST_NB, 2, false, true>(C, A, warps, st);
      case 128: return launch_t<BMPC_INST_NB, 4, false, true>(C, A, warps, st);
      default: return cudaErrorNotSupported;
    }
  }
  // Obstacle predictions staged in shared memory (bulk copies with the
  // constants) when the scene(s) of a block fit next to the scratch: n <= 128,
  // fp64; a block spans at most two scenes when l >= its instance count.
  const size_t xs = xs_stage_bytes(C, A, warps);
  // obstacle culling by bounding boxes (host decides: A.boxes set for many
  // obstacles, where it pays): a separate instantiation of every throughput kernel
  const bool cull = A.boxes != nullptr;
  if (!f32 && xs > 0) {
    switch (C.npad) {
      case 64: return cull ? launch_t<BMPC_INST_NB, 2, false, false, true, true>(C, A, warps, st, xs)
                           : launch_t<BMPC_INST_NB, 2, false, false, true>(C, A, warps, st, xs);
      case 128: return cull ? launch_t<BMPC_INST_NB, 4, false, false, true, true>(C, A, warps, st, xs)
                            : launch_t<BMPC_INST_NB, 4, false, false, true>(C, A, warps, st, xs);
      default: break;
    }
  }
#define BMPC_LAUNCH(NK)                                                                            \
  (f32 ? (cull ? launch_t<BMPC_INST_NB, NK, true, false, false, true>(C, A, warps, st)              \
               : launch_t<BMPC_INST_NB, NK, true>(C, A, warps, st))                                \
       : (cull ? launch_t<BMPC_INST_NB, NK, false, false, false, true>(C, A, warps, st)             \
               : launch_t<BMPC_INST_NB, NK, false>(C, A, warps, st)))
  switch (C.npad) {  // the host pads n to 64, 128, 224 or 256 samples
    case 64: return BMPC_LAUNCH(2);
    case 128: return BMPC_LAUNCH(4);
    case 224: return BMPC_LAUNCH(7);
    case 256: return BMPC_LAUNCH(8);
    default: return cudaErrorInvalidValue;
  }
#undef BMPC_LAUNCH
}

#ifdef BMPC_PHASE_PROF
// read (and optionally clear) this unit's phase counters
extern "C" int BMPC_CAT(bmpc_phase_prof_nb, BMPC_INST_NB)(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles)) != cudaSuccess) return 2;
  if (reset) {
    static const unsigned long long z[20] = {};
    if (cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)) != cudaSuccess) return 2;
  }
  return 0;
}
#endif

}  // namespace bmpc
