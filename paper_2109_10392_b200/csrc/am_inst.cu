// am_inst.cu -- one n_b instantiation of the persistent AM kernel (compiled
// once per n_b with -DBMPC_INST_NB=<n_b> so the builds run in parallel).
#include <atomic>

#include "am_solve_kernel.cuh"

namespace bmpc {

size_t am_solve_smem_bytes(int nb, int npad, int kxs, int kps, int warps, int team);

template <int NB, int NKM, bool F32, bool TEAMS = false>
static cudaError_t launch_t(const bmpc_dev_consts& C, const bmpc_solve_args& A, int warps,
                            cudaStream_t st) {
  const size_t smem = am_solve_smem_bytes(NB, C.npad, C.kxs, C.kps, warps, A.team);
  auto kfn = am_solve_kernel<NB, NKM, F32, TEAMS>;
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
  kfn<<<grid, warps * 32, smem, st>>>(C, A);
  return cudaGetLastError();
}

#define BMPC_CAT2(a, b) a##b
#define BMPC_CAT(a, b) BMPC_CAT2(a, b)

cudaError_t BMPC_CAT(launch_am_nb_, BMPC_INST_NB)(const bmpc_dev_consts& C,
                                                   const bmpc_solve_args& A, int warps,
                                                   cudaStream_t st) {
  const bool f32 = (A.flags & BMPC_F_F32) != 0;
  if (A.team > 1) {  // teams: the small-batch latency mode, fp64, n <= 128
    if (f32) return cudaErrorNotSupported;
    switch (C.npad) {
      case 64: return launch_t<BMPC_INST_NB, 2, false, true>(C, A, warps, st);
      case 128: return launch_t<BMPC_INST_NB, 4, false, true>(C, A, warps, st);
      default: return cudaErrorNotSupported;
    }
  }
  switch (C.npad) {  // the host pads n to 64, 128, 224 or 256 samples
    case 64: return f32 ? launch_t<BMPC_INST_NB, 2, true>(C, A, warps, st)
                                 : launch_t<BMPC_INST_NB, 2, false>(C, A, warps, st);
    case 128: return f32 ? launch_t<BMPC_INST_NB, 4, true>(C, A, warps, st)
                                 : launch_t<BMPC_INST_NB, 4, false>(C, A, warps, st);
    case 224: return f32 ? launch_t<BMPC_INST_NB, 7, true>(C, A, warps, st)
                                 : launch_t<BMPC_INST_NB, 7, false>(C, A, warps, st);
    case 256: return f32 ? launch_t<BMPC_INST_NB, 8, true>(C, A, warps, st)
                                 : launch_t<BMPC_INST_NB, 8, false>(C, A, warps, st);
    default: return cudaErrorInvalidValue;
  }
}

#ifdef BMPC_PHASE_PROF
// read (and optionally clear) this unit's phase counters
extern "C" int BMPC_CAT(bmpc_phase_prof_nb, BMPC_INST_NB)(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles)) != cudaSuccess) return 2;
  if (reset) {
    static const unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)) != cudaSuccess) return 2;
  }
  return 0;
}
#endif

}  // namespace bmpc
