// am_solve.cu -- host-side dispatch of the persistent AM kernel over n_b.
// The kernel itself lives in am_solve_kernel.cuh; each n_b is instantiated by a
// separate compile of am_inst.cu.
#include <cuda_runtime.h>

#include "am_args.h"

namespace bmpc {

size_t am_solve_smem_bytes(int nb, int npad, int kxs, int kps, int warps, int team, bool f32) {
  // the constant image (am_args.h; the fp32 mode holds its basis in fp32) and
  // the per-team scratch
  (void)kxs;
  (void)kps;
  static_assert(bmpc_f32_sample_doubles(64) <= 5 * 64 && bmpc_f32_sample_doubles(128) <= 5 * 128 &&
                    bmpc_f32_sample_doubles(224) <= 3 * 224 && bmpc_f32_sample_doubles(256) <= 3 * 256,
                "fp32 sample arrays must fit the fp64 region");
  return sizeof(double) * (bmpc_const_image_doubles(nb, npad) - bmpc_basis_doubles(nb, npad, false) +
                           bmpc_basis_doubles(nb, npad, f32) +
                           (size_t)(warps / team) * bmpc_team_doubles(npad, team)) +
         ((f32 && team == 1) ? bmpc_skip_bytes(npad, warps) : 0);  // fp32 mode: clearance arrays
}

#define BMPC_DECL(NB)                                                                      \
  cudaError_t launch_am_nb_##NB(const bmpc_dev_consts& C, const bmpc_solve_args& A, int w, \
                                cudaStream_t st);
BMPC_DECL(4) BMPC_DECL(5) BMPC_DECL(6) BMPC_DECL(7) BMPC_DECL(8) BMPC_DECL(9) BMPC_DECL(10)
BMPC_DECL(11) BMPC_DECL(12) BMPC_DECL(13) BMPC_DECL(14) BMPC_DECL(15) BMPC_DECL(16)

cudaError_t launch_am_solve(const bmpc_dev_consts& C, const bmpc_solve_args& A, int warps,
                            cudaStream_t st) {
  switch (C.nb) {
    case 4: return launch_am_nb_4(C, A, warps, st);
    case 5: return launch_am_nb_5(C, A, warps, st);
    case 6: return launch_am_nb_6(C, A, warps, st);
    case 7: return launch_am_nb_7(C, A, warps, st);
    case 8: return launch_am_nb_8(C, A, warps, st);
    case 9: return launch_am_nb_9(C, A, warps, st);
    case 10: return launch_am_nb_10(C, A, warps, st);
    case 11: return launch_am_nb_11(C, A, warps, st);
    case 12: return launch_am_nb_12(C, A, warps, st);
    case 13: return launch_am_nb_13(C, A, warps, st);
    case 14: return launch_am_nb_14(C, A, warps, st);
    case 15: return launch_am_nb_15(C, A, warps, st);
    case 16: return launch_am_nb_16(C, A, warps, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bmpc
