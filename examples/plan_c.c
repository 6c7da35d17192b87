/* Plain-C caller of the B200 solver ABI (include/batchmpc_b200.h): what a
 * C/C++ host integrating the path would write.  Reads one problem dumped by
 * tests/test_gpu_c_abi.py (constants + one scene), runs bmpc_plan_host from
 * host buffers, and prints the best index, sweep count and an FNV-1a hash of
 * the coefficient bytes.
 *
 *   gcc -O2 examples/plan_c.c -Iinclude -Lpaper_2109_10392_b200/_lib \
 *       -lbatchmpc_b200 -Wl,-rpath,$PWD/paper_2109_10392_b200/_lib -o plan_c
 *   ./plan_c problem.bin
 */
#include <stdio.h>
#include <stdlib.h>

#include "batchmpc_b200.h"

static double* read_doubles(FILE* f, long count) {
  double* p = (double*)malloc((size_t)count * sizeof(double));
  if (!p || fread(p, sizeof(double), (size_t)count, f) != (size_t)count) {
    fprintf(stderr, "short read\n");
    exit(2);
  }
  return p;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s problem.bin\n", argv[0]);
    return 2;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) {
    perror("open");
    return 2;
  }
  /* header: n, nb, m, l, max_iter as doubles; then rho, a, b, v_min, v_max, a_max */
  double* hd = read_doubles(f, 11);
  const int n = (int)hd[0], nb = (int)hd[1], m = (int)hd[2], l = (int)hd[3], iters = (int)hd[4];
  const int rx = nb + 6, rp = nb + 4;
  double* P = read_doubles(f, (long)n * nb);
  double* Pd = read_doubles(f, (long)n * nb);
  double* Pdd = read_doubles(f, (long)n * nb);
  double* tau = read_doubles(f, n);
  double* kinv_axis = read_doubles(f, (long)rx * rx);
  double* k_axis = read_doubles(f, (long)rx * rx);
  double* kinv_psi = read_doubles(f, (long)rp * rp);
  double* k_psi = read_doubles(f, (long)rp * rp);
  double* ftf = read_doubles(f, (long)nb * nb);
  double* xi_x = read_doubles(f, (long)m * n);
  double* xi_y = read_doubles(f, (long)m * n);
  double* b_xy = read_doubles(f, 12L * l);
  double* b_psi = read_doubles(f, 4L * l);
  fclose(f);

  bmpc_ctx* ctx = NULL;
  if (bmpc_ctx_create(n, nb, hd[5], P, Pd, Pdd, tau, kinv_axis, k_axis, kinv_psi, k_psi, ftf, &ctx)) {
    fprintf(stderr, "ctx: %s\n", bmpc_last_error());
    return 1;
  }
  bmpc_problem prob = {m, l, 1, xi_x, xi_y, b_xy, b_psi, hd[6], hd[7], hd[8], hd[9], hd[10]};
  bmpc_solve_opts opts = {0};
  opts.max_iter = iters;
  opts.tol = 0.0;
  double* coef = (double*)calloc(3 * (size_t)nb * l, sizeof(double));
  double* res = (double*)calloc(3 * (size_t)l, sizeof(double));
  bmpc_solve_out out = {0};
  out.c_x = coef;
  out.c_y = coef + (size_t)nb * l;
  out.c_psi = coef + 2 * (size_t)nb * l;
  out.res_final = res;
  /* cruise meta cost at 20 m/s, the planner's default filter limits */
  bmpc_score_spec spec = {0, 20.0, 20.0, 0.0, 1.0, 1.0, 0.2268928027592628, 1e-3, 0.01};
  double* meta = (double*)calloc(3 * (size_t)l, sizeof(double));
  unsigned char* flags = (unsigned char*)calloc((size_t)l, 1);
  long long idx[4] = {0, 0, 0, 0};
  bmpc_score_out sc = {meta, meta + l, meta + 2 * l, flags, idx, idx + 1, idx + 2, idx + 3};
  if (bmpc_plan_host(ctx, &prob, &opts, &out, &spec, &sc, NULL)) {
    fprintf(stderr, "plan: %s\n", bmpc_last_error());
    return 1;
  }
  /* FNV-1a over the coefficient bytes (c_x, c_y, c_psi, each (nb, l) row-major) */
  unsigned long long h = 1469598103934665603ull;
  const unsigned char* by = (const unsigned char*)coef;
  for (size_t i = 0; i < 3 * (size_t)nb * l * sizeof(double); ++i) {
    h ^= by[i];
    h *= 1099511628211ull;
  }
  printf("best_index %lld argmin_all %lld n_feasible %lld iterations %d fnv %llu\n", idx[0], idx[1],
         idx[3], out.iterations, h);
  bmpc_ctx_destroy(ctx);
  return 0;
}
