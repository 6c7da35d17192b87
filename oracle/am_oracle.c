/*
 * am_oracle.c -- CPU ORACLE (test infrastructure only; never on the product path).
 *
 * Plain-C restatement of the reference's compiled per-iteration kernels, used
 * as the checker for the CUDA path and as the CPU baseline ("port") timed by
 * bench.py.  Each routine follows the scalar loop of the reference's Cython
 * kernel (file:line relative to /root/reference/pkg/src/batchmpc/kernels/):
 *
 *   oracle_obstacle_update  <- _speedups.pyx:12-39   (numpy twin _numpy.py:11-22)
 *   oracle_accel_update     <- _speedups.pyx:42-60   (_numpy.py:25-29)
 *   oracle_v_update         <- _speedups.pyx:63-78   (_numpy.py:32-34)
 *   oracle_assemble_g       <- _speedups.pyx:81-111  (_numpy.py:37-49)
 *   oracle_tail_core        <- _speedups.pyx:114-218 (_numpy.py:69-131)
 *
 * Layout is the reference's: sampled arrays (n, l) row-major with the instance
 * (column) index fastest; obstacle-stacked arrays (m*n, l) with row j*n + k for
 * obstacle j at sample k.  The evaluation order of every expression matches
 * the reference ((a * d) * ca, etc.) and the file is compiled with plain -O3
 * (no FMA contraction on x86-64 baseline), so results are expected to be
 * bitwise identical to the reference's compiled backend -- the tests pin that.
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

typedef ptrdiff_t idx_t;

void oracle_obstacle_update(idx_t n, idx_t l, idx_t mn,
                            const double *x, const double *y,
                            const double *xi_x, const double *xi_y,
                            double a, double b, double *alpha, double *d)
{
    for (idx_t row = 0; row < mn; ++row) {
        idx_t k = row % n;
        for (idx_t c = 0; c < l; ++c) {
            double wx = x[k * l + c] - xi_x[row];
            double wy = y[k * l + c] - xi_y[row];
            double al = atan2(a * wy, b * wx);
            double ca = cos(al), sa = sin(al);
            double num = a * ca * wx + b * sa * wy;
            double den = (a * ca) * (a * ca) + (b * sa) * (b * sa);
            double dd = num / den;
            if (dd < 1.0) dd = 1.0;
            alpha[row * l + c] = al;
            d[row * l + c] = dd;
        }
    }
}

void oracle_accel_update(idx_t n, idx_t l, const double *xddot, const double *yddot,
                         double a_max, double *alpha_a, double *d_a)
{
    for (idx_t i = 0; i < n * l; ++i) {
        double ax = xddot[i], ay = yddot[i];
        alpha_a[i] = atan2(ay, ax);
        double mag = sqrt(ax * ax + ay * ay);
        if (mag > a_max) mag = a_max;
        d_a[i] = mag;
    }
}

void oracle_v_update(idx_t n, idx_t l, const double *xdot, const double *ydot,
                     double v_min, double v_max, double *v)
{
    for (idx_t i = 0; i < n * l; ++i) {
        double s = sqrt(xdot[i] * xdot[i] + ydot[i] * ydot[i]);
        if (s < v_min) s = v_min;
        else if (s > v_max) s = v_max;
        v[i] = s;
    }
}

void oracle_assemble_g(idx_t n, idx_t l, idx_t mn,
                       const double *xi_x, const double *xi_y,
                       const double *alpha, const double *d,
                       const double *alpha_a, const double *d_a,
                       const double *v, const double *psi,
                       double a, double b, double *g_x, double *g_y)
{
    for (idx_t row = 0; row < mn; ++row)
        for (idx_t c = 0; c < l; ++c) {
            double ang = alpha[row * l + c], ad = d[row * l + c];
            g_x[row * l + c] = xi_x[row] + a * ad * cos(ang);
            g_y[row * l + c] = xi_y[row] + b * ad * sin(ang);
        }
    for (idx_t k = 0; k < n; ++k)
        for (idx_t c = 0; c < l; ++c) {
            double ang = alpha_a[k * l + c], ad = d_a[k * l + c];
            g_x[(mn + k) * l + c] = ad * cos(ang);
            g_y[(mn + k) * l + c] = ad * sin(ang);
            ang = psi[k * l + c];
            ad = v[k * l + c];
            g_x[(mn + n + k) * l + c] = ad * cos(ang);
            g_y[(mn + n + k) * l + c] = ad * sin(ang);
        }
}

/* Fused closed forms + residual vectors + next targets + squared block sums.
 * sq_* must be zero-initialised by the caller (the reference starts them at 0). */
void oracle_tail_core(idx_t n, idx_t l, idx_t mn,
                      const double *x, const double *y,
                      const double *xdot, const double *ydot,
                      const double *xddot, const double *yddot,
                      const double *psi,
                      const double *xi_x, const double *xi_y,
                      double v_min, double v_max, double a_max, double a, double b,
                      double *d, double *d_a, double *v,
                      double *r_x, double *r_y, double *g_x, double *g_y,
                      double *sq_obs, double *sq_acc, double *sq_nonhol)
{
    for (idx_t row = 0; row < mn; ++row) {
        idx_t k = row % n;
        for (idx_t c = 0; c < l; ++c) {
            double wx = x[k * l + c] - xi_x[row];
            double wy = y[k * l + c] - xi_y[row];
            double px = b * wx, py = a * wy;
            double r = sqrt(px * px + py * py);
            double ca, sa;
            if (r > 0.0) { ca = px / r; sa = py / r; }
            else { ca = 1.0; sa = 0.0; }
            double dd = r / (a * b);
            if (dd < 1.0) dd = 1.0;
            d[row * l + c] = dd;
            double adca = a * dd * ca, bdsa = b * dd * sa;
            double rx = wx - adca, ry = wy - bdsa;
            r_x[row * l + c] = rx;
            r_y[row * l + c] = ry;
            sq_obs[c] += rx * rx + ry * ry;
            g_x[row * l + c] = xi_x[row] + adca;
            g_y[row * l + c] = xi_y[row] + bdsa;
        }
    }
    for (idx_t k = 0; k < n; ++k) {
        for (idx_t c = 0; c < l; ++c) {
            idx_t i = k * l + c;
            double ax = xddot[i], ay = yddot[i];
            double mag = sqrt(ax * ax + ay * ay);
            double caa, saa;
            if (mag > 0.0) { caa = ax / mag; saa = ay / mag; }
            else { caa = 1.0; saa = 0.0; }
            double dd = mag < a_max ? mag : a_max;
            d_a[i] = dd;
            double daca = dd * caa, dasa = dd * saa;
            double rx = ax - daca, ry = ay - dasa;
            r_x[(mn + k) * l + c] = rx;
            r_y[(mn + k) * l + c] = ry;
            sq_acc[c] += rx * rx + ry * ry;
            g_x[(mn + k) * l + c] = daca;
            g_y[(mn + k) * l + c] = dasa;

            double s = sqrt(xdot[i] * xdot[i] + ydot[i] * ydot[i]);
            if (s < v_min) s = v_min;
            else if (s > v_max) s = v_max;
            v[i] = s;
            double cp = cos(psi[i]), sp = sin(psi[i]);
            double vcp = s * cp, vsp = s * sp;
            rx = xdot[i] - vcp;
            ry = ydot[i] - vsp;
            r_x[(mn + n + k) * l + c] = rx;
            r_y[(mn + n + k) * l + c] = ry;
            sq_nonhol[c] += rx * rx + ry * ry;
            g_x[(mn + n + k) * l + c] = vcp;
            g_y[(mn + n + k) * l + c] = vsp;
        }
    }
}
