/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference RHS hot path.
 * See oracle.h for the usage rule and pinning status.  Every function cites
 * the reference file:line (paths relative to /root/reference/proj) it
 * restates.  Compiled with -ffp-contract=off so sums are evaluated exactly in
 * the written order (the reference's own summation order). */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ M */
/* Affine entries c + p*m47 + q*m48 of rows 1..s (PAPER.md:263-300 for order
 * 8, PAPER.md:320-345 for order 6, same layout as core/src/stencil.cpp:19-73). */
typedef struct {
  double c, p, q;
} affine_t;

static const affine_t T8[4][8] = {
    {{5.0 / 336, 0, 1}, {-83.0 / 3600, -1.0 / 5, -14.0 / 5}, {299.0 / 50400, 2.0 / 5, 13.0 / 5},
     {17.0 / 12600, -1.0 / 5, -4.0 / 5}, {1.0 / 1120, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{-11.0 / 560, 0, -2}, {-31.0 / 360, 1, 3}, {41.0 / 200, -9.0 / 5, 4.0 / 5},
     {-5927.0 / 50400, 4.0 / 5, -9.0 / 5}, {17.0 / 600, -1.0 / 5, -4.0 / 5},
     {-503.0 / 50400, 1.0 / 5, 4.0 / 5}, {0, 0, 0}, {0, 0, 0}},
    {{-1.0 / 280, 0, 0}, {1097.0 / 5040, -2, 6}, {-1349.0 / 10080, 3, -12},
     {-887.0 / 5040, -1, 6}, {3613.0 / 50400, 4.0 / 5, -9.0 / 5},
     {467.0 / 25200, -3.0 / 5, 18.0 / 5}, {139.0 / 25200, -1.0 / 5, -9.0 / 5}, {0, 0, 0}},
    {{17.0 / 1680, 0, 2}, {-319.0 / 2520, 2, -8}, {-919.0 / 5040, -2, 6}, {-445.0 / 2016, 0, 0},
     {583.0 / 720, -1, 6}, {-65.0 / 224, 0, -7}, {0, 1, 0}, {0, 0, 1}},
};
static const affine_t T6[3][6] = {
    {{-11.0 / 180, 1, 0}, {1.0 / 9, -2, 0}, {-1.0 / 18, 1, 0}, {1.0 / 180, 0, 0}, {0, 0, 0},
     {0, 0, 0}},
    {{7.0 / 60, -3, 0}, {-1.0 / 120, 5, 0}, {-17.0 / 90, -2, 0}, {5.0 / 72, 1, 0},
     {1.0 / 90, -1, 0}, {0, 0, 0}},
    {{-1.0 / 15, 3, 0}, {-11.0 / 60, -3, 0}, {-101.0 / 360, 0, 0}, {137.0 / 180, -2, 0},
     {-83.0 / 360, 1, 0}, {0, 1, 0}},
};

int or_build_narrow(int order, const double* params, int nparams, double* m64, int* s_out) {
  if (!((order == 8 && nparams == 2) || (order == 6 && nparams == 1))) return 1;
  const int s = order == 8 ? 4 : 3;
  const double x = params[0];
  const double y = order == 8 ? params[1] : 0.0;
  memset(m64, 0, sizeof(double) * 64);
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < 2 * s; ++j) {
      const affine_t t = order == 8 ? T8[i][j] : T6[i][j];
      const double v = t.c + t.p * x + t.q * y; /* stencil.cpp:85 eval() order */
      m64[i * 8 + j] = v;
      m64[(2 * s - 1 - i) * 8 + (2 * s - 1 - j)] = -v; /* central antisymmetry */
    }
  *s_out = s;
  return 0;
}

/* ------------------------------------------------------- line kernels */
void or_narrow_interfaces(int s, const double* a, const double* u, int n, const double* m64,
                          double* h) {
  /* stencil_kernel.hpp:13-25 */
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int mm = -s + 1; mm <= s; ++mm) {
      double v = 0.0;
      for (int nn = -s + 1; nn <= s; ++nn) v += m64[(mm + s - 1) * 8 + nn + s - 1] * u[i + nn];
      acc += a[i + mm] * v;
    }
    h[i] = acc;
  }
}

/* periodic copy into a buffer valid on [-l, n + r) (stencil.cpp:105-113,
 * pde.cpp:79-83) */
static double* pad(const double* f, int n, int l, int r, double* buf) {
  double* p = buf + l;
  for (int i = 0; i < n; ++i) p[i] = f[i];
  for (int i = 1; i <= l; ++i) p[-i] = f[((n - i) % n + n) % n];
  for (int i = 0; i < r; ++i) p[n + i] = f[i % n];
  return p;
}

int or_apply_narrow(const double* m64, int s, const double* a, const double* u, int n, double dx,
                    double* out) {
  /* stencil.cpp:134-155 */
  if (n < 2 * s || !(dx > 0.0)) return 1;
  double* ab = malloc(sizeof(double) * (n + 2 * s));
  double* ub = malloc(sizeof(double) * (n + 2 * s));
  double* h = malloc(sizeof(double) * n);
  const double* ap = pad(a, n, s - 1, s, ab);
  const double* up = pad(u, n, s - 1, s, ub);
  or_narrow_interfaces(s, ap, up, n, m64, h);
  const double inv = 1.0 / (dx * dx);
  out[0] = (h[0] - h[n - 1]) * inv;
  for (int i = 1; i < n; ++i) out[i] = (h[i] - h[i - 1]) * inv;
  free(ab);
  free(ub);
  free(h);
  return 0;
}

static const double C1 = 4.0 / 5.0, C2 = -1.0 / 5.0, C3 = 4.0 / 105.0, C4 = -1.0 / 280.0;

int or_first_derivative8(const double* u, int n, double dx, double* out) {
  /* stencil.cpp:157-169, stencil_kernel.hpp:48-54 */
  if (n < 9 || !(dx > 0.0)) return 1;
  double* b = malloc(sizeof(double) * (n + 8));
  const double* p = pad(u, n, 4, 4, b);
  const double inv = 1.0 / dx;
  for (int i = 0; i < n; ++i)
    out[i] = (C1 * (p[i + 1] - p[i - 1]) + C2 * (p[i + 2] - p[i - 2]) +
              C3 * (p[i + 3] - p[i - 3]) + C4 * (p[i + 4] - p[i - 4])) *
             inv;
  free(b);
  return 0;
}

int or_apply_wide(const double* a, const double* u, int n, double dx, double* out) {
  /* stencil.cpp:171-176 */
  double* du = malloc(sizeof(double) * n);
  if (or_first_derivative8(u, n, dx, du)) {
    free(du);
    return 1;
  }
  for (int i = 0; i < n; ++i) du[i] *= a[i];
  const int rc = or_first_derivative8(du, n, dx, out);
  free(du);
  return rc;
}

/* ------------------------------------------------------ 3-D operators */
static inline long long lin(int i, int j, int k, int nx, int ny) {
  return ((long long)k * ny + j) * nx + i;
}

void or_narrow_dir(const double* m64, int s, const double* c, const double* u, int nx, int ny,
                   int nz, int dir, double inv_d2, int accumulate, double* out) {
  /* One direction of narrow_rhs_rows<S> (pde.cpp:85-129): interfaces once per
   * line, then differenced.  Lines along dir are gathered with periodic wrap;
   * lines are independent, so they are shared out over OpenMP threads (the
   * reference's parallel_for over rows, parallel.cpp:20-36) with the same
   * per-element arithmetic: bitwise independent of the thread count. */
  const int n = dir == 0 ? nx : dir == 1 ? ny : nz;
  const int n1 = dir == 0 ? ny : nx, n2 = dir == 2 ? ny : nz;
  const long long lines = (long long)n1 * n2;
#pragma omp parallel if (lines * n > 4096)
  {
    double* cl = malloc(sizeof(double) * n);
    double* ul = malloc(sizeof(double) * n);
    double* cb = malloc(sizeof(double) * (n + 2 * s));
    double* ub = malloc(sizeof(double) * (n + 2 * s));
    double* h = malloc(sizeof(double) * n);
#pragma omp for schedule(static)
    for (long long line = 0; line < lines; ++line) {
      const int b1 = (int)(line % n1), b2 = (int)(line / n1);
      for (int q = 0; q < n; ++q) {
        int i, j, k;
        if (dir == 0) { i = q; j = b1; k = b2; }
        else if (dir == 1) { i = b1; j = q; k = b2; }
        else { i = b1; j = b2; k = q; }
        const long long o = lin(i, j, k, nx, ny);
        cl[q] = c[o];
        ul[q] = u[o];
      }
      const double* cp = pad(cl, n, s - 1, s, cb);
      const double* up = pad(ul, n, s - 1, s, ub);
      or_narrow_interfaces(s, cp, up, n, m64, h);
      for (int q = 0; q < n; ++q) {
        int i, j, k;
        if (dir == 0) { i = q; j = b1; k = b2; }
        else if (dir == 1) { i = b1; j = q; k = b2; }
        else { i = b1; j = b2; k = q; }
        const long long o = lin(i, j, k, nx, ny);
        const double v = (h[q] - h[(q - 1 + n) % n]) * inv_d2;
        out[o] = accumulate ? out[o] + v : v;
      }
    }
    free(cl);
    free(ul);
    free(cb);
    free(ub);
    free(h);
  }
}

void or_deriv8_dir(const double* u, int nx, int ny, int nz, int dir, double inv_d, double* out) {
  /* stencil_kernel.hpp:48-54 along dir with periodic wrap.  The wrapped
   * neighbour offsets come from a table (no modulo per access); the
   * arithmetic is the reference's expression in its order. */
  const long long st = dir == 0 ? 1 : dir == 1 ? nx : (long long)nx * ny;
  const int n = dir == 0 ? nx : dir == 1 ? ny : nz;
  long long* wrap = malloc(sizeof(long long) * (n + 8));
  for (int q = -4; q < n + 4; ++q) wrap[q + 4] = (long long)(((q % n) + n) % n) * st;
#pragma omp parallel for schedule(static) if ((long long)nx * ny * nz > 4096)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int q = dir == 0 ? i : dir == 1 ? j : k;
        const long long base = lin(i, j, k, nx, ny) - (long long)q * st;
        const long long* w = wrap + q + 4;
#define AT(d) u[base + w[d]]
        out[lin(i, j, k, nx, ny)] =
            (C1 * (AT(1) - AT(-1)) + C2 * (AT(2) - AT(-2)) + C3 * (AT(3) - AT(-3)) +
             C4 * (AT(4) - AT(-4))) *
            inv_d;
#undef AT
      }
  free(wrap);
}

int or_narrow3d(const double* m64, int s, const double* a, const double* u, int nx, int ny,
                int nz, double dx, double dy, double dz, double* out) {
  if (nx < 2 * s || ny < 2 * s || nz < 2 * s) return 1;
  /* out = dHx/dx^2 + dHy/dy^2 + dHz/dz^2, added in that order (pde.cpp:118-120) */
  or_narrow_dir(m64, s, a, u, nx, ny, nz, 0, 1.0 / (dx * dx), 0, out);
  or_narrow_dir(m64, s, a, u, nx, ny, nz, 1, 1.0 / (dy * dy), 1, out);
  or_narrow_dir(m64, s, a, u, nx, ny, nz, 2, 1.0 / (dz * dz), 1, out);
  return 0;
}

int or_heat2d_rhs(int kind, const double* m64, int s, const double* a, const double* b,
                  const double* g0, double gt, const double* u, int nx, int ny, double dx,
                  double dy, double* out) {
  const long long n = (long long)nx * ny;
  if (kind == 0 || kind == 1) {
    /* narrow_rhs_rows<S> (pde.cpp:85-129) */
    if (nx < 2 * s + 1 || ny < 2 * s + 1) return 1;
    or_narrow_dir(m64, s, a, u, nx, ny, 1, 0, 1.0 / (dx * dx), 0, out);
    or_narrow_dir(m64, s, b, u, nx, ny, 1, 1, 1.0 / (dy * dy), 1, out);
  } else {
    /* wide_pass1 / wide_pass2 (pde.cpp:131-194) */
    if (nx < 9 || ny < 9) return 1;
    double* w1 = malloc(sizeof(double) * n);
    double* w2 = malloc(sizeof(double) * n);
    double* t = malloc(sizeof(double) * n);
    or_deriv8_dir(u, nx, ny, 1, 0, 1.0 / dx, t);
    for (long long q = 0; q < n; ++q) w1[q] = a[q] * t[q];
    or_deriv8_dir(u, nx, ny, 1, 1, 1.0 / dy, t);
    for (long long q = 0; q < n; ++q) w2[q] = b[q] * t[q];
    or_deriv8_dir(w1, nx, ny, 1, 0, 1.0 / dx, out);
    or_deriv8_dir(w2, nx, ny, 1, 1, 1.0 / dy, t);
    for (long long q = 0; q < n; ++q) out[q] = out[q] + t[q];
    free(w1);
    free(w2);
    free(t);
  }
  if (g0)
    for (long long q = 0; q < n; ++q) out[q] += g0[q] * gt; /* pde.cpp:121-123 */
  return 0;
}

/* ------------------------------------------------------------- SDC */
static int stalled(const double* hist, int len, double cutoff) {
  /* sdc.cpp:9-16 */
  if (cutoff <= 0.0 || len < 2) return 0;
  const double prev = hist[len - 2], cur = hist[len - 1];
  if (cur == 0.0) return 1;
  const double ratio = prev / cur;
  return ratio >= 1.0 - cutoff && ratio <= 1.0 + cutoff;
}

int or_integrate_sdc(or_rhs_cb f, void* ctx, long long dim, const double* u0, double t0,
                     double t1, int nsteps, int m, const double* tau, const double* q,
                     const double* smat, int iterations, double cutoff, int reuse_first,
                     double* u_out, double* residuals, int max_res, int* sweeps,
                     int* fresh_evals, int* early_stop) {
  if (nsteps < 0 || iterations < 1) return 1;
  const size_t bytes = sizeof(double) * dim;
  double* U = malloc(bytes * (m + 1));
  double* F = malloc(bytes * (m + 1));
  double* I = malloc(bytes * m);
  double* fold = malloc(bytes);
  double* u = malloc(bytes);
  double* fcarry = malloc(bytes);
  double* hist = malloc(sizeof(double) * (iterations + 1));
  memcpy(u, u0, bytes);
  *sweeps = 0;
  *fresh_evals = 0;
  *early_stop = 0;
  int nres = 0;
  const double dt = (t1 - t0) / (nsteps > 1 ? nsteps : 1);
  for (int step = 0; step < nsteps; ++step) {
    const double tn = t0 + step * dt;
    /* SdcStepper::step, sdc.cpp:38-96 */
    for (int k = 0; k <= m; ++k) memcpy(U + k * dim, u, bytes);
    if (step > 0 && reuse_first) {
      memcpy(F, fcarry, bytes);
    } else {
      f(tn, u, F, dim, ctx);
      ++*fresh_evals;
    }
    for (int k = 1; k <= m; ++k) memcpy(F + k * dim, F, bytes);
    int hl = 0;
    for (int it = 1; it <= iterations; ++it) {
      for (int r = 0; r < m; ++r)
#pragma omp parallel for schedule(static) if (dim > 4096)
        for (long long i = 0; i < dim; ++i) {
          double acc = 0.0;
          for (int j = 0; j <= m; ++j) acc += smat[r * (m + 1) + j] * F[j * dim + i];
          I[r * dim + i] = dt * acc;
        }
      for (int r = 0; r < m; ++r) {
        const double dtm = (tau[r + 1] - tau[r]) * dt;
        double* next = U + (r + 1) * dim;
        const double* cur = U + r * dim;
        if (r == 0) {
#pragma omp parallel for schedule(static) if (dim > 4096)
          for (long long i = 0; i < dim; ++i) next[i] = cur[i] + I[i];
        } else {
#pragma omp parallel for schedule(static) if (dim > 4096)
          for (long long i = 0; i < dim; ++i)
            next[i] = cur[i] + dtm * (F[r * dim + i] - fold[i]) + I[r * dim + i];
        }
        memcpy(fold, F + (r + 1) * dim, bytes);
        f(tn + tau[r + 1] * dt, next, F + (r + 1) * dim, dim, ctx);
        ++*fresh_evals;
      }
      /* sdc_residual, sdc.cpp:20-30 */
      double res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res) if (dim > 4096)
      for (long long i = 0; i < dim; ++i) {
        double acc = 0.0;
        for (int j = 0; j <= m; ++j) acc += q[(m - 1) * (m + 1) + j] * F[j * dim + i];
        const double r = fabs(u[i] + dt * acc - U[m * dim + i]);
        if (r > res) res = r;
      }
      hist[hl++] = res;
      if (residuals && nres < max_res) residuals[nres] = res;
      ++nres;
      ++*sweeps;
      if (stalled(hist, hl, cutoff)) {
        *early_stop = 1;
        break;
      }
    }
    memcpy(u, U + m * dim, bytes);
    memcpy(fcarry, F + m * dim, bytes);
  }
  memcpy(u_out, u, bytes);
  free(U);
  free(F);
  free(I);
  free(fold);
  free(u);
  free(fcarry);
  free(hist);
  return 0;
}

/* ------------------------------------------------------------ MRSDC */
int or_integrate_mrsdc1(or_rhs_cb f1, void* c1, or_rhs_cb f2, void* c2, long long dim,
                        const double* u0, double t0, double tend, int nsteps, int m1,
                        const double* t1, int m2, const double* t2, const double* s21,
                        const double* q21, const double* s22, const double* q22,
                        const int* fine_of_coarse, const int* p_map, int iterations,
                        double cutoff, double* u_out, double* residuals, int max_res,
                        int* sweeps, int* f1_evals, int* f2_evals) {
  if (nsteps < 0 || iterations < 1) return 1;
  const size_t bytes = sizeof(double) * dim;
  double* U = malloc(bytes * (m2 + 1));
  double* F1 = malloc(bytes * (m1 + 1));
  double* F2 = malloc(bytes * (m2 + 1));
  double* OF1 = malloc(bytes * (m1 + 1));
  double* SO = malloc(bytes * m2);
  double* fold = malloc(bytes);
  double* u = malloc(bytes);
  double* c1s = malloc(bytes);
  double* c2s = malloc(bytes);
  double* hist = malloc(sizeof(double) * (iterations + 1));
  int* coarse_at = malloc(sizeof(int) * (m2 + 1));
  memcpy(u, u0, bytes);
  *sweeps = *f1_evals = *f2_evals = 0;
  int nres = 0;
  const double dt = (tend - t0) / (nsteps > 1 ? nsteps : 1);
  for (int q = 0; q <= m2; ++q) coarse_at[q] = -1;
  for (int p = 0; p <= m1; ++p) coarse_at[fine_of_coarse[p]] = p;
  for (int step = 0; step < nsteps; ++step) {
    const double tn = t0 + step * dt;
    /* provisional, mrsdc.cpp:43-66 (reuse_first_eval defaults to true) */
    for (int q = 0; q <= m2; ++q) memcpy(U + q * dim, u, bytes);
    if (step > 0) memcpy(F1, c1s, bytes); else { f1(tn, u, F1, dim, c1); ++*f1_evals; }
    if (step > 0) memcpy(F2, c2s, bytes); else { f2(tn, u, F2, dim, c2); ++*f2_evals; }
    for (int p = 1; p <= m1; ++p) memcpy(F1 + p * dim, F1, bytes);
    for (int q = 1; q <= m2; ++q) memcpy(F2 + q * dim, F2, bytes);
    int hl = 0;
    for (int it = 1; it <= iterations; ++it) {
      /* accumulate_node_terms, mrsdc.cpp:69-82 */
      for (int q = 0; q < m2; ++q)
#pragma omp parallel for schedule(static) if (dim > 4096)
        for (long long i = 0; i < dim; ++i) {
          double acc = 0.0;
          for (int j = 0; j <= m1; ++j) acc += s21[q * (m1 + 1) + j] * F1[j * dim + i];
          for (int j = 0; j <= m2; ++j) acc += s22[q * (m2 + 1) + j] * F2[j * dim + i];
          SO[q * dim + i] = dt * acc;
        }
      memcpy(OF1, F1, bytes * (m1 + 1));
      memcpy(fold, F2, bytes);
      /* step_mode1 fine sweep, mrsdc.cpp:105-120 */
      for (int q = 0; q < m2; ++q) {
        const double dtq = (t2[q + 1] - t2[q]) * dt;
        const int p = p_map[q];
        double* next = U + (q + 1) * dim;
        const double* cur = U + q * dim;
#pragma omp parallel for schedule(static) if (dim > 4096)
        for (long long i = 0; i < dim; ++i)
          next[i] = cur[i] + dtq * (F1[p * dim + i] - OF1[p * dim + i]) +
                    dtq * (F2[q * dim + i] - fold[i]) + SO[q * dim + i];
        memcpy(fold, F2 + (q + 1) * dim, bytes);
        f2(tn + t2[q + 1] * dt, next, F2 + (q + 1) * dim, dim, c2);
        ++*f2_evals;
        const int pc = coarse_at[q + 1];
        if (pc > 0) {
          f1(tn + t1[pc] * dt, next, F1 + pc * dim, dim, c1);
          ++*f1_evals;
        }
      }
      /* mrsdc_residual, mrsdc.cpp:23-35 */
      double res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res) if (dim > 4096)
      for (long long i = 0; i < dim; ++i) {
        double acc = 0.0;
        for (int j = 0; j <= m1; ++j) acc += q21[(m2 - 1) * (m1 + 1) + j] * F1[j * dim + i];
        for (int j = 0; j <= m2; ++j) acc += q22[(m2 - 1) * (m2 + 1) + j] * F2[j * dim + i];
        const double r = fabs(u[i] + dt * acc - U[m2 * dim + i]);
        if (r > res) res = r;
      }
      hist[hl++] = res;
      if (residuals && nres < max_res) residuals[nres] = res;
      ++nres;
      ++*sweeps;
      if (stalled(hist, hl, cutoff)) break;
    }
    memcpy(u, U + m2 * dim, bytes);
    memcpy(c1s, F1 + m1 * dim, bytes);
    memcpy(c2s, F2 + m2 * dim, bytes);
  }
  memcpy(u_out, u, bytes);
  free(U); free(F1); free(F2); free(OF1); free(SO); free(fold); free(u); free(c1s); free(c2s);
  free(hist); free(coarse_at);
  return 0;
}

/* ------------------------------------------------- implicit (mode 2) */
static double max_keep(double a, double b) { return (a < b) ? b : a; } /* std::max(a, b) */

static long long blk_at(long long b, long long j, long long B, long long nb, int inter) {
  return inter ? j * nb + b : b * B + j;
}

/* lu_factor (core/src/matrix.cpp:9-33) on one row-major n x n block */
static int lu_factor_blk(double* m, int n, int* piv) {
  for (int col = 0; col < n; ++col) {
    int best = col;
    double best_mag = fabs(m[col * n + col]);
    for (int r = col + 1; r < n; ++r) {
      const double mag = fabs(m[r * n + col]);
      if (mag > best_mag) {
        best = r;
        best_mag = mag;
      }
    }
    piv[col] = best;
    if (best_mag == 0.0) return 0;
    if (best != col)
      for (int c = 0; c < n; ++c) {
        const double tmp = m[col * n + c];
        m[col * n + c] = m[best * n + c];
        m[best * n + c] = tmp;
      }
    const double inv = 1.0 / m[col * n + col];
    for (int r = col + 1; r < n; ++r) {
      const double l = m[r * n + col] * inv;
      m[r * n + col] = l;
      for (int c = col + 1; c < n; ++c) m[r * n + c] -= l * m[col * n + c];
    }
  }
  return 1;
}

/* lu_solve (core/src/matrix.cpp:35-51) */
static void lu_solve_blk(const double* m, int n, const int* piv, double* b) {
  for (int i = 0; i < n; ++i)
    if (piv[i] != i) {
      const double tmp = b[i];
      b[i] = b[piv[i]];
      b[piv[i]] = tmp;
    }
  for (int i = 1; i < n; ++i) {
    double s = b[i];
    for (int j = 0; j < i; ++j) s -= m[i * n + j] * b[j];
    b[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= m[i * n + j] * b[j];
    b[i] = s / m[i * n + i];
  }
}

int or_solve_backward_euler(or_rhs_cb f, void* ctx, long long dim, double t, double beta,
                            const double* c, const double* guess, const or_stiff* o, double* w,
                            or_newton_report* rep) {
  const long long B = o->block > 0 ? o->block : dim;
  if (dim < 1 || B < 1 || dim % B != 0 || B > 4096) return 1;
  const long long nb = dim / B;
  const int inter = o->block > 0 && o->interleaved;
  const size_t bytes = sizeof(double) * dim;
  double* fw = malloc(bytes);
  double* fp = malloc(bytes);
  double* wp = malloc(bytes);
  double* delta = malloc(bytes);
  double* jac = malloc(sizeof(double) * nb * B * B);
  double* hcol = malloc(sizeof(double) * nb);
  double* rhs = malloc(sizeof(double) * B);
  int* piv = malloc(sizeof(int) * nb * B);
  const double root_eps = sqrt(2.220446049250313e-16); /* sqrt(DBL_EPSILON), stiff.cpp:19 */
  memcpy(w, guess, bytes);
  rep->iterations = 0;
  rep->final_residual = 0.0;
  rep->converged = 0;
  rep->f_evals = 0;
  for (int iter = 0; iter < o->max_newton_iters; ++iter) {
    f(t, w, fw, dim, ctx);
    ++rep->f_evals;
    double rnorm = 0.0;
    for (long long i = 0; i < dim; ++i) {
      delta[i] = w[i] - beta * fw[i] - c[i];
      rnorm = max_keep(rnorm, fabs(delta[i]));
    }
    rep->final_residual = rnorm;
    double wn = 0.0; /* max_norm, field.hpp:18-22 */
    for (long long i = 0; i < dim; ++i) wn = max_keep(wn, fabs(w[i]));
    if (rnorm <= o->atol + o->rtol * wn) {
      rep->converged = 1;
      break;
    }
    /* fd_jacobian (stiff.cpp:16-30), one block column at a time */
    memcpy(wp, w, bytes);
    for (long long j = 0; j < B; ++j) {
      for (long long b = 0; b < nb; ++b) {
        const long long i = blk_at(b, j, B, nb, inter);
        hcol[b] = root_eps * max_keep(fabs(w[i]), o->atol);
        wp[i] = w[i] + hcol[b];
      }
      f(t, wp, fp, dim, ctx);
      ++rep->f_evals;
      for (long long b = 0; b < nb; ++b) {
        const long long i = blk_at(b, j, B, nb, inter);
        wp[i] = w[i];
        const double inv = 1.0 / hcol[b];
        for (long long r = 0; r < B; ++r) {
          const long long k = blk_at(b, r, B, nb, inter);
          jac[(b * B + r) * B + j] = (fp[k] - fw[k]) * inv;
        }
      }
    }
    /* jg = I - beta J (stiff.cpp:63-65), factored block by block */
    int ok = 1;
    for (long long b = 0; b < nb && ok; ++b) {
      double* m = jac + b * B * B;
      for (long long r = 0; r < B; ++r)
        for (long long cc = 0; cc < B; ++cc)
          m[r * B + cc] = (r == cc ? 1.0 : 0.0) - beta * m[r * B + cc];
      ok = lu_factor_blk(m, (int)B, piv + b * B);
    }
    if (!ok) break;
    for (long long b = 0; b < nb; ++b) {
      for (long long r = 0; r < B; ++r) rhs[r] = delta[blk_at(b, r, B, nb, inter)];
      lu_solve_blk(jac + b * B * B, (int)B, piv + b * B, rhs);
      for (long long r = 0; r < B; ++r) delta[blk_at(b, r, B, nb, inter)] = rhs[r];
    }
    for (long long i = 0; i < dim; ++i) w[i] -= delta[i];
    rep->iterations = iter + 1;
  }
  free(fw); free(fp); free(wp); free(delta); free(jac); free(hcol); free(rhs); free(piv);
  return 0;
}

int or_integrate_mrsdc2(or_rhs_cb f1, void* c1, or_rhs_cb f2, void* c2, long long dim,
                        const double* u0, double t0, double tend, int nsteps, int m1,
                        const double* t1, int m2, const double* t2, const double* s21,
                        const double* q21, const double* s22, const double* q22,
                        const int* fine_of_coarse, int iterations, double cutoff,
                        const or_stiff* opts, double* u_out, double* residuals, int max_res,
                        int* sweeps, int* f1_evals, int* f2_evals, int* implicit_solves,
                        int* newton_f1_evals, int* fail_node, int* fail_sweep) {
  if (nsteps < 0 || iterations < 1) return 1;
  const size_t bytes = sizeof(double) * dim;
  double* U = malloc(bytes * (m2 + 1));
  double* F1 = malloc(bytes * (m1 + 1));
  double* F2 = malloc(bytes * (m2 + 1));
  double* OF1 = malloc(bytes * (m1 + 1));
  double* SO = malloc(bytes * m2);
  double* fold = malloc(bytes);
  double* cvec = malloc(bytes);
  double* wsol = malloc(bytes);
  double* u = malloc(bytes);
  double* c1s = malloc(bytes);
  double* c2s = malloc(bytes);
  double* hist = malloc(sizeof(double) * (iterations + 1));
  int rc = 0;
  memcpy(u, u0, bytes);
  *sweeps = *f1_evals = *f2_evals = *implicit_solves = *newton_f1_evals = 0;
  *fail_node = *fail_sweep = -1;
  int nres = 0;
  const double dt = (tend - t0) / (nsteps > 1 ? nsteps : 1);
  for (int step = 0; step < nsteps && rc == 0; ++step) {
    const double tn = t0 + step * dt;
    /* provisional, mrsdc.cpp:43-66 */
    for (int q = 0; q <= m2; ++q) memcpy(U + q * dim, u, bytes);
    if (step > 0) memcpy(F1, c1s, bytes); else { f1(tn, u, F1, dim, c1); ++*f1_evals; }
    if (step > 0) memcpy(F2, c2s, bytes); else { f2(tn, u, F2, dim, c2); ++*f2_evals; }
    for (int p = 1; p <= m1; ++p) memcpy(F1 + p * dim, F1, bytes);
    for (int q = 1; q <= m2; ++q) memcpy(F2 + q * dim, F2, bytes);
    int hl = 0;
    for (int it = 1; it <= iterations && rc == 0; ++it) {
      /* accumulate_node_terms, mrsdc.cpp:69-82 */
      for (int q = 0; q < m2; ++q)
#pragma omp parallel for schedule(static) if (dim > 4096)
        for (long long i = 0; i < dim; ++i) {
          double acc = 0.0;
          for (int j = 0; j <= m1; ++j) acc += s21[q * (m1 + 1) + j] * F1[j * dim + i];
          for (int j = 0; j <= m2; ++j) acc += s22[q * (m2 + 1) + j] * F2[j * dim + i];
          SO[q * dim + i] = dt * acc;
        }
      memcpy(OF1, F1, bytes * (m1 + 1));
      memcpy(fold, F2, bytes);
      /* step_mode2 coarse intervals, mrsdc.cpp:156-194 */
      for (int p = 0; p < m1; ++p) {
        const int qa = fine_of_coarse[p], qb = fine_of_coarse[p + 1];
        const double dt1 = (t1[p + 1] - t1[p]) * dt;
        const double t_right = tn + t1[p + 1] * dt;
        for (long long i = 0; i < dim; ++i) {
          double acc = 0.0;
          for (int q = qa; q < qb; ++q) acc += SO[q * dim + i];
          cvec[i] = U[qa * dim + i] + acc - dt1 * OF1[(p + 1) * dim + i];
        }
        or_newton_report rep;
        or_solve_backward_euler(f1, c1, dim, t_right, dt1, cvec, U + qb * dim, opts, wsol, &rep);
        ++*implicit_solves;
        *newton_f1_evals += rep.f_evals;
        if (!rep.converged) {
          *fail_node = p + 1;
          *fail_sweep = it;
          rc = 2;
          break;
        }
        f1(t_right, wsol, F1 + (p + 1) * dim, dim, c1);
        ++*f1_evals;
        for (int q = qa; q < qb; ++q) {
          const double dtq = (t2[q + 1] - t2[q]) * dt;
          double* next = U + (q + 1) * dim;
          const double* cur = U + q * dim;
          for (long long i = 0; i < dim; ++i)
            next[i] = cur[i] + dtq * (F1[(p + 1) * dim + i] - OF1[(p + 1) * dim + i]) +
                      dtq * (F2[q * dim + i] - fold[i]) + SO[q * dim + i];
          memcpy(fold, F2 + (q + 1) * dim, bytes);
          f2(tn + t2[q + 1] * dt, next, F2 + (q + 1) * dim, dim, c2);
          ++*f2_evals;
        }
      }
      if (rc) break;
      /* mrsdc_residual, mrsdc.cpp:23-35 */
      double res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res) if (dim > 4096)
      for (long long i = 0; i < dim; ++i) {
        double acc = 0.0;
        for (int j = 0; j <= m1; ++j) acc += q21[(m2 - 1) * (m1 + 1) + j] * F1[j * dim + i];
        for (int j = 0; j <= m2; ++j) acc += q22[(m2 - 1) * (m2 + 1) + j] * F2[j * dim + i];
        res = max_keep(res, fabs(u[i] + dt * acc - U[m2 * dim + i]));
      }
      hist[hl++] = res;
      if (residuals && nres < max_res) residuals[nres] = res;
      ++nres;
      ++*sweeps;
      if (stalled(hist, hl, cutoff)) break;
    }
    memcpy(u, U + m2 * dim, bytes);
    memcpy(c1s, F1 + m1 * dim, bytes);
    memcpy(c2s, F2 + m2 * dim, bytes);
  }
  memcpy(u_out, u, bytes);
  free(U); free(F1); free(F2); free(OF1); free(SO); free(fold); free(cvec); free(wsol);
  free(u); free(c1s); free(c2s); free(hist);
  return rc;
}

/* ------------------------------------------------- integrate_stiff */
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* bdf2_coeff (stiff.cpp:118-121) */
static double bdf2_coeff(double rho) {
  return -(1.0 + rho) * (1.0 + rho) / (6.0 * rho * (1.0 + 2.0 * rho));
}

/* be_solve / bdf2_solve (stiff.cpp:82-106): 1 when Newton converged */
static int be_step(or_rhs_cb f, void* ctx, long long dim, double t_new, double h,
                   const double* u_n, const or_stiff* o, double* out) {
  or_newton_report rep;
  or_solve_backward_euler(f, ctx, dim, t_new, h, u_n, u_n, o, out, &rep);
  return rep.converged;
}
static int bdf2_step(or_rhs_cb f, void* ctx, long long dim, double t_new, double h, double rho,
                     const double* u_nm1, const double* u_n, const or_stiff* o, double* out,
                     double* c, double* guess) {
  const double denom = 1.0 + 2.0 * rho;
  for (long long i = 0; i < dim; ++i) {
    c[i] = ((1.0 + rho) * (1.0 + rho) * u_n[i] - rho * rho * u_nm1[i]) / denom;
    guess[i] = u_n[i] + rho * (u_n[i] - u_nm1[i]);
  }
  or_newton_report rep;
  or_solve_backward_euler(f, ctx, dim, t_new, h * (1.0 + rho) / denom, c, guess, o, out, &rep);
  return rep.converged;
}

int or_integrate_stiff(or_rhs_cb f, void* ctx, long long dim, const double* u0, double t0,
                       double t1, const or_stiff* o, double initial_step_fraction,
                       double* u_out, int* accepted, int* rejected, double* t_fail) {
  const double span = t1 - t0;
  const size_t bytes = sizeof(double) * dim;
  *accepted = *rejected = 0;
  *t_fail = 0.0;
  if (span == 0.0) {
    memcpy(u_out, u0, bytes);
    return 0;
  }
  if (span < 0.0 || o->rtol <= 0.0 || o->atol < 0.0) return 1;
  double* u = malloc(bytes);
  double* u_prev = malloc(bytes);
  double* y_full = malloc(bytes);
  double* y_mid = malloc(bytes);
  double* y_half = malloc(bytes);
  double* c = malloc(bytes);
  double* guess = malloc(bytes);
  memcpy(u, u0, bytes);
  double t = t0, h_prev = 0.0;
  double h = clampd(initial_step_fraction, 1e-12, 1.0) * span;
  const double h_min = 1e-14 * span;
  int have_history = 0, rc = 0;
  while (t < t1) {
    h = h < t1 - t ? h : t1 - t;
    if (h < h_min) {
      *t_fail = t;
      rc = 2;
      break;
    }
    int ok;
    double weight;
    if (!have_history) {
      ok = be_step(f, ctx, dim, t + h, h, u, o, y_full) &&
           be_step(f, ctx, dim, t + 0.5 * h, 0.5 * h, u, o, y_mid) &&
           be_step(f, ctx, dim, t + h, 0.5 * h, y_mid, o, y_half);
      weight = 1.0;
    } else {
      const double rho_full = h / h_prev;
      const double rho_mid = 0.5 * h / h_prev;
      ok = bdf2_step(f, ctx, dim, t + h, h, rho_full, u_prev, u, o, y_full, c, guess) &&
           bdf2_step(f, ctx, dim, t + 0.5 * h, 0.5 * h, rho_mid, u_prev, u, o, y_mid, c, guess) &&
           bdf2_step(f, ctx, dim, t + h, 0.5 * h, 1.0, u, y_mid, o, y_half, c, guess);
      const double c_full = bdf2_coeff(rho_full);
      const double c_half = ((4.0 / 3.0) * bdf2_coeff(rho_mid) + bdf2_coeff(1.0)) / 8.0;
      weight = clampd(c_half / (c_full - c_half), 0.05, 2.0);
    }
    if (!ok) {
      h *= 0.5;
      ++*rejected;
      continue;
    }
    double diff = 0.0, yn = 0.0;
    for (long long i = 0; i < dim; ++i) {
      diff = max_keep(diff, fabs(y_full[i] - y_half[i]));
      yn = max_keep(yn, fabs(y_half[i]));
    }
    const double err = weight * diff;
    const double p = have_history ? 3.0 : 2.0;
    const double tol = o->rtol * yn + o->atol;
    if (err <= tol) {
      for (long long i = 0; i < dim; ++i) y_half[i] += weight * (y_half[i] - y_full[i]);
      double* tmp = u_prev;
      u_prev = u;
      u = y_half;
      y_half = tmp;
      t += h;
      h_prev = h;
      have_history = 1;
      ++*accepted;
    } else {
      ++*rejected;
    }
    double factor = err > 0.0 ? 0.9 * pow(tol / err, 1.0 / p) : 5.0;
    factor = clampd(factor, 0.2, 5.0);
    h *= factor;
  }
  memcpy(u_out, u, bytes);
  free(u); free(u_prev); free(y_full); free(y_mid); free(y_half); free(c); free(guess);
  return rc;
}

/* Thread count of the OpenMP loops (0: the runtime default, i.e. every host
 * thread or OMP_NUM_THREADS).  Results do not depend on it. */
void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
  (void)n;
#endif
}

int or_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------- physical boundaries (§8(f) 4)
 * Non-periodic lines with the closure of PAPER.md:449-461: 8th-order stencils
 * from the fifth cell on, 6th and 4th-order centred stencils at the fourth
 * and third cells, centred 2nd order (diffusion) / biased 3rd order
 * (advection) at the second cell, completely biased 2nd (diffusion) / 3rd
 * (advection) order at the boundary cell; mirrored at the far end.  The
 * paper gives the orders, not the coefficients: the centred narrow
 * interfaces of order 6 use the reference's 6th-order matrix at its default
 * parameter (stencil.hpp:33, m36 = 281/3600), order 4 the narrow matrix of
 * the 2-parameter 4th-order family with zero corners (m33 = 0, m32 = -1/12:
 * for a = 1 the classic (-1, 16, -30, 16, -1)/12), order 2
 * H = (a_i + a_{i+1})/2 (u_{i+1} - u_i); the biased formulas are the
 * classical one-sided ones. */
static const double M4B[4][4] = {{0.0, 1.0 / 12.0, -1.0 / 12.0, 0.0},
                                 {1.0 / 12.0, -3.0 / 4.0, 2.0 / 3.0, 0.0},
                                 {0.0, -2.0 / 3.0, 3.0 / 4.0, -1.0 / 12.0},
                                 {0.0, 1.0 / 12.0, -1.0 / 12.0, 0.0}};

/* one narrow interface i+1/2 of half width s from an 8x8 (or smaller) matrix */
static double iface(int s, const double* mat, int pitch, const double* a, const double* u, int i) {
  double acc = 0.0;
  for (int mm = -s + 1; mm <= s; ++mm) {
    double v = 0.0;
    for (int nn = -s + 1; nn <= s; ++nn) v += mat[(mm + s - 1) * pitch + nn + s - 1] * u[i + nn];
    acc += a[i + mm] * v;
  }
  return acc;
}

/* interface i+1/2 at the order of cell `cell` (the cell it is differenced for) */
static double iface_bounded(const double* m8, const double* m6, const double* a, const double* u,
                            int n, int cell, int i) {
  const int d = cell < n - 1 - cell ? cell : n - 1 - cell; /* distance to the boundary */
  if (d >= 4) return iface(4, m8, 8, a, u, i);
  if (d == 3) return iface(3, m6, 8, a, u, i);
  if (d == 2) return iface(2, &M4B[0][0], 4, a, u, i);
  return 0.5 * (a[i] + a[i + 1]) * (u[i + 1] - u[i]); /* d == 1 */
}

/* (a u_x)_x with one-sided 2nd-order formulas at a boundary cell; dir = +1
 * at the left end (cells 0, 1, 2, 3), -1 at the right end (mirrored) */
static double diff_biased(const double* a, const double* u, int i, int dir, double dx) {
  const double* ua = u + i;
  const double* aa = a + i;
  const double ux = dir * (-3.0 * ua[0] + 4.0 * ua[dir] - ua[2 * dir]) / (2.0 * dx);
  const double ax = dir * (-3.0 * aa[0] + 4.0 * aa[dir] - aa[2 * dir]) / (2.0 * dx);
  const double uxx = (2.0 * ua[0] - 5.0 * ua[dir] + 4.0 * ua[2 * dir] - ua[3 * dir]) / (dx * dx);
  return aa[0] * uxx + ax * ux;
}

int or_apply_narrow_bounded(const double* m8, const double* m6, const double* a, const double* u,
                            int n, double dx, double* out) {
  if (n < 8 || !(dx > 0.0)) return 1;
  const double id2 = 1.0 / (dx * dx);
  for (int i = 0; i < n; ++i) {
    if (i == 0 || i == n - 1) {
      out[i] = diff_biased(a, u, i, i == 0 ? 1 : -1, dx);
      continue;
    }
    const double hr = iface_bounded(m8, m6, a, u, n, i, i);
    const double hl = iface_bounded(m8, m6, a, u, n, i, i - 1);
    out[i] = (hr - hl) * id2;
  }
  return 0;
}

int or_first_derivative_bounded(const double* u, int n, double dx, double* out) {
  if (n < 8 || !(dx > 0.0)) return 1;
  for (int i = 0; i < n; ++i) {
    const int d = i < n - 1 - i ? i : n - 1 - i;
    const int dir = i < n - 1 - i ? 1 : -1;
    const double* w = u + i;
    double v;
    if (d >= 4)
      v = C1 * (w[1] - w[-1]) + C2 * (w[2] - w[-2]) + C3 * (w[3] - w[-3]) + C4 * (w[4] - w[-4]);
    else if (d == 3)
      v = 0.75 * (w[1] - w[-1]) - 0.15 * (w[2] - w[-2]) + (1.0 / 60.0) * (w[3] - w[-3]);
    else if (d == 2)
      v = (2.0 / 3.0) * (w[1] - w[-1]) - (1.0 / 12.0) * (w[2] - w[-2]);
    else if (d == 1) /* biased 3rd order: (-2 u_{i-1} - 3 u_i + 6 u_{i+1} - u_{i+2}) / 6 */
      v = dir * (-2.0 * w[-dir] - 3.0 * w[0] + 6.0 * w[dir] - w[2 * dir]) / 6.0;
    else /* completely biased 3rd order: (-11 u_0 + 18 u_1 - 9 u_2 + 2 u_3) / 6 */
      v = dir * (-11.0 * w[0] + 18.0 * w[dir] - 9.0 * w[2 * dir] + 2.0 * w[3 * dir]) / 6.0;
    out[i] = v / dx;
  }
  return 0;
}
