/*
 * fvb_oracle.c -- TEST INFRASTRUCTURE ONLY (see fvb_oracle.h).
 *
 * Plain-C restatement of the reference's default engine, one patch at a time
 * (the patch-wise ordering, vectorized.run, vectorized.py:277-288), with the
 * same pass structure and the same floating-point operation order:
 *
 *   _pass_copy              vectorized.py:114-116
 *   _pass_fill_eigenvalues  vectorized.py:123-139  -> euler_max_eigenvalue pde.py:62-70
 *   _pass_dissipation       vectorized.py:161-180
 *   _pass_fill_fluxes       vectorized.py:142-158  -> euler_flux pde.py:45-59
 *   _pass_flux_accumulate   vectorized.py:183-200
 *   _pass_reduce            vectorized.py:226-231
 *
 * Build with -O2 -ffp-contract=off (no FMA contraction, no fast-math): every
 * + - * / sqrt is then one IEEE-754 binary64 round-to-nearest operation, which
 * is what numpy's elementwise ufuncs execute.  Patches run in parallel with
 * OpenMP (the reference parallelises over patch chunks with host threads,
 * vectorized.py:234-288).
 */
#include "fvb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* numpy.maximum: NaN-propagating (vectorized.py:178). */
static inline double np_maximum(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

/* euler_pressure, pde.py:33-42: (gamma-1) * (E - 0.5*mom2/rho), with
 * mom2 = q1*q1 (+ q2*q2 (+ q3*q3)) accumulated left to right. */
static inline double pressure(const double* q, int d, double g1) {
  double mom2 = q[1] * q[1];
  for (int a = 1; a < d; ++a) mom2 = mom2 + q[1 + a] * q[1 + a];
  return g1 * (q[d + 1] - (0.5 * mom2) / q[0]);
}

/* The quantity _locate_bad_state tests (vectorized.py:88-89); np.sum over
 * <= 3 elements is a sequential left-to-right sum of q*q. */
static inline double pressure_like(const double* q, int d) {
  double mom2 = q[1] * q[1];
  for (int a = 1; a < d; ++a) mom2 = mom2 + q[1 + a] * q[1 + a];
  return q[d + 1] - (0.5 * mom2) / q[0];
}

/* euler_max_eigenvalue, pde.py:62-70: |j_n/rho| + sqrt((gamma*p)/rho). */
static inline double max_eig(const double* q, int d, int n, double gamma, double g1) {
  double p = pressure(q, d, g1);
  double c = sqrt((gamma * p) / q[0]);
  return fabs(q[1 + n] / q[0]) + c;
}

/* euler_flux, pde.py:45-59. */
static inline void flux(const double* q, int d, int n, double g1, double* f) {
  double rho = q[0];
  double p = pressure(q, d, g1);
  double jn = q[1 + n];
  f[0] = jn;
  for (int a = 0; a < d; ++a) f[1 + a] = (jn * q[1 + a]) / rho;
  f[1 + n] = f[1 + n] + p;
  f[d + 1] = ((q[d + 1] + p) * jn) / rho;
}

typedef struct { int lo[3], hi[3]; } box_t;  /* haloed ranges per direction x,y,z */

/* vectorized._plan (vectorized.py:42-53): interior box, then per direction
 * the low and the high face slab (no edges / corners). */
static int make_boxes(int d, int p, box_t* boxes) {
  int nb = 0;
  box_t in;
  for (int a = 0; a < 3; ++a) { in.lo[a] = a < d ? 1 : 0; in.hi[a] = a < d ? p + 1 : 1; }
  boxes[nb++] = in;
  for (int n = 0; n < d; ++n) {
    box_t lo = in, hi = in;
    lo.lo[n] = 0; lo.hi[n] = 1;
    hi.lo[n] = p + 1; hi.hi[n] = p + 2;
    boxes[nb++] = lo;
    boxes[nb++] = hi;
  }
  return nb;
}

static inline int64_t vol_index(int d, int e, int x, int y, int z) {
  return d == 3 ? ((int64_t)z * e + y) * e + x : (int64_t)y * e + x;
}

/* One patch; returns 1 when a face-box volume triggers a NonPhysicalStateError. */
static int patch_update(int d, int p, double gamma, const double* q, double* out,
                        double cs0, double dtp, double* maxeig_out,
                        double* eig, double* flx) {
  const int s = d + 2, e = p + 2;
  const double g1 = gamma - 1.0; /* runtime, as pde.py:42 does */
  box_t boxes[7];
  const int nb = make_boxes(d, p, boxes);
  const int pz = d == 3 ? p : 1;

  /* _pass_copy */
  for (int z = 0; z < pz; ++z)
    for (int y = 0; y < p; ++y)
      for (int x = 0; x < p; ++x) {
        int64_t c = vol_index(d, p, x, y, z);
        int64_t v = vol_index(d, e, x + 1, y + 1, d == 3 ? z + 1 : 0);
        for (int u = 0; u < s; ++u) out[c * s + u] = q[v * s + u];
      }

  /* _pass_fill_eigenvalues with the euler_pressure / euler_max_eigenvalue
   * raise conditions evaluated box by box */
  for (int b = 0; b < nb; ++b) {
    const box_t* B = &boxes[b];
    int bad_rho = 0, bad_p = 0;
    for (int z = B->lo[2]; z < B->hi[2]; ++z)
      for (int y = B->lo[1]; y < B->hi[1]; ++y)
        for (int x = B->lo[0]; x < B->hi[0]; ++x) {
          const double* qv = q + vol_index(d, e, x, y, z) * s;
          if (qv[0] <= 0.0) bad_rho = 1;
          if (pressure(qv, d, g1) < 0.0) bad_p = 1;
        }
    if (bad_rho || bad_p) return 1;
    for (int z = B->lo[2]; z < B->hi[2]; ++z)
      for (int y = B->lo[1]; y < B->hi[1]; ++y)
        for (int x = B->lo[0]; x < B->hi[0]; ++x) {
          int64_t v = vol_index(d, e, x, y, z);
          for (int n = 0; n < d; ++n) eig[v * d + n] = max_eig(q + v * s, d, n, gamma, g1);
        }
  }

  const double dx = cs0 / (double)p;       /* vectorized.py:169 */
  const double inv = dtp / dx;             /* vectorized.py:170 */
  const double half_inv = 0.5 * inv;       /* `0.5 * inv * a` evaluates 0.5*inv first */

  /* _pass_dissipation: direction outer, shift (-1, +1) inner */
  for (int n = 0; n < d; ++n)
    for (int sh = -1; sh <= 1; sh += 2)
      for (int z = 0; z < pz; ++z)
        for (int y = 0; y < p; ++y)
          for (int x = 0; x < p; ++x) {
            int hc[3] = {x + 1, y + 1, d == 3 ? z + 1 : 0};
            int hn[3] = {hc[0], hc[1], hc[2]};
            hn[n] += sh;
            int64_t vc = vol_index(d, e, hc[0], hc[1], hc[2]);
            int64_t vn = vol_index(d, e, hn[0], hn[1], hn[2]);
            double a = np_maximum(eig[vn * d + n], eig[vc * d + n]);
            double coeff = half_inv * a;
            double* o = out + vol_index(d, p, x, y, z) * s;
            for (int u = 0; u < s; ++u) o[u] = o[u] + coeff * (q[vn * s + u] - q[vc * s + u]);
          }

  /* _pass_fill_fluxes over the same boxes */
  for (int b = 0; b < nb; ++b) {
    const box_t* B = &boxes[b];
    for (int z = B->lo[2]; z < B->hi[2]; ++z)
      for (int y = B->lo[1]; y < B->hi[1]; ++y)
        for (int x = B->lo[0]; x < B->hi[0]; ++x) {
          int64_t v = vol_index(d, e, x, y, z);
          for (int n = 0; n < d; ++n) flux(q + v * s, d, n, g1, flx + (v * d + n) * s);
        }
  }

  /* _pass_flux_accumulate */
  for (int n = 0; n < d; ++n)
    for (int z = 0; z < pz; ++z)
      for (int y = 0; y < p; ++y)
        for (int x = 0; x < p; ++x) {
          int hc[3] = {x + 1, y + 1, d == 3 ? z + 1 : 0};
          int hm[3] = {hc[0], hc[1], hc[2]}, hp[3] = {hc[0], hc[1], hc[2]};
          hm[n] -= 1; hp[n] += 1;
          const double* fc = flx + (vol_index(d, e, hc[0], hc[1], hc[2]) * d + n) * s;
          const double* fm = flx + (vol_index(d, e, hm[0], hm[1], hm[2]) * d + n) * s;
          const double* fp = flx + (vol_index(d, e, hp[0], hp[1], hp[2]) * d + n) * s;
          double* o = out + vol_index(d, p, x, y, z) * s;
          for (int u = 0; u < s; ++u) {
            double favg_m = 0.5 * (fm[u] + fc[u]);
            double favg_p = 0.5 * (fc[u] + fp[u]);
            o[u] = o[u] + inv * (favg_m - favg_p);
          }
        }

  /* _pass_reduce: numpy max over interior volumes x directions (NaN wins) */
  double m = -INFINITY;
  int first = 1;
  for (int z = 0; z < pz; ++z)
    for (int y = 0; y < p; ++y)
      for (int x = 0; x < p; ++x) {
        int64_t v = vol_index(d, e, x + 1, y + 1, d == 3 ? z + 1 : 0);
        for (int n = 0; n < d; ++n) {
          double l = eig[v * d + n];
          if (first) { m = l; first = 0; }
          else m = np_maximum(m, l);
        }
      }
  *maxeig_out = m;
  return 0;
}

static int thread_count(int nthreads) {
#ifdef _OPENMP
  return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}

int fvb_oracle_update(int dim, int p, int64_t n, double gamma,
                      const double* qin, double* qout,
                      const double* cell_size, const double* dt,
                      double* max_eig, int nthreads) {
  if ((dim != 2 && dim != 3) || p < 1 || n < 0) return 1;
  const int d = dim, s = d + 2, e = p + 2;
  const int64_t V = d == 3 ? (int64_t)e * e * e : (int64_t)e * e;
  const int64_t I = d == 3 ? (int64_t)p * p * p : (int64_t)p * p;
  int bad = 0;
  const int nt = thread_count(nthreads);
#pragma omp parallel num_threads(nt) reduction(| : bad)
  {
    double* eig = (double*)malloc(sizeof(double) * V * d);
    double* flx = (double*)malloc(sizeof(double) * V * d * s);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      bad |= patch_update(d, p, gamma, qin + i * V * s, qout + i * I * s,
                          cell_size[i * d], dt[i], &max_eig[i], eig, flx);
    }
    free(eig);
    free(flx);
  }
  return bad ? 2 : 0;
}

int fvb_oracle_locate(int dim, int p, int64_t n, double gamma,
                      const double* qin, fvb_oracle_boxinfo* info, int nthreads) {
  if ((dim != 2 && dim != 3) || p < 1 || n < 0) return 1;
  const int d = dim, s = d + 2, e = p + 2, nbox = 2 * d + 1;
  const int64_t V = d == 3 ? (int64_t)e * e * e : (int64_t)e * e;
  const double g1 = gamma - 1.0;
  box_t boxes[7];
  make_boxes(d, p, boxes);
  const int nt = thread_count(nthreads);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* q = qin + i * V * s;
    for (int b = 0; b < nbox; ++b) {
      const box_t* B = &boxes[b];
      fvb_oracle_boxinfo r = {0, 0, -1, -1};
      int64_t lin = 0;
      for (int z = B->lo[2]; z < B->hi[2]; ++z)
        for (int y = B->lo[1]; y < B->hi[1]; ++y)
          for (int x = B->lo[0]; x < B->hi[0]; ++x, ++lin) {
            const double* qv = q + vol_index(d, e, x, y, z) * s;
            if (qv[0] <= 0.0) r.trig_rho = 1;
            if (pressure(qv, d, g1) < 0.0) r.trig_p = 1;
            if (r.first_nonpos < 0 && !(qv[0] > 0.0)) r.first_nonpos = lin;
            if (r.first_badpl < 0 && !(pressure_like(qv, d) >= 0.0)) r.first_badpl = lin;
          }
      info[i * nbox + b] = r;
    }
  }
  return 0;
}

/* Chunk bounds of vectorized._patch_chunks (vectorized.py:234-243). */
static void chunk_bounds(int64_t n, int64_t chunks, int64_t k, int64_t* lo, int64_t* hi) {
  int64_t base = n / chunks, extra = n % chunks;
  int64_t start = k * base + (k < extra ? k : extra);
  *lo = start;
  *hi = start + base + (k < extra ? 1 : 0);
}

int fvb_oracle_first_error(int dim, int p, int64_t n,
                           const fvb_oracle_boxinfo* info, int ordering,
                           int64_t nchunks, int64_t* patch, int* box,
                           int64_t* lin, int* kind) {
  (void)p;
  const int nbox = 2 * dim + 1;
  if (n <= 0) return 0;
  if (ordering == 0) {
    /* patch-wise: patches in order (futures are joined in submission
     * order, vectorized.py:283-288), boxes in order inside a patch */
    for (int64_t i = 0; i < n; ++i)
      for (int b = 0; b < nbox; ++b) {
        const fvb_oracle_boxinfo* r = &info[i * nbox + b];
        if (r->trig_rho || r->trig_p) {
          *patch = i; *box = b; *kind = r->trig_rho ? 1 : 2;
          *lin = r->first_nonpos >= 0 ? r->first_nonpos : r->first_badpl;
          return 1;
        }
      }
    return 0;
  }
  /* batched: chunks in order (launch() joins futures in order,
   * vectorized.py:263-265); inside a chunk, box by box over the whole chunk */
  int64_t chunks = nchunks < 1 ? 1 : (nchunks > n ? n : nchunks);
  for (int64_t k = 0; k < chunks; ++k) {
    int64_t lo, hi;
    chunk_bounds(n, chunks, k, &lo, &hi);
    for (int b = 0; b < nbox; ++b) {
      int any_rho = 0, any_p = 0;
      for (int64_t i = lo; i < hi; ++i) {
        any_rho |= (int)info[i * nbox + b].trig_rho;
        any_p |= (int)info[i * nbox + b].trig_p;
      }
      if (!(any_rho || any_p)) continue;
      *box = b;
      *kind = any_rho ? 1 : 2;
      for (int64_t i = lo; i < hi; ++i)
        if (info[i * nbox + b].first_nonpos >= 0) {
          *patch = i; *lin = info[i * nbox + b].first_nonpos; return 1;
        }
      for (int64_t i = lo; i < hi; ++i)
        if (info[i * nbox + b].first_badpl >= 0) {
          *patch = i; *lin = info[i * nbox + b].first_badpl; return 1;
        }
      *patch = lo; *lin = -1;  /* unreachable for consistent info */
      return 1;
    }
  }
  return 0;
}
