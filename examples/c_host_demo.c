/* c_host_demo.c -- the drop-in boundary from a plain C host (no Python, no torch):
 * one Rusanov step of a random 3D p = 16 batch (and a 2D p = 17 one) through
 * libfvb200.so's host pipeline (fvb_update_host: chunked H2D, fused kernel, D2H),
 * checked bit for bit against the CPU oracle (test infrastructure, oracle/).
 *
 *   make -C examples && ./examples/c_host_demo
 */
#include <cuda_runtime_api.h>
#include <inttypes.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fvb200.h"
#include "fvb_oracle.h"

static uint64_t rng = 88172645463325252ull;
static double uniform(double lo, double hi) {   /* xorshift64 */
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return lo + (hi - lo) * (double)(rng >> 11) * (1.0 / 9007199254740992.0);
}

static int run(int dim, int p, int64_t n) {
  const int s = dim + 2, e = p + 2;
  const int64_t V = dim == 3 ? (int64_t)e * e * e : (int64_t)e * e;
  const int64_t I = dim == 3 ? (int64_t)p * p * p : (int64_t)p * p;
  const double gamma = 1.4;
  double* qin = malloc(sizeof(double) * n * V * s);
  double* qout = malloc(sizeof(double) * n * I * s);
  double* ref = malloc(sizeof(double) * n * I * s);
  double* cs = malloc(sizeof(double) * n * dim);
  double* dt = malloc(sizeof(double) * n);
  double* lam = malloc(sizeof(double) * n);
  double* lam_ref = malloc(sizeof(double) * n);
  for (int64_t v = 0; v < n * V; ++v) {   /* admissible states */
    const double rho = uniform(0.5, 2.0), pr = uniform(0.5, 2.0);
    double ke = 0.0;
    qin[v * s] = rho;
    for (int a = 0; a < dim; ++a) {
      const double u = uniform(-1.0, 1.0);
      qin[v * s + 1 + a] = rho * u;
      ke += u * u;
    }
    qin[v * s + s - 1] = pr / (gamma - 1.0) + 0.5 * rho * ke;
  }
  for (int64_t i = 0; i < n * dim; ++i) cs[i] = 1.0;
  for (int64_t i = 0; i < n; ++i) dt[i] = 0.4 * (1.0 / p) / 3.4;

  fvb_spec spec = {dim, p, s, 0, n, gamma};
  const int64_t chunk = n < 32 ? n : n / 8;
  const size_t ws_bytes = fvb_update_host_workspace(&spec, chunk);
  void* ws = NULL;
  if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  int rc = fvb_update_host(&spec, qin, qout, cs, dt, lam, ws, ws_bytes, chunk, FVB_KERNEL_AUTO, NULL);
  if (rc != FVB_OK) {
    fprintf(stderr, "fvb_update_host: %s\n", fvb_strerror(rc));
    return 1;
  }
  rc = fvb_oracle_update(dim, p, n, gamma, qin, ref, cs, dt, lam_ref, 0);
  int64_t diff = 0;
  for (int64_t i = 0; i < n * I * s; ++i) diff += memcmp(&qout[i], &ref[i], sizeof(double)) != 0;
  for (int64_t i = 0; i < n; ++i) diff += memcmp(&lam[i], &lam_ref[i], sizeof(double)) != 0;
  printf("%dD p=%d N=%" PRId64 " (%s kernel): %s (%" PRId64 " differing words)\n", dim, p, n,
         fvb_select_kernel(&spec) == FVB_KERNEL_FUSED ? "fused" : "generic",
         (rc == 0 && diff == 0) ? "bit-identical to the oracle" : "MISMATCH", diff);
  cudaFree(ws);
  free(qin); free(qout); free(ref); free(cs); free(dt); free(lam); free(lam_ref);
  return (rc == 0 && diff == 0) ? 0 : 1;
}

int main(void) {
  int bad = run(3, 16, 96);
  bad |= run(2, 17, 500);
  return bad;
}
