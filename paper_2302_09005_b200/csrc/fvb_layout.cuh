// fvb_layout.cuh -- index maps of the batch arrays in HBM.
//
// AoS (the reference's PatchBatch layout, mesh.py:174-177): volume-major,
//   unknown fastest:  (patch * V + vol) * S + u
// SoA (LayoutEnumerator(SOA), mesh.py:129-130): one plane per unknown,
//   (u * N + patch) * V + vol
// Volumes linearise x fastest: vol = (z * E + y) * E + x (mesh.py:111-117).
#pragma once

#include <cstdint>

namespace fvb {

enum Layout : int { kAoS = 0, kSoA = 1 };

struct Geom {
  int d, p, s, e;       // dimensions, volumes per axis, unknowns, haloed extent p+2
  int64_t n;            // patches
  int64_t V, I;         // haloed / interior volumes per patch
};

__host__ __device__ inline Geom make_geom(int d, int p, int64_t n) {
  Geom g;
  g.d = d;
  g.p = p;
  g.s = d + 2;
  g.e = p + 2;
  g.n = n;
  g.V = d == 3 ? (int64_t)g.e * g.e * g.e : (int64_t)g.e * g.e;
  g.I = d == 3 ? (int64_t)p * p * p : (int64_t)p * p;
  return g;
}

__host__ __device__ inline int64_t elem_index(int layout, int64_t patch, int64_t vol, int u,
                                              int64_t n, int64_t vols, int s) {
  return layout == kAoS ? (patch * vols + vol) * s + u : ((int64_t)u * n + patch) * vols + vol;
}

}  // namespace fvb
