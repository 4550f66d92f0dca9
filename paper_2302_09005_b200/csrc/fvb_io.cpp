// fvb_io.cpp -- FVB1 batch files on the C side.
//
// Byte-compatible with the reference's fixture dumps (save_batch / load_batch,
// mesh.py:313-353): the 4-byte magic "FVB1", the header (d, p, s, N) as four
// little-endian int64, then seven little-endian float64 arrays in PatchBatch
// order -- QIn (N*(p+2)^d*s), QOut (N*p^d*s), cell_centre (N*d), cell_size
// (N*d), t (N), dt (N), max_eigenvalue (N).  Lets golden vectors travel between
// the CPU oracle and the GPU box without Python.  Host code only (x86-64 is
// little-endian, so the arrays are written as they lie in memory).
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/fvb200.h"

namespace {

const char kMagic[4] = {'F', 'V', 'B', '1'};

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// element counts of the seven arrays
void counts(const int64_t h[4], int64_t c[7]) {
  const int64_t d = h[0], p = h[1], s = h[2], n = h[3];
  c[0] = n * ipow(p + 2, (int)d) * s;
  c[1] = n * ipow(p, (int)d) * s;
  c[2] = n * d;
  c[3] = n * d;
  c[4] = c[5] = c[6] = n;
}

bool header_ok(const int64_t h[4]) {
  return (h[0] == 2 || h[0] == 3) && h[1] >= 1 && h[1] <= 4096 && h[2] >= 1 && h[2] <= 64 && h[3] >= 0;
}

}  // namespace

extern "C" {

int fvb_fvb1_header(const char* path, int64_t* header) {
  if (!path || !header) return FVB_ERR_CONTRACT;
  FILE* f = fopen(path, "rb");
  if (!f) return FVB_ERR_IO;
  char magic[4];
  int64_t h[4];
  const bool ok = fread(magic, 1, 4, f) == 4 && memcmp(magic, kMagic, 4) == 0 && fread(h, 8, 4, f) == 4;
  fclose(f);
  if (!ok || !header_ok(h)) return FVB_ERR_CONTRACT;
  memcpy(header, h, sizeof(h));
  return FVB_OK;
}

int fvb_fvb1_read(const char* path, const int64_t* header, double* qin, double* qout, double* cell_centre,
                  double* cell_size, double* t, double* dt, double* max_eig) {
  int64_t h[4];
  int rc = fvb_fvb1_header(path, h);
  if (rc) return rc;
  if (!header || memcmp(h, header, sizeof(h)) != 0) return FVB_ERR_CONTRACT;   // caller sized for another batch
  double* dst[7] = {qin, qout, cell_centre, cell_size, t, dt, max_eig};
  int64_t c[7];
  counts(h, c);
  FILE* f = fopen(path, "rb");
  if (!f) return FVB_ERR_IO;
  bool ok = fseek(f, 36, SEEK_SET) == 0;
  for (int k = 0; k < 7 && ok; ++k) {
    if (!dst[k]) ok = fseek(f, (long)(c[k] * 8), SEEK_CUR) == 0;   // NULL: skip the array
    else ok = fread(dst[k], 8, (size_t)c[k], f) == (size_t)c[k];
  }
  fclose(f);
  return ok ? FVB_OK : FVB_ERR_IO;
}

int fvb_fvb1_write(const char* path, const int64_t* header, const double* qin, const double* qout,
                   const double* cell_centre, const double* cell_size, const double* t, const double* dt,
                   const double* max_eig) {
  if (!path || !header || !header_ok(header)) return FVB_ERR_CONTRACT;
  const double* src[7] = {qin, qout, cell_centre, cell_size, t, dt, max_eig};
  for (int k = 0; k < 7; ++k)
    if (!src[k] && header[3] > 0) return FVB_ERR_CONTRACT;
  int64_t c[7];
  counts(header, c);
  FILE* f = fopen(path, "wb");
  if (!f) return FVB_ERR_IO;
  bool ok = fwrite(kMagic, 1, 4, f) == 4 && fwrite(header, 8, 4, f) == 4;
  for (int k = 0; k < 7 && ok; ++k) ok = fwrite(src[k], 8, (size_t)c[k], f) == (size_t)c[k];
  ok = (fclose(f) == 0) && ok;
  return ok ? FVB_OK : FVB_ERR_IO;
}

}  // extern "C"
