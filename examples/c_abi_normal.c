/* Pure-C consumer of the C ABI (no Python, no torch): builds a library-owned Cartesian plan
 * from a host trajectory, runs the sketched-style SENSE normal operator
 *   out = sum_c conj(m_c) F^H M F (m_c x)        (forward_model.py:168-180, linops.py:332-364)
 * on the GPU and checks it against a direct O(D^2) DFT on the CPU.  The normal operator of the
 * reference's centered unitary DFT pair only depends on the sampled frequencies f = points mod n:
 *   out[r] = sum_c conj(m_c[r]) / D sum_f e^{2 pi i f.(r - r')/n} sum_r' m_c[r'] x[r'].
 * Build: see examples/Makefile.  Exit code 0 = relative L2 error below 1e-4. */
#define _USE_MATH_DEFINES
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sketchrecon_b200.h"

#define NY 24
#define NX 20
#define NC 3
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static unsigned long long lcg = 12345;
static double urand(void) {
  lcg = lcg * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(lcg >> 11) / 9007199254740992.0;
}

int main(void) {
  const int D = NY * NX;
  /* trajectory: centered integer bins (ky, kx) in [-n/2, n/2), ~35 % sampled, plus duplicates */
  double* pts = malloc(sizeof(double) * 2 * (D + 16));
  int* fmask = calloc(D, sizeof(int));
  long long n = 0;
  for (int y = 0; y < NY; ++y)
    for (int x = 0; x < NX; ++x)
      if (urand() < 0.35) {
        pts[2 * n] = y - NY / 2;
        pts[2 * n + 1] = x - NX / 2;
        ++n;
      }
  for (int i = 0; i < 8 && i < n; ++i, ++n) {  /* duplicated bins */
    pts[2 * n] = pts[2 * i];
    pts[2 * n + 1] = pts[2 * i + 1];
  }
  for (long long i = 0; i < n; ++i) {
    const int fy = ((int)pts[2 * i] % NY + NY) % NY, fx = ((int)pts[2 * i + 1] % NX + NX) % NX;
    fmask[fy * NX + fx] = 1;
  }
  sr_c64* maps = malloc(sizeof(sr_c64) * NC * D);
  sr_c64* img = malloc(sizeof(sr_c64) * D);
  sr_c64* out = malloc(sizeof(sr_c64) * D);
  for (int i = 0; i < NC * D; ++i) { maps[i].x = (float)(urand() - 0.5); maps[i].y = (float)(urand() - 0.5); }
  for (int i = 0; i < D; ++i) { img[i].x = (float)(urand() - 0.5); img[i].y = (float)(urand() - 0.5); }

  /* GPU: plan + normal op through the C ABI */
  sr_cart_plan* plan = NULL;
  const int dims[2] = {NY, NX};
  const long long counts[1] = {n};
  int rc = sr_cart_plan_create(pts, counts, 1, 2, dims, 0, &plan, NULL);
  if (rc) { fprintf(stderr, "plan_create: %d\n", rc); return 2; }
  const long long wsb = sr_cart_plan_ws_bytes(plan, NC);
  sr_c64 *dmaps, *dimg, *dout;
  void* dws;
  cudaMalloc((void**)&dmaps, sizeof(sr_c64) * NC * D);
  cudaMalloc((void**)&dimg, sizeof(sr_c64) * D);
  cudaMalloc((void**)&dout, sizeof(sr_c64) * D);
  cudaMalloc(&dws, (size_t)wsb);
  cudaMemcpy(dmaps, maps, sizeof(sr_c64) * NC * D, cudaMemcpyHostToDevice);
  cudaMemcpy(dimg, img, sizeof(sr_c64) * D, cudaMemcpyHostToDevice);
  rc = sr_cart_plan_normal(plan, dimg, NULL, dmaps, (long long)NC * D, NC, dout, (sr_c64*)dws, NULL, NULL, NULL, NULL);
  if (rc) { fprintf(stderr, "plan_normal: %d\n", rc); return 2; }
  cudaMemcpy(out, dout, sizeof(sr_c64) * D, cudaMemcpyDeviceToHost);
  sr_cart_plan_destroy(plan);

  /* CPU reference, double precision */
  double err = 0.0, nrm = 0.0;
  double* kr = malloc(sizeof(double) * D);
  double* ki = malloc(sizeof(double) * D);
  double* acc = calloc(2 * D, sizeof(double));
  for (int c = 0; c < NC; ++c) {
    for (int f = 0; f < D; ++f) { /* forward DFT of m_c x at the sampled frequencies */
      kr[f] = ki[f] = 0.0;
      if (!fmask[f]) continue;
      const int fy = f / NX, fx = f % NX;
      for (int r = 0; r < D; ++r) {
        const int ry = r / NX, rx = r % NX;
        const sr_c64 m = maps[c * D + r], v = img[r];
        const double ur = (double)m.x * v.x - (double)m.y * v.y, ui = (double)m.x * v.y + (double)m.y * v.x;
        const double a = -2.0 * M_PI * ((double)fy * ry / NY + (double)fx * rx / NX);
        kr[f] += ur * cos(a) - ui * sin(a);
        ki[f] += ur * sin(a) + ui * cos(a);
      }
    }
    for (int r = 0; r < D; ++r) { /* inverse DFT, 1/D, conj(m_c) */
      const int ry = r / NX, rx = r % NX;
      double sr = 0.0, si = 0.0;
      for (int f = 0; f < D; ++f) {
        if (!fmask[f]) continue;
        const int fy = f / NX, fx = f % NX;
        const double a = 2.0 * M_PI * ((double)fy * ry / NY + (double)fx * rx / NX);
        sr += kr[f] * cos(a) - ki[f] * sin(a);
        si += kr[f] * sin(a) + ki[f] * cos(a);
      }
      sr /= D;
      si /= D;
      const sr_c64 m = maps[c * D + r];
      acc[2 * r] += m.x * sr + m.y * si;
      acc[2 * r + 1] += m.x * si - m.y * sr;
    }
  }
  for (int r = 0; r < D; ++r) {
    const double dr = out[r].x - acc[2 * r], di = out[r].y - acc[2 * r + 1];
    err += dr * dr + di * di;
    nrm += acc[2 * r] * acc[2 * r] + acc[2 * r + 1] * acc[2 * r + 1];
  }
  const double rel = sqrt(err / nrm);
  printf("c_abi_normal: %lld samples, %d coils, rel L2 vs CPU DFT %.3e\n", n, NC, rel);
  return rel < 1e-4 ? 0 : 1;
}
