// Total-variation pieces of the PDHG sub-solver (l1-tv regulariser).
//
// Reference: FiniteDiffOp (circular forward differences stacked over axes),
//   /root/reference/pkg/src/sketchrecon/linops.py:717-741
// _clamp_magnitude  solvers.py:138-142;  pdhg  solvers.py:315-362;
// the sub-problem's K = D, prox_dual = clamp, prox_data = inner CG
//   coil_sketch.py:200-216.
//
// Layout: images (B, n0, n1, n2) (leading 1s for 2-D / 1-D), dual variables
// (B, ndim, D) -- axis-major like the reference's concatenation.  Each kernel
// is one pass over HBM: the dual step reads z and p and writes p, the primal
// step reads x and the ndim dual planes and writes v.
#include "common.cuh"

namespace {

struct TvGeom {
  int n[3];  // dims padded with leading 1s to 3-D
  int ndim;  // active axes (the last ndim of n)
  long long D;
};

// neighbour of cell (i0, i1, i2) along active axis a (0 = first active), shift +1 or -1
__device__ __forceinline__ long long tv_nb(const TvGeom& g, int i0, int i1, int i2, int a, int s) {
  const int ax = 3 - g.ndim + a;
  int i[3] = {i0, i1, i2};
  i[ax] += s;
  if (i[ax] >= g.n[ax]) i[ax] -= g.n[ax];
  if (i[ax] < 0) i[ax] += g.n[ax];
  return ((long long)i[0] * g.n[1] + i[1]) * g.n[2] + i[2];
}

__device__ __forceinline__ float2 clamp_mag(float2 v, float r) {
  const float m2 = v.x * v.x + v.y * v.y;
  if (m2 > r * r) {
    const float f = r * rsqrtf(m2);
    return make_float2(v.x * f, v.y * f);
  }
  return v;
}

// p[a] = clamp(p[a] + sigma * (z[i + e_a] - z[i]), lam)   (mode 0)
// out[a] = z[i + e_a] - z[i]                               (mode 1: plain forward differences)
__global__ void k_tv_dual(float2* __restrict__ p, const float2* __restrict__ z, TvGeom g, int mode,
                          const float* __restrict__ sigma, float lam, int batch) {
  const long long total = g.D * batch;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / g.D);
    const long long i = e - (long long)b * g.D;
    const int i2 = (int)(i % g.n[2]);
    const long long t = i / g.n[2];
    const int i1 = (int)(t % g.n[1]), i0 = (int)(t / g.n[1]);
    const float2* zb = z + (long long)b * g.D;
    const float2 zc = zb[i];
    for (int a = 0; a < g.ndim; ++a) {
      const float2 zn = zb[tv_nb(g, i0, i1, i2, a, +1)];
      const float2 dz = make_float2(zn.x - zc.x, zn.y - zc.y);
      float2* pp = p + ((long long)b * g.ndim + a) * g.D + i;
      if (mode == 1) {
        *pp = dz;
      } else {
        const float s = sigma[b];
        const float2 q = *pp;
        *pp = clamp_mag(make_float2(fmaf(s, dz.x, q.x), fmaf(s, dz.y, q.y)), lam);
      }
    }
  }
}

// v = x - tau * sum_a (p[a][i - e_a] - p[a][i])
__global__ void k_tv_primal(float2* __restrict__ v, const float2* __restrict__ x, const float2* __restrict__ p,
                            TvGeom g, const float* __restrict__ tau, int batch) {
  const long long total = g.D * batch;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / g.D);
    const long long i = e - (long long)b * g.D;
    const int i2 = (int)(i % g.n[2]);
    const long long t = i / g.n[2];
    const int i1 = (int)(t % g.n[1]), i0 = (int)(t / g.n[1]);
    float2 acc = make_float2(0.f, 0.f);
    for (int a = 0; a < g.ndim; ++a) {
      const float2* pa = p + ((long long)b * g.ndim + a) * g.D;
      const float2 pm = pa[tv_nb(g, i0, i1, i2, a, -1)], pc = pa[i];
      acc.x += pm.x - pc.x;
      acc.y += pm.y - pc.y;
    }
    const float tb = tau[b];
    const float2 xv = x[e];
    v[e] = make_float2(fmaf(-tb, acc.x, xv.x), fmaf(-tb, acc.y, xv.y));
  }
}

bool make_tv_geom(const int* dims, int ndim, TvGeom& g) {
  if (ndim < 1 || ndim > 3) return false;
  g.n[0] = g.n[1] = g.n[2] = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return false;
    g.n[3 - ndim + a] = dims[a];
  }
  g.ndim = ndim;
  g.D = (long long)g.n[0] * g.n[1] * g.n[2];
  return true;
}

}  // namespace

extern "C" {

int sr_tv_dual(sr_c64* p, const sr_c64* z, const int* dims, int ndim, int mode, const float* sigma, float lam,
               int batch, void* stream) {
  TvGeom g;
  if (!make_tv_geom(dims, ndim, g) || batch < 1 || mode < 0 || mode > 1 || (mode == 0 && !sigma))
    return SR_EINVAL;
  k_tv_dual<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((float2*)p, (const float2*)z, g, mode, sigma, lam, batch);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_tv_primal(sr_c64* v, const sr_c64* x, const sr_c64* p, const int* dims, int ndim, const float* tau,
                 int batch, void* stream) {
  TvGeom g;
  if (!make_tv_geom(dims, ndim, g) || batch < 1 || !tau) return SR_EINVAL;
  k_tv_primal<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((float2*)v, (const float2*)x, (const float2*)p, g, tau,
                                                        batch);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // extern "C"
