// K3/K4: Kaiser-Bessel gridded NUFFT SENSE operator (2-D and 3-D), B200.
//
// Reference: _GriddedNUFFTKernel (/root/reference/pkg/src/sketchrecon/linops.py:424-516),
// _kb_kernel / _kb_apodization (linops.py:404-421), with density weights applied
// as sqrt(w) on both sides by SenseOperator (forward_model.py:168-180).
//
// Shift-free formulation: the image pixel with centered
// coordinate r sits at oversampled index r mod g, the spectrum is the plain
// (uncentered) unnormalised DFT, and tap `col` reads bin col mod g; the
// reference's ifftshift / embed / fftshift are pure index arithmetic.
//   forward : y_i = sqrt(w_i) / sqrt(D) * sum_taps KB * DFT(embed(c x / apod))[taps]
//   adjoint : x  = 1/sqrt(D) / apod * crop(IDFT(spread(sqrt(w) y)))
//   normal  : sum_j conj(c_j) 1/D / apod crop IDFT spread(w * interp(DFT embed(c_j x / apod)))
// Grids are (C, g0, g1, g2) complex64 (2-D: g0 = 1); FFTs run per axis with the
// same two-level register FFT as the Cartesian path (perm order per axis).
//
// Interpolation weights are evaluated on the fly from fp64-derived tap bases
// (int) and fp32 offsets t = u - base: KB(t - k) = I0(beta sqrt(1 - (2(t-k)/w)^2))
// for |t - k| < w/2, exactly 0 otherwise (the reference's edge discontinuity),
// with I0 from the Abramowitz-Stegun 9.8.1/9.8.2 rational fits (|rel err| < 2e-7).
// Spreading uses float2 vector atomics (red.global.add.v2.f32): results are
// reproducible to fp32 rounding, not bit-identical across runs.
#include "fft2step.cuh"

namespace {

// ----------------------------------------------------------------- FFT along an axis
template <int P, int Q>
struct AxCfg {
  static constexpr int BASE = 32 / (P % 32 == 0 ? 32 : (P % 16 == 0 ? 16 : (P % 8 == 0 ? 8 : (P % 4 == 0 ? 4 : (P % 2 == 0 ? 2 : 1)))));
  static constexpr int ROWS0 = BASE * ((128 / (BASE * P)) > 1 ? (128 / (BASE * P)) : 1);
  static constexpr int ROWS = ROWS0 > 64 ? 64 : ROWS0;
  static constexpr int T = ROWS * P;
  static constexpr int CB = (P >= 16) ? 16 : (P >= 4 ? 32 : 64);
  static constexpr int TS = CB * P;
  static constexpr int VSP = FftShape<P, Q>::VS0 | 1;
};

// contiguous rows of length N: fwd natural -> perm, inv perm -> natural (in place, unnormalised)
template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::T)
k_fft_rows(float2* __restrict__ data, long long nrows, int inv) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, ROWS = A::ROWS, T = A::T;
  extern __shared__ __align__(16) float2 dsm[];
  float2* tw = dsm;
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long row0 = (long long)blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  const bool valid = row0 + lr < nrows;
  const int nvalid = (int)min((long long)ROWS, nrows - row0) * N;
  float2* base = data + row0 * N;
  if (inv) init_tw_s2<P, Q>(tw, tid, T); else init_tw_s1<P, Q>(tw, tid, T);
  if (!inv) {
    __syncthreads();
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = valid ? base[(long long)lr * N + p + P * q] : make_float2(0.f, 0.f);
    fft_s1_fwd<P, Q>(r, p, tw);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[lr * S::VS + S::GS * k2 + p] = r[k2];
    __syncthreads();
    if (P > 1) {
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        float2 g[P];
        float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
        fft_s2_fwd<P>(g);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
      }
      __syncthreads();
    }
    for (int e = tid; e < nvalid; e += T) {
      const int l3 = e / N, pos = e - l3 * N;
      base[e] = buf[l3 * S::VS + S::pad(pos)];
    }
  } else {
    for (int e = tid; e < nvalid; e += T) {
      const int l3 = e / N, pos = e - l3 * N;
      buf[l3 * S::VS + S::pad(pos)] = base[e];
    }
    __syncthreads();
    if (P > 1) {
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        float2 g[P];
        float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
        fft_s2_inv<P, Q>(g, k2, tw);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
      }
      __syncthreads();
    }
    float2 r[Q];
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[lr * S::VS + S::GS * k2 + p];
    fft_s1_inv<Q>(r);
    if (valid) {
#pragma unroll
      for (int q = 0; q < Q; ++q) base[(long long)lr * N + p + P * q] = r[q];
    }
  }
}

// strided axis of [outer][N][inner]: CTA = CB consecutive inner indices of one outer
template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::TS)
k_fft_strided(float2* __restrict__ data, long long inner, int inv) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, CB = A::CB, T = A::TS, VSP = A::VSP;
  extern __shared__ __align__(16) float2 dsm[];
  float2* tw = dsm;
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long c0 = (long long)blockIdx.x * CB;
  const long long o = blockIdx.y;
  float2* img = data + o * N * inner;
  const int ncols = (int)min((long long)CB, inner - c0);
  const int c = tid % CB, p = tid / CB;
  const bool cvalid = c < ncols;
  if (inv) init_tw_s2<P, Q>(tw, tid, T); else init_tw_s1<P, Q>(tw, tid, T);
  __syncthreads();
  if (!inv) {
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = cvalid ? img[(long long)(p + P * q) * inner + c0 + c] : make_float2(0.f, 0.f);
    fft_s1_fwd<P, Q>(r, p, tw);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[c * VSP + S::GS * k2 + p] = r[k2];
    __syncthreads();
    for (int it = tid; it < CB * Q; it += T) {
      const int cc = it % CB, k2 = it / CB;
      if (cc >= ncols || P == 1) continue;
      float2 g[P];
      float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
      fft_s2_fwd<P>(g);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
    }
    __syncthreads();
    for (int e = tid; e < CB * N; e += T) {
      const int cc = e % CB, pos = e / CB;
      if (cc < ncols) img[(long long)pos * inner + c0 + cc] = buf[cc * VSP + S::pad(pos)];
    }
  } else {
    for (int e = tid; e < CB * N; e += T) {
      const int cc = e % CB, pos = e / CB;
      if (cc < ncols) buf[cc * VSP + S::pad(pos)] = img[(long long)pos * inner + c0 + cc];
    }
    __syncthreads();
    for (int it = tid; it < CB * Q; it += T) {
      const int cc = it % CB, k2 = it / CB;
      if (cc >= ncols || P == 1) continue;
      float2 g[P];
      float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
      fft_s2_inv<P, Q>(g, k2, tw);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
    }
    __syncthreads();
    float2 r[Q];
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[c * VSP + S::GS * k2 + p];
    fft_s1_inv<Q>(r);
    if (cvalid) {
#pragma unroll
      for (int q = 0; q < Q; ++q) img[(long long)(p + P * q) * inner + c0 + c] = r[q];
    }
  }
}

template <int P, int Q>
int launch_rows(float2* data, long long nrows, int inv, cudaStream_t st) {
  using A = AxCfg<P, Q>;
  using S = FftShape<P, Q>;
  const size_t smem = sizeof(float2) * (S::N + A::ROWS * S::VS);
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(k_fft_rows<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SR_ECUDA;
    cfg = true;
  }
  const long long nb = (nrows + A::ROWS - 1) / A::ROWS;
  if (nb > 0x7fffffffLL) return SR_EINVAL;
  k_fft_rows<P, Q><<<(unsigned)nb, A::T, smem, st>>>(data, nrows, inv);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

template <int P, int Q>
int launch_strided(float2* data, long long outer, long long inner, int inv, cudaStream_t st) {
  using A = AxCfg<P, Q>;
  using S = FftShape<P, Q>;
  const size_t smem = sizeof(float2) * (S::N + A::CB * A::VSP);
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(k_fft_strided<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SR_ECUDA;
    cfg = true;
  }
  if (outer > 65535) return SR_EINVAL;
  dim3 grid((unsigned)((inner + A::CB - 1) / A::CB), (unsigned)outer);
  k_fft_strided<P, Q><<<grid, A::TS, smem, st>>>(data, inner, inv);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int fft_axis(float2* data, long long outer, int n, long long inner, int inv, cudaStream_t st) {
  if (n == 1) return SR_OK;
  if (inner == 1) {
    switch (n) {
#define X(N_, P_, Q_) case N_: return launch_rows<P_, Q_>(data, outer, inv, st);
      SR_FFT_SIZES(X)
#undef X
      default: return SR_EUNSUPPORTED;
    }
  }
  switch (n) {
#define X(N_, P_, Q_) case N_: return launch_strided<P_, Q_>(data, outer, inner, inv, st);
    SR_FFT_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

// ----------------------------------------------------------------- geometry
struct NufftGeom {
  int n[3];      // image dims (leading 1 for 2-D)
  int g[3];      // oversampled dims
  int P[3], Q[3];  // FFT split per axis (perm order)
  float beta[3];
  int width;
  long long D, G;
};

__device__ __forceinline__ float bessel_i0f(float x) {
  // Abramowitz & Stegun 9.8.1 / 9.8.2
  const float ax = fabsf(x);
  if (ax < 3.75f) {
    const float t = (x / 3.75f) * (x / 3.75f);
    return 1.0f + t * (3.5156229f + t * (3.0899424f + t * (1.2067492f + t * (0.2659732f + t * (0.0360768f + t * 0.0045813f)))));
  }
  const float t = 3.75f / ax;
  const float pol = 0.39894228f + t * (0.01328592f + t * (0.00225319f + t * (-0.00157565f + t * (0.00916281f +
                    t * (-0.02057706f + t * (0.02635537f + t * (-0.01647633f + t * 0.00392377f)))))));
  return pol * (expf(ax) * rsqrtf(ax));
}

__device__ __forceinline__ float kb_weight(float u, float beta, float w) {
  const float a = 2.0f * u / w;
  const float arg = 1.0f - a * a;
  return arg > 0.f ? bessel_i0f(beta * sqrtf(arg)) : 0.f;
}

__device__ __forceinline__ int perm_of(int k, int P, int Q) { return P * (k % Q) + k / Q; }

constexpr int MAXW = 8;

// tap table of one sample: spectrum offsets and weights per axis
struct Taps {
  int off[3][MAXW];
  float wt[3][MAXW];
};

__device__ __forceinline__ void sample_taps(const NufftGeom& g, const int* __restrict__ base,
                                            const float* __restrict__ frac, long long i, long long N,
                                            Taps& tp) {
  const long long stride[3] = {(long long)g.g[1] * g.g[2], (long long)g.g[2], 1};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (g.n[a] == 1) {
      tp.off[a][0] = 0;
      tp.wt[a][0] = 1.f;
      for (int k = 1; k < MAXW; ++k) { tp.off[a][k] = 0; tp.wt[a][k] = 0.f; }
      continue;
    }
    const int b = base[a * N + i];
    const float t = frac[a * N + i];
    for (int k = 0; k < MAXW; ++k) {
      if (k < g.width) {
        int col = (b + k) % g.g[a];
        if (col < 0) col += g.g[a];
        tp.off[a][k] = (int)(perm_of(col, g.P[a], g.Q[a]) * stride[a]);
        tp.wt[a][k] = kb_weight(t - (float)k, g.beta[a], (float)g.width);
      } else {
        tp.off[a][k] = 0;
        tp.wt[a][k] = 0.f;
      }
    }
  }
}

// shared-memory float2 accumulate: one 64-bit CAS per update (no native shared FADD)
__device__ __forceinline__ void smem_add_f2(float2* p, float2 v) {
  unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
  unsigned long long old = *q, assumed;
  do {
    assumed = old;
    float2 cur = *reinterpret_cast<float2*>(&assumed);
    cur.x += v.x;
    cur.y += v.y;
    old = atomicCAS(q, assumed, *reinterpret_cast<unsigned long long*>(&cur));
  } while (old != assumed);
}

__device__ __forceinline__ void red_add_f2(float2* p, float2 v) {
  atomicAdd(p, v);  // sm_90+: vector float2 atomic add
}

// ----------------------------------------------------------------- kernels
// grid[j][cell] = embed(c_j x / apod) (zero outside the image); batch = 1
__global__ void k_nufft_embed(const float2* __restrict__ x, const float2* __restrict__ maps,
                              const float* __restrict__ ia0, const float* __restrict__ ia1,
                              const float* __restrict__ ia2, float2* __restrict__ grid, NufftGeom g,
                              int ncoils, const float2* __restrict__ anchor) {
  const long long G = g.G;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < G * ncoils;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / G);
    const long long cell = e - (long long)j * G;
    const int k2 = (int)(cell % g.g[2]);
    const long long t1 = cell / g.g[2];
    const int k1 = (int)(t1 % g.g[1]);
    const int k0 = (int)(t1 / g.g[1]);
    int idx[3];
    const int k[3] = {k0, k1, k2};
    bool inside = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int n = g.n[a], h = n / 2;
      int r;
      if (k[a] < n - h) r = k[a];
      else if (k[a] >= g.g[a] - h) r = k[a] - g.g[a];
      else { inside = false; r = 0; }
      idx[a] = r + h;
    }
    float2 v = make_float2(0.f, 0.f);
    if (inside) {
      const long long pix = ((long long)idx[0] * g.n[1] + idx[1]) * g.n[2] + idx[2];
      float2 xv = x[pix];
      if (anchor) xv = csub(xv, anchor[pix]);
      const float s = ia0[idx[0]] * ia1[idx[1]] * ia2[idx[2]];
      v = cscale(cmul(maps[(long long)j * g.D + pix], xv), s);
    }
    grid[e] = v;
  }
}

// out = e( sum_j conj(c_j) * crop(grid_j) / apod * scale )
__global__ void k_nufft_crop(const float2* __restrict__ grid, const float2* __restrict__ maps,
                             const float* __restrict__ ia0, const float* __restrict__ ia1,
                             const float* __restrict__ ia2, float2* __restrict__ out, NufftGeom g,
                             int ncoils, float scale, const float4* __restrict__ coef,
                             const float2* __restrict__ u, const float2* __restrict__ d) {
  for (long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x; pix < g.D;
       pix += (long long)gridDim.x * blockDim.x) {
    const int i2 = (int)(pix % g.n[2]);
    const long long t1 = pix / g.n[2];
    const int i1 = (int)(t1 % g.n[1]);
    const int i0 = (int)(t1 / g.n[1]);
    const int ii[3] = {i0, i1, i2};
    long long cell = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int r = ii[a] - g.n[a] / 2;
      if (r < 0) r += g.g[a];
      cell = cell * g.g[a] + r;
    }
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < ncoils; ++j) cfma_conj(acc, maps[(long long)j * g.D + pix], grid[(long long)j * g.G + cell]);
    const float s = ia0[i0] * ia1[i1] * ia2[i2] * scale;
    acc = cscale(acc, s);
    if (coef) {
      const float4 c = coef[0];
      float2 v = cscale(acc, c.x);
      if (u) { const float2 uu = u[pix]; v.x = fmaf(c.y, uu.x, v.x); v.y = fmaf(c.y, uu.y, v.y); }
      if (d) { const float2 dd = d[pix]; v.x = fmaf(c.z, dd.x, v.x); v.y = fmaf(c.z, dd.y, v.y); }
      acc = v;
    }
    out[pix] = acc;
  }
}

// mode 0: normal (interp -> * w * scale -> spread into dst)
// mode 1: forward (interp -> y[j][orig] = scale * sqrt_w * v - ymeas, partial |.|^2)
// mode 2: adjoint (spread scale * sqrt_w * y[j][orig] into dst)
__global__ void __launch_bounds__(128)
k_nufft_samples(int mode, const float2* __restrict__ src, float2* __restrict__ dst,
                const int* __restrict__ base, const float* __restrict__ frac,
                const float* __restrict__ wgt, const int* __restrict__ orig, long long N,
                NufftGeom g, int ncoils, float scale, float2* __restrict__ y,
                const float2* __restrict__ ymeas, double* __restrict__ partial) {
  double acc2 = 0.0;
  const int w = g.width;
  const int w0 = (g.n[0] == 1) ? 1 : w, w1 = (g.n[1] == 1) ? 1 : w;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    Taps tp;
    sample_taps(g, base, frac, i, N, tp);
    const float wi = wgt ? wgt[i] : 1.f;  // mode 0: w; modes 1/2: sqrt(w)
    const long long oi = orig ? orig[i] : i;
    for (int j = 0; j < ncoils; ++j) {
      const long long go = (long long)j * g.G;
      if (mode == 2) {
        const float2 yv = cscale(y[(long long)j * N + oi], wi * scale);
        for (int a0 = 0; a0 < w0; ++a0)
          for (int a1 = 0; a1 < w1; ++a1) {
            const float wa = tp.wt[0][a0] * tp.wt[1][a1];
            const int o01 = tp.off[0][a0] + tp.off[1][a1];
            for (int a2 = 0; a2 < w; ++a2) {
              const float wt = wa * tp.wt[2][a2];
              red_add_f2(dst + go + o01 + tp.off[2][a2], cscale(yv, wt));
            }
          }
        continue;
      }
      float2 v = make_float2(0.f, 0.f);
      for (int a0 = 0; a0 < w0; ++a0)
        for (int a1 = 0; a1 < w1; ++a1) {
          const float wa = tp.wt[0][a0] * tp.wt[1][a1];
          const int o01 = tp.off[0][a0] + tp.off[1][a1];
          for (int a2 = 0; a2 < w; ++a2) {
            const float2 sv = src[go + o01 + tp.off[2][a2]];
            const float wt = wa * tp.wt[2][a2];
            v.x = fmaf(wt, sv.x, v.x);
            v.y = fmaf(wt, sv.y, v.y);
          }
        }
      if (mode == 1) {
        float2 yv = cscale(v, wi * scale);
        if (ymeas) {
          yv = csub(yv, ymeas[(long long)j * N + oi]);
          acc2 += (double)yv.x * yv.x + (double)yv.y * yv.y;
        }
        y[(long long)j * N + oi] = yv;
        continue;
      }
      v = cscale(v, wi * scale);
      for (int a0 = 0; a0 < w0; ++a0)
        for (int a1 = 0; a1 < w1; ++a1) {
          const float wa = tp.wt[0][a0] * tp.wt[1][a1];
          const int o01 = tp.off[0][a0] + tp.off[1][a1];
          for (int a2 = 0; a2 < w; ++a2) red_add_f2(dst + go + o01 + tp.off[2][a2], cscale(v, wa * tp.wt[2][a2]));
        }
    }
  }
  if (partial) {
    __shared__ double red[128];
    red[threadIdx.x] = acc2;
    __syncthreads();
    for (int s = 64; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
  }
}

// ----------------------------------------------------------------- binned gridding
// Samples sorted by the tile (bin) of their first tap; one CTA per chunk of <= BIN_CHUNK
// samples of one bin.  The CTA stages the bin's (B + w - 1)^d spectrum tile in shared
// memory (interp reads), accumulates the spread into a shared tile (shared atomics) and
// flushes it with one global float2 atomic per cell: ~ (1 + (w-1)/B)^d global accesses
// per grid cell instead of w^d per sample.  KB weights are computed once per sample into
// shared memory and reused for every coil.
constexpr int BIN_CHUNK = 256;
constexpr int BIN_THREADS = 256;

template <int ND, int W, int B>
struct BinCfg {
  static constexpr int TB = B + W - 1;                       // tile extent per active axis
  static constexpr int T0 = (ND == 3) ? TB : 1, T1 = TB, T2 = TB;
  static constexpr int CELLS = T0 * T1 * T2;
  static constexpr int NTAPS = (ND == 3 ? W : 1) * W * W;
};

// 0 normal (interp, *w, spread), 1 forward (interp -> y), 2 adjoint (spread y).
// Pass 1 (interp): L lanes per sample, each owning RPL rows (a0, a1) of W taps along the
// contiguous axis; the partial sums are reduced over the L lanes (log2 L shuffles).  With the
// odd tile pitch TB the 8 row starts of a W = 4 sample fall in distinct banks.
// Pass 2 (spread): warp per sample, lanes over taps, into a fixed-point int32 tile with native
// shared atomics (exact and order independent within the tile), converted back to float at
// the flush (one global float2 atomic per touched cell).
template <int ND, int W>
struct BinLanes {
  static constexpr int W0 = (ND == 3) ? W : 1;
  static constexpr int ROWS = W0 * W;  // (a0, a1) rows of a sample
  static constexpr int L = (ROWS % 8 == 0) ? 8 : ((ROWS % 4 == 0) ? 4 : ((ROWS % 2 == 0) ? 2 : 1));
  static constexpr int RPL = ROWS / L;
  static constexpr int SPW = 32 / L;  // samples per warp
};

constexpr int BIN_CPB = 1;  // coils per pass (2 shares tap weights over a pair but drops to 3 CTAs/SM: no gain measured)

template <int MODE, int ND, int W, int B>
struct BinSmem {
  using C = BinCfg<ND, W, B>;
  static constexpr int WS = 3 * W + 1;  // odd per-sample stride of the tap weights
  static constexpr size_t TILE = (MODE == 2) ? 0 : sizeof(float2) * BIN_CPB * C::CELLS;
  static constexpr size_t ACC = (MODE == 1) ? 0 : sizeof(int2) * BIN_CPB * C::CELLS;
  static constexpr size_t SV = sizeof(float2) * BIN_CPB * BIN_CHUNK;
  static constexpr size_t PER = sizeof(float) * (WS + 2) * BIN_CHUNK + sizeof(int) * 2 * BIN_CHUNK;
  static constexpr size_t BYTES = TILE + ACC + SV + PER + sizeof(int) * C::CELLS + 16;
};

template <int MODE, int ND, int W, int B>
__global__ void __launch_bounds__(BIN_THREADS)
k_nufft_bins(const float2* __restrict__ src, float2* __restrict__ dst, const int* __restrict__ base,
             const float* __restrict__ frac, const float* __restrict__ wgt, const int* __restrict__ orig,
             long long N, const int* __restrict__ chunks, NufftGeom g, int ncoils, float scale,
             float2* __restrict__ y, const float2* __restrict__ ymeas, double* __restrict__ partial) {
  using C = BinCfg<ND, W, B>;
  using LN = BinLanes<ND, W>;
  using SM = BinSmem<MODE, ND, W, B>;
  constexpr int CELLS = C::CELLS, T1 = C::T1, T2 = C::T2;
  constexpr int A0 = 3 - ND;  // first active axis
  constexpr int L = LN::L, RPL = LN::RPL, SPW = LN::SPW;
  constexpr int NWARPS = BIN_THREADS / 32;
  constexpr int CPB = BIN_CPB, WS = SM::WS;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* tile = reinterpret_cast<float2*>(smraw);                  // [CPB][CELLS] spectrum (modes 0, 1)
  int2* acc = reinterpret_cast<int2*>(smraw + SM::TILE);            // [CPB][CELLS] fixed-point spread (0, 2)
  float2* sv = reinterpret_cast<float2*>(smraw + SM::TILE + SM::ACC);  // [CPB][BIN_CHUNK] sample values
  float* wts = reinterpret_cast<float*>(sv + CPB * BIN_CHUNK);     // [BIN_CHUNK][WS]
  float* swi = wts + WS * BIN_CHUNK;                                // [BIN_CHUNK] sqrt weights
  float* swm = swi + BIN_CHUNK;                                     // [BIN_CHUNK] max tap weight
  int* soi = reinterpret_cast<int*>(swm + BIN_CHUNK);               // [BIN_CHUNK] output index
  int* scb = soi + BIN_CHUNK;                                       // [BIN_CHUNK] first-tap cell
  int* coff = scb + BIN_CHUNK;                                      // [CELLS] grid offsets
  __shared__ float s_red[NWARPS];
  const int* ch = chunks + 5 * blockIdx.x;
  const int org0 = ch[0], org1 = ch[1], org2 = ch[2];
  const int s0 = ch[3], ns = ch[4];
  const int tid = threadIdx.x;
  const long long sg12 = (long long)g.g[1] * g.g[2];
  // per-sample KB weights, first-tap cell, density weight, output index and the largest tap
  // weight (once per chunk, reused by every coil)
  for (int i = tid; i < ns; i += BIN_THREADS) {
    const long long sidx = s0 + i;
    swi[i] = wgt ? wgt[sidx] : 1.f;
    soi[i] = orig ? orig[sidx] : (int)sidx;
    float wm = 1.f;
    int lc[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a < A0) {
#pragma unroll
        for (int k = 0; k < W; ++k) wts[i * WS + a * W + k] = (k == 0) ? 1.f : 0.f;
        continue;
      }
      int bb = base[a * N + sidx] % g.g[a];
      if (bb < 0) bb += g.g[a];
      int l = bb - (a == 0 ? org0 : (a == 1 ? org1 : org2));
      if (l < 0) l += g.g[a];
      lc[a] = l;
      const float t = frac[a * N + sidx];
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const float wk = kb_weight(t - (float)k, g.beta[a], (float)W);
        wts[i * WS + a * W + k] = wk;
        m = fmaxf(m, wk);
      }
      wm *= m;
    }
    swm[i] = wm;
    scb[i] = (lc[0] * T1 + lc[1]) * T2 + lc[2];
  }
  for (int e = tid; e < CELLS; e += BIN_THREADS) {
    const int c2 = e % T2, c1 = (e / T2) % T1, c0 = e / (T2 * T1);
    int k0 = org0 + c0, k1 = org1 + c1, k2 = org2 + c2;
    k0 -= (k0 >= g.g[0]) ? g.g[0] : 0;
    k1 -= (k1 >= g.g[1]) ? g.g[1] : 0;
    k2 -= (k2 >= g.g[2]) ? g.g[2] : 0;
    if (k0 >= g.g[0]) k0 %= g.g[0];  // tiles wider than the grid (tiny grids)
    if (k1 >= g.g[1]) k1 %= g.g[1];
    if (k2 >= g.g[2]) k2 %= g.g[2];
    coff[e] = (int)((long long)perm_of(k0, g.P[0], g.Q[0]) * sg12 +
                    (long long)perm_of(k1, g.P[1], g.Q[1]) * g.g[2] + perm_of(k2, g.P[2], g.Q[2]));
  }
  const int lane = tid & 31, warp = tid >> 5;
  const int sub = lane % L, slot = lane / L;
  double acc2 = 0.0;
  // the spectrum tiles of the next coil pair are gathered with cp.async while the current pair
  // spreads (pass 2 does not read the tiles)
  auto fetch_tiles = [&](int j0) {
    __syncthreads();  // coff complete / previous tile readers done
#pragma unroll
    for (int c = 0; c < CPB; ++c) {
      if (j0 + c >= ncoils) break;
      const float2* sj = src + (long long)(j0 + c) * g.G;
      for (int e = tid; e < CELLS; e += BIN_THREADS) cp_async8(tile + c * CELLS + e, sj + coff[e]);
    }
    cp_async_commit();
  };
  if (MODE != 2) fetch_tiles(0);
  for (int j0 = 0; j0 < ncoils; j0 += CPB) {
    const int nc = min(CPB, ncoils - j0);
    if (MODE != 1) {
      __syncthreads();  // previous flush done
      for (int e = tid; e < CPB * CELLS; e += BIN_THREADS) acc[e] = make_int2(0, 0);
    }
    if (MODE != 2) cp_async_wait<0>();
    __syncthreads();
    // pass 1: the value of every sample for each coil of the pair (interp: L lanes per sample)
    if (MODE != 2) {
      for (int i0 = warp * SPW; i0 < ns; i0 += NWARPS * SPW) {
        const int i = i0 + slot;
        const bool has = i < ns;
        const int ii = has ? i : i0;
        const int cbase = scb[ii];
        const float* wi_ = wts + ii * WS;
        float2 v[CPB];
#pragma unroll
        for (int c = 0; c < CPB; ++c) v[c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const int r = sub * RPL + k, a0 = r / W, a1 = r - a0 * W;
          const float wr = wi_[a0] * wi_[W + a1];
          const int ro = cbase + (a0 * T1 + a1) * T2;
#pragma unroll
          for (int a2 = 0; a2 < W; ++a2) {
            const float wt = wr * wi_[2 * W + a2];
#pragma unroll
            for (int c = 0; c < CPB; ++c) {
              const float2 tv = tile[c * CELLS + ro + a2];
              v[c].x = fmaf(wt, tv.x, v[c].x);
              v[c].y = fmaf(wt, tv.y, v[c].y);
            }
          }
        }
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
          for (int c = 0; c < CPB; ++c) {
            v[c].x += __shfl_xor_sync(0xffffffffu, v[c].x, o);
            v[c].y += __shfl_xor_sync(0xffffffffu, v[c].y, o);
          }
        }
        if (!has || sub != 0) continue;
        const float sc = swi[i] * scale;
#pragma unroll
        for (int c = 0; c < CPB; ++c) {
          if (c >= nc) break;
          const float2 vs = cscale(v[c], sc);
          if (MODE == 1) {
            const long long yo = (long long)(j0 + c) * N + soi[i];
            float2 yv = vs;
            if (ymeas) {
              yv = csub(yv, ymeas[yo]);
              acc2 += (double)yv.x * yv.x + (double)yv.y * yv.y;
            }
            y[yo] = yv;
          } else {
            sv[c * BIN_CHUNK + i] = vs;
          }
        }
      }
    } else {
      for (int i = tid; i < ns; i += BIN_THREADS) {
        const float sc = swi[i] * scale;
#pragma unroll
        for (int c = 0; c < CPB; ++c)
          sv[c * BIN_CHUNK + i] = (c < nc) ? cscale(y[(long long)(j0 + c) * N + soi[i]], sc) : make_float2(0.f, 0.f);
      }
    }
    if (MODE != 2 && j0 + CPB < ncoils) fetch_tiles(j0 + CPB);  // (its barrier also publishes sv)
    if (MODE == 1) continue;
    // fixed-point scale: every cell sum is bounded by B = sum_s max(|re|, |im|) * max tap weight
    // (over the pair); integers are scaled so that B maps below 2^30.  int32 shared atomics are
    // native, exact and order independent (a float CAS loop retries under contention).
    __syncthreads();
    float bsum = 0.f;
    for (int i = tid; i < ns; i += BIN_THREADS) {
      float m = 0.f;
#pragma unroll
      for (int c = 0; c < CPB; ++c) m = fmaxf(m, fmaxf(fabsf(sv[c * BIN_CHUNK + i].x), fabsf(sv[c * BIN_CHUNK + i].y)));
      bsum += m * swm[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    if (lane == 0) s_red[warp] = bsum;
    __syncthreads();
    float bnd = 0.f;
#pragma unroll
    for (int w = 0; w < NWARPS; ++w) bnd += s_red[w];
    bnd *= 1.0001f;  // float rounding of the bound itself
    if (!(bnd > 0.f)) continue;  // nothing to spread (all zero)
    int ex;
    frexpf(bnd, &ex);  // bnd < 2^ex
    const int S = min(126, max(-126, 30 - ex));
    const float up = ldexpf(1.f, S), down = ldexpf(1.f, -S);
    // pass 2: spread, one sample at a time per warp, lanes over taps (distinct cells)
    for (int i = warp; i < ns; i += NWARPS) {
      float2 v[CPB];
#pragma unroll
      for (int c = 0; c < CPB; ++c) v[c] = cscale(sv[c * BIN_CHUNK + i], up);
      const int cb = scb[i];
      const float* wi_ = wts + i * WS;
#pragma unroll
      for (int t0 = 0; t0 < C::NTAPS; t0 += 32) {
        const int t = t0 + lane;
        if (C::NTAPS % 32 == 0 || t < C::NTAPS) {
          const int a2 = t % W, a1 = (t / W) % W, a0 = (ND == 3) ? t / (W * W) : 0;
          const float wt = wi_[a0] * wi_[W + a1] * wi_[2 * W + a2];
          const int cell = cb + (a0 * T1 + a1) * T2 + a2;
#pragma unroll
          for (int c = 0; c < CPB; ++c) {
            atomicAdd(&acc[c * CELLS + cell].x, __float2int_rn(v[c].x * wt));
            atomicAdd(&acc[c * CELLS + cell].y, __float2int_rn(v[c].y * wt));
          }
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < CELLS; e += BIN_THREADS) {
      const int off = coff[e];
#pragma unroll
      for (int c = 0; c < CPB; ++c) {
        if (c >= nc) break;
        const int2 av = acc[c * CELLS + e];
        if (av.x == 0 && av.y == 0) continue;
        red_add_f2(dst + (long long)(j0 + c) * g.G + off, make_float2((float)av.x * down, (float)av.y * down));
      }
    }
  }
  if (MODE == 1 && partial) {
    __shared__ double red[BIN_THREADS];
    red[tid] = acc2;
    __syncthreads();
    for (int st = BIN_THREADS / 2; st > 0; st >>= 1) {
      if (tid < st) red[tid] += red[tid + st];
      __syncthreads();
    }
    if (tid == 0) partial[blockIdx.x] = red[0];
  }
}

template <int MODE, int ND, int W, int B>
int launch_bins_t(const float2* src, float2* dst, const int* base, const float* frac, const float* wgt,
                  const int* orig, long long N, const int* chunks, int nchunks, const NufftGeom& g, int ncoils,
                  float scale, float2* y, const float2* ymeas, double* partial, cudaStream_t st) {
  const size_t smem = BinSmem<MODE, ND, W, B>::BYTES;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(k_nufft_bins<MODE, ND, W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  if (nchunks < 1) return SR_OK;
  k_nufft_bins<MODE, ND, W, B><<<nchunks, BIN_THREADS, smem, st>>>(src, dst, base, frac, wgt, orig, N, chunks, g,
                                                                   ncoils, scale, y, ymeas, partial);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// binned gridding instantiations: (ND, W, B)
#define SR_BIN_CFGS(X) X(3, 4, 8) X(3, 4, 4) X(3, 6, 8) X(3, 6, 4) X(2, 4, 16) X(2, 4, 4) X(2, 6, 16) X(2, 6, 4)

bool bins_supported(const NufftGeom& g, int B) {
  const int nd = (g.n[0] > 1) ? 3 : 2;
#define X(ND_, W_, B_) if (nd == ND_ && g.width == W_ && B == B_) return true;
  SR_BIN_CFGS(X)
#undef X
  return false;
}

template <int MODE>
int launch_bins(const float2* src, float2* dst, const int* base, const float* frac, const float* wgt,
                const int* orig, long long N, const int* chunks, int nchunks, const NufftGeom& g, int B,
                int ncoils, float scale, float2* y, const float2* ymeas, double* partial, cudaStream_t st) {
  const int nd = (g.n[0] > 1) ? 3 : 2;
#define X(ND_, W_, B_)                                                                                     \
  if (nd == ND_ && g.width == W_ && B == B_)                                                              \
    return launch_bins_t<MODE, ND_, W_, B_>(src, dst, base, frac, wgt, orig, N, chunks, nchunks, g, ncoils, \
                                           scale, y, ymeas, partial, st);
  SR_BIN_CFGS(X)
#undef X
  return SR_EUNSUPPORTED;
}

int grid_fft(float2* grid, const NufftGeom& g, int ncoils, int inv, cudaStream_t st) {
  // axis 2 (contiguous), axis 1 ([C*g0][g1][g2]), axis 0 ([C][g0][g1*g2])
  int rc = fft_axis(grid, (long long)ncoils * g.g[0] * g.g[1], g.g[2], 1, inv, st);
  if (rc) return rc;
  rc = fft_axis(grid, (long long)ncoils * g.g[0], g.g[1], g.g[2], inv, st);
  if (rc) return rc;
  return fft_axis(grid, ncoils, g.g[0], (long long)g.g[1] * g.g[2], inv, st);
}

bool make_geom(const int* dims, const int* gdims, const float* betas, int width, NufftGeom& g) {
  for (int a = 0; a < 3; ++a) {
    g.n[a] = dims[a];
    g.g[a] = gdims[a];
    g.beta[a] = betas[a];
    if (dims[a] < 1 || gdims[a] < dims[a]) return false;
    if (gdims[a] == 1) { g.P[a] = 1; g.Q[a] = 1; continue; }
    int P = 0, Q = 0;
    switch (gdims[a]) {
#define X(N_, P_, Q_) case N_: P = P_; Q = Q_; break;
      SR_FFT_SIZES(X)
#undef X
      default: return false;
    }
    g.P[a] = P;
    g.Q[a] = Q;
  }
  if (width < 1 || width > MAXW) return false;
  g.width = width;
  g.D = (long long)dims[0] * dims[1] * dims[2];
  g.G = (long long)gdims[0] * gdims[1] * gdims[2];
  return true;
}

unsigned sample_blocks(long long N) {
  long long b = (N + 127) / 128;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

extern "C" {


// Plan arrays (device): base (3, N) int32 tap bases (fp64-derived, ceil(u - w/2)),
// frac (3, N) fp32 offsets u - base, wgt (N) = density weight w (normal op) and
// sqrtw (N) = sqrt(w) (forward/adjoint) or NULL, orig (N) original sample index of
// the (locality-sorted) sample order or NULL; inverse apodisation per axis ia0/ia1/ia2.
// dims/gdims: 3 entries (leading 1 for 2-D).  grids: 2 * ncoils * G complex64 workspace.
int sr_nufft_normal(const sr_c64* x, const sr_c64* anchor, const sr_c64* maps, int ncoils,
                    const int* dims, const int* gdims, const float* betas, int width,
                    const float* ia0, const float* ia1, const float* ia2, const int* base,
                    const float* frac, const float* wgt, long long nsamples, sr_c64* out,
                    sr_c64* grids, const float* coef, const sr_c64* u, const sr_c64* d, const int* chunks,
                    int nchunks, int binsize, void* stream) {
  NufftGeom g;
  if (!make_geom(dims, gdims, betas, width, g) || ncoils < 1) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  float2* src = (float2*)grids;
  float2* dst = src + (long long)ncoils * g.G;
  k_nufft_embed<<<148 * 8, 256, 0, st>>>((const float2*)x, (const float2*)maps, ia0, ia1, ia2, src, g,
                                         ncoils, (const float2*)anchor);
  SR_CHECK_LAUNCH();
  int rc = grid_fft(src, g, ncoils, 0, st);
  if (rc) return rc;
  if (cudaMemsetAsync(dst, 0, sizeof(float2) * ncoils * g.G, st) != cudaSuccess) return SR_ECUDA;
  if (chunks && bins_supported(g, binsize)) {
    rc = launch_bins<0>(src, dst, base, frac, wgt, nullptr, nsamples, chunks, nchunks, g, binsize, ncoils,
                        (float)(1.0 / (double)g.D), nullptr, nullptr, nullptr, st);
    if (rc) return rc;
  } else {
    k_nufft_samples<<<sample_blocks(nsamples), 128, 0, st>>>(0, src, dst, base, frac, wgt, nullptr, nsamples,
                                                             g, ncoils, (float)(1.0 / (double)g.D), nullptr,
                                                             nullptr, nullptr);
    SR_CHECK_LAUNCH();
  }
  rc = grid_fft(dst, g, ncoils, 1, st);
  if (rc) return rc;
  k_nufft_crop<<<148 * 8, 256, 0, st>>>(dst, (const float2*)maps, ia0, ia1, ia2, (float2*)out, g, ncoils, 1.f,
                                        (const float4*)coef, (const float2*)u, (const float2*)d);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_nufft_partial_blocks(long long nsamples) { return (int)sample_blocks(nsamples); }

// y (ncoils, N) in original sample order = sqrt(w) A x (- ymeas; partial |.|^2 per block)
int sr_nufft_forward(const sr_c64* x, const sr_c64* maps, int ncoils, const int* dims, const int* gdims,
                     const float* betas, int width, const float* ia0, const float* ia1, const float* ia2,
                     const int* base, const float* frac, const float* sqrtw, const int* orig,
                     long long nsamples, sr_c64* y, const sr_c64* ymeas, double* partial, sr_c64* grids,
                     const int* chunks, int nchunks, int binsize, void* stream) {
  NufftGeom g;
  if (!make_geom(dims, gdims, betas, width, g) || ncoils < 1) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  float2* src = (float2*)grids;
  k_nufft_embed<<<148 * 8, 256, 0, st>>>((const float2*)x, (const float2*)maps, ia0, ia1, ia2, src, g,
                                         ncoils, nullptr);
  SR_CHECK_LAUNCH();
  int rc = grid_fft(src, g, ncoils, 0, st);
  if (rc) return rc;
  if (chunks && bins_supported(g, binsize))
    return launch_bins<1>(src, nullptr, base, frac, sqrtw, orig, nsamples, chunks, nchunks, g, binsize, ncoils,
                          (float)(1.0 / sqrt((double)g.D)), (float2*)y, (const float2*)ymeas, partial, st);
  k_nufft_samples<<<sample_blocks(nsamples), 128, 0, st>>>(1, src, nullptr, base, frac, sqrtw, orig, nsamples,
                                                           g, ncoils, (float)(1.0 / sqrt((double)g.D)),
                                                           (float2*)y, (const float2*)ymeas, partial);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// out = A^H y (y (ncoils, N) original order)
int sr_nufft_adjoint(const sr_c64* y, const sr_c64* maps, int ncoils, const int* dims, const int* gdims,
                     const float* betas, int width, const float* ia0, const float* ia1, const float* ia2,
                     const int* base, const float* frac, const float* sqrtw, const int* orig,
                     long long nsamples, sr_c64* out, sr_c64* grids, const float* coef, const sr_c64* u,
                     const sr_c64* d, const int* chunks, int nchunks, int binsize, void* stream) {
  NufftGeom g;
  if (!make_geom(dims, gdims, betas, width, g) || ncoils < 1) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  float2* dst = (float2*)grids;
  if (cudaMemsetAsync(dst, 0, sizeof(float2) * ncoils * g.G, st) != cudaSuccess) return SR_ECUDA;
  if (chunks && bins_supported(g, binsize)) {
    int rc0 = launch_bins<2>(nullptr, dst, base, frac, sqrtw, orig, nsamples, chunks, nchunks, g, binsize, ncoils,
                             (float)(1.0 / sqrt((double)g.D)), (float2*)y, nullptr, nullptr, st);
    if (rc0) return rc0;
  } else {
    k_nufft_samples<<<sample_blocks(nsamples), 128, 0, st>>>(2, nullptr, dst, base, frac, sqrtw, orig, nsamples,
                                                             g, ncoils, (float)(1.0 / sqrt((double)g.D)),
                                                             (float2*)y, nullptr, nullptr);
    SR_CHECK_LAUNCH();
  }
  int rc = grid_fft(dst, g, ncoils, 1, st);
  if (rc) return rc;
  // the 1/sqrt(D) scale was applied with the spread
  k_nufft_crop<<<148 * 8, 256, 0, st>>>(dst, (const float2*)maps, ia0, ia1, ia2, (float2*)out, g, ncoils,
                                        1.f, (const float4*)coef, (const float2*)u, (const float2*)d);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// Batched FFT along one axis of a [outer][n][inner] array, in place, unnormalised;
// fwd: natural -> perm order, inv: perm -> natural (test/diagnostic entry point).
int sr_fft_axis(sr_c64* data, long long outer, int n, long long inner, int inv, void* stream) {
  if (outer < 1 || n < 1 || inner < 1) return SR_EINVAL;
  return fft_axis((float2*)data, outer, n, inner, inv, (cudaStream_t)stream);
}

}  // extern "C"
