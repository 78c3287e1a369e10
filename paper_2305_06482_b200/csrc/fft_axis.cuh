// Per-axis FFT kernels of the gridded NUFFT (contiguous rows and strided axes), shared by
// the size-bucket translation units fft_axis_inst_<k>.cu (nufft.cu chains the buckets).
#pragma once
#include "fft2step.cuh"

// minimum resident CTAs per SM for the fused row passes of the gridded NUFFT (register caps)
#ifndef SR_EMBED_MINB
#define SR_EMBED_MINB 1
#endif
#ifndef SR_CROP_MINB
#define SR_CROP_MINB 1
#endif
#ifndef SR_EMBED_LOOP_MINB
#define SR_EMBED_LOOP_MINB 1
#endif

// Zero-padding structure of an oversampled NUFFT axis of length g holding an image axis of
// length n (centered: image index i sits at grid index (i - n/2) mod g, linops.py:438-446).
static __device__ __forceinline__ bool ax_inside(int k, int n, int g) {
  const int h = n >> 1;
  return k < n - h || k >= g - h;
}
static __device__ __forceinline__ int ax_wrap(int i, int n, int g) {
  const int r = i - (n >> 1);
  return r < 0 ? r + g : r;
}

// Pruning of one strided FFT pass: inputs outside the image extent nin are zero (forward
// passes over a zero-padded axis), outputs outside nout are not needed (inverse passes before
// a crop), and of the outer planes only the on (of og) image planes are live.
struct AxPrune {
  int nin, nout;  // extents along the FFT axis (== N: no pruning)
  int on, og;     // live / total planes of the axis just outside (on == og: all planes)
  int oa = 0;     // first live image plane (a slab of the image planes: oa .. oa + on of onf)
  int onf = 0;    // image planes of that axis when only a slab is live (0: on)
  __device__ __forceinline__ bool in(int k, int N) const { return nin == N || ax_inside(k, nin, N); }
  __device__ __forceinline__ bool out(int k, int N) const { return nout == N || ax_inside(k, nout, N); }
  __device__ __forceinline__ long long plane(long long o) const {
    if (onf == 0) {
      if (on == og) return o;
      const long long j = o / on;
      return j * og + ax_wrap((int)(o - j * on), on, og);
    }
    const long long j = o / on;
    const int i = oa + (int)(o - j * on);
    return j * og + (onf == og ? i : ax_wrap(i, onf, og));
  }
};

// ----------------------------------------------------------------- fused NUFFT row passes
// The first forward FFT pass (contiguous axis 2) fused with the embed (c_j (x - a) / apod
// into the zero-padded grid), and the last inverse pass fused with the crop, the conjugate
// coil sum and the solver epilogue.  Only rows whose (k0, k1) lie inside the image are
// touched: the strided passes treat the others as zero (AxPrune).
struct RowGeom {
  const float2* x;
  const float2* anchor;
  const float2* maps;
  const float* ia0;
  const float* ia1;
  const float* ia2;
  float2* grid;
  float2* out;
  int n0, n1, n2, g0, g1, g2;
  long long D, G;
  int ncoils;
  float scale;
  const float4* coef;
  const float2* u;
  const float2* d;
  // inverse row pass: only the image planes i0 in [i0a, i0b) (i0b < 0: all n0) -- one slab of the
  // coil-sharded pipeline whose coil sum is all-reduced while the next slab computes
  int i0a = 0, i0b = -1;
};


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
k_fft_rows(float2* __restrict__ data, long long nrows, int inv, int nat) {
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
    // nat: the row leaves in natural frequency order (perm position of k read from shared memory)
    for (int e = tid; e < nvalid; e += T) {
      const int l3 = e / N, pos = e - l3 * N;
      base[e] = buf[l3 * S::VS + S::pad(nat ? S::perm_pos(pos) : pos)];
    }
  } else {
    // nat (natural-order frequency rows, Q <= P): the row is staged as it is, step 2' reads its
    // group at the natural positions k2 + Q k1 and writes the perm layout after a barrier
    constexpr bool NATOK = (Q <= P) && (P > 1);
    const bool natload = NATOK && nat;
    for (int e = tid; e < nvalid; e += T) {
      const int l3 = e / N, pos = e - l3 * N;
      buf[l3 * S::VS + (natload ? pos : S::pad(nat ? S::perm_pos(pos) : pos))] = base[e];
    }
    __syncthreads();
    if (natload) {
      const bool has = tid < ROWS * Q;
      const int l2 = tid / Q, k2 = tid - l2 * Q;
      float2 g[P];
      if (has) {
        const float2* gn = buf + l2 * S::VS + k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gn[Q * k1];
        fft_s2_inv<P, Q>(g, k2, tw);
      }
      __syncthreads();
      if (has) {
        float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
      }
      __syncthreads();
    } else if (P > 1) {
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

// strided axis of [outer][N][inner]: CTA = CB consecutive inner indices of PLANES outer
// planes, walked in turn.  Forward: step 1 reads the natural-order column strip from global
// (coil/plane p+1's strip is prefetched into registers while plane p transforms), step 2 writes
// its perm-order groups straight to global.  Inverse: step 2' reads its perm-order group from
// global, step 1' writes natural order.  One shared-memory exchange per plane either way.
template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::TS)
k_fft_strided(float2* __restrict__ data, long long inner, int inv, AxPrune pr, int nplanes, int planes) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, CB = A::CB, T = A::TS, VSP = A::VSP;
  extern __shared__ __align__(16) float2 dsm[];
  float2* tw = dsm;
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long c0 = (long long)blockIdx.x * CB;
  const int ncols = (int)min((long long)CB, inner - c0);
  const int c = tid % CB, p = tid / CB;
  const bool cvalid = c < ncols;
  const long long step = (long long)P * inner;  // distance between q and q+1 along the axis
  const int o0 = blockIdx.y * planes, o1 = min(nplanes, o0 + planes);
  if (inv) init_tw_s2<P, Q>(tw, tid, T); else init_tw_s1<P, Q>(tw, tid, T);
  if (!inv) {
    // this thread's natural positions p + P q; pruned inputs are zero
    float2 rn[Q];
    auto fetch = [&](int o) {
      const float2* col = data + pr.plane(o) * N * inner + (long long)p * inner + c0 + c;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        rn[q] = (cvalid && pr.in(p + P * q, N)) ? __ldcg(col + q * step) : make_float2(0.f, 0.f);
    };
    fetch(o0);
    __syncthreads();
    for (int o = o0; o < o1; ++o) {
      float2* img = data + pr.plane(o) * N * inner;
      float2 r[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = rn[q];
      if (o + 1 < o1) fetch(o + 1);
      fft_s1_fwd<P, Q>(r, p, tw);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) buf[c * VSP + S::GS * k2 + p] = r[k2];
      __syncthreads();
      for (int it = tid; it < CB * Q; it += T) {
        const int cc = it % CB, k2 = it / CB;
        if (cc >= ncols) continue;
        float2 g[P];
        const float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
        if (P > 1) fft_s2_fwd<P>(g);
        float2* dst = img + (long long)(P * k2) * inner + c0 + cc;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) dst[(long long)k1 * inner] = g[k1];
      }
      __syncthreads();  // buf is rewritten by the next plane
    }
  } else {
    __syncthreads();
    for (int o = o0; o < o1; ++o) {
      float2* img = data + pr.plane(o) * N * inner;
      for (int it = tid; it < CB * Q; it += T) {
        const int cc = it % CB, k2 = it / CB;
        if (cc >= ncols) continue;
        float2 g[P];
        const float2* src = img + (long long)(P * k2) * inner + c0 + cc;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = __ldcg(src + (long long)k1 * inner);
        if (P > 1) fft_s2_inv<P, Q>(g, k2, tw);
        float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
      }
      __syncthreads();
      float2 r[Q];
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[c * VSP + S::GS * k2 + p];
      fft_s1_inv<Q>(r);
      if (cvalid) {
        float2* col = img + (long long)p * inner + c0 + c;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (pr.out(p + P * q, N)) col[q * step] = r[q];
      }
      __syncthreads();
    }
  }
}

template <int P, int Q>
int launch_rows(float2* data, long long nrows, int inv, cudaStream_t st, int nat = 0) {
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
  k_fft_rows<P, Q><<<(unsigned)nb, A::T, smem, st>>>(data, nrows, inv, nat);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

template <int P, int Q>
int launch_strided(float2* data, long long outer, long long inner, int inv, cudaStream_t st,
                   AxPrune pr = AxPrune{P * Q, P * Q, 1, 1}) {
  using A = AxCfg<P, Q>;
  using S = FftShape<P, Q>;
  const size_t smem = sizeof(float2) * (S::N + A::CB * A::VSP);
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(k_fft_strided<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SR_ECUDA;
    cfg = true;
  }
  // planes per CTA: enough column strips to fill the GPU ~4 times, the rest walked in turn
  const long long strips = (inner + A::CB - 1) / A::CB;
  const long long target = 148LL * 16;
  int planes = (int)((strips * outer + target - 1) / target);
  planes = planes < 1 ? 1 : (planes > 8 ? 8 : planes);
  const long long gy = (outer + planes - 1) / planes;
  if (gy > 65535) return SR_EINVAL;
  dim3 grid((unsigned)strips, (unsigned)gy);
  k_fft_strided<P, Q><<<grid, A::TS, smem, st>>>(data, inner, inv, pr, (int)outer, planes);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::T, SR_EMBED_MINB)
k_embed_rows(const RowGeom rg) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, ROWS = A::ROWS, T = A::T;
  extern __shared__ __align__(16) float2 dsm[];
  __shared__ long long rbase[ROWS];
  float2* tw = dsm;
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long nrows = (long long)rg.ncoils * rg.n0 * rg.n1;
  const long long row0 = (long long)blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  init_tw_s1<P, Q>(tw, tid, T);
  const long long rid = row0 + lr;
  const bool valid = rid < nrows;
  // coil index fastest: the CTAs (and rows) of one image row run together, so the image row
  // is read from DRAM once and from L2 for the other coils (coil-slowest order streamed the
  // whole image through DRAM once per coil: 2.68 -> 1.43 GB read, 1.28 -> 1.21 ms at config 4;
  // four row groups per CTA with the next group's loads in flight measured slower, 1.75 ms)
  const int j = valid ? (int)(rid % rg.ncoils) : 0;
  const long long rem = valid ? rid / rg.ncoils : 0;
  const int i0 = (int)(rem / rg.n1), i1 = (int)(rem - (long long)i0 * rg.n1);
  if (p == 0)
    rbase[lr] = (long long)j * rg.G +
                ((long long)ax_wrap(i0, rg.n0, rg.g0) * rg.g1 + ax_wrap(i1, rg.n1, rg.g1)) * N;
  const long long pixrow = ((long long)i0 * rg.n1 + i1) * rg.n2;
  const float s01 = valid ? rg.ia0[i0] * rg.ia1[i1] : 0.f;
  const float2* mj = rg.maps + (long long)j * rg.D + pixrow;
  const float2* xr = rg.x + pixrow;
  const float2* ar = rg.anchor ? rg.anchor + pixrow : xr;  // never null-based
  const int h2 = rg.n2 >> 1;
  float2 r[Q];
  {
    // all loads of the thread issued back to back from clamped (always valid) addresses, then
    // selected: the rows are short, so the kernel lives on load latency
    float2 mv[Q], xv[Q];
    float iv[Q];
    bool in[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int k2 = p + P * q;
      in[q] = valid && ax_inside(k2, rg.n2, N);
      const int i2 = in[q] ? ((k2 < rg.n2 - h2) ? k2 + h2 : k2 - N + h2) : 0;
      mv[q] = mj[i2];
      xv[q] = xr[i2];
      iv[q] = rg.ia2[i2];
    }
    if (rg.anchor) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int k2 = p + P * q;
        const int i2 = in[q] ? ((k2 < rg.n2 - h2) ? k2 + h2 : k2 - N + h2) : 0;
        xv[q] = csub(xv[q], ar[i2]);
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q)
      r[q] = in[q] ? cscale(cmul(mv[q], xv[q]), s01 * iv[q]) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  fft_s1_fwd<P, Q>(r, p, tw);
#pragma unroll
  for (int k2 = 0; k2 < Q; ++k2) buf[lr * S::VS + S::GS * k2 + p] = r[k2];
  __syncthreads();
  // Step 2 writes straight from registers: the grid row is stored in natural frequency order
  // along axis 2 (a gridding tile row is one contiguous run), frequency k2 + Q k1 of group k2 --
  // lanes run over k2, so each k1 is a coalesced run of Q consecutive cells.  The strided axes
  // stay in perm order.
  const int nv = (int)min((long long)ROWS, nrows - row0);
  if (P > 1) {
    for (int it = tid; it < ROWS * Q; it += T) {
      const int l2 = it / Q, k2 = it - l2 * Q;
      if (l2 >= nv) continue;
      float2 g[P];
      const float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
      fft_s2_fwd<P>(g);
      float2* gr = rg.grid + rbase[l2] + k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) gr[Q * k1] = g[k1];
    }
  } else {
    for (int e = tid; e < nv * N; e += T) {
      const int l3 = e / N, pos = e - l3 * N;
      rg.grid[rbase[l3] + pos] = buf[l3 * S::VS + S::pad(pos)];
    }
  }
}

// The same pass with the coils looped inside the CTA (enough image rows to fill the GPU, short
// rows): a CTA owns ROWS image rows, keeps (x - a) / apod of its pixels in registers and streams the
// coil maps through them, the next coil's map values in flight (registers) while the current coil
// transforms -- the one-shot kernel above lives on load latency (config 4: 41 % of the DRAM peak).
template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::T, SR_EMBED_LOOP_MINB)
k_embed_rows_loop(const RowGeom rg) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, ROWS = A::ROWS, T = A::T;
  extern __shared__ __align__(16) float2 dsm[];
  __shared__ long long rbase[ROWS];
  float2* tw = dsm;
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long nrows = (long long)rg.n0 * rg.n1;  // image rows
  const long long row0 = (long long)blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  init_tw_s1<P, Q>(tw, tid, T);
  const long long rid = row0 + lr;
  const bool valid = rid < nrows;
  const int i0 = valid ? (int)(rid / rg.n1) : 0, i1 = valid ? (int)(rid - (long long)i0 * rg.n1) : 0;
  if (p == 0) rbase[lr] = ((long long)ax_wrap(i0, rg.n0, rg.g0) * rg.g1 + ax_wrap(i1, rg.n1, rg.g1)) * N;
  const long long pixrow = ((long long)i0 * rg.n1 + i1) * rg.n2;
  const float s01 = valid ? rg.ia0[i0] * rg.ia1[i1] : 0.f;
  const int h2 = rg.n2 >> 1;
  // pixel of each of the thread's positions k2 = p + P q (clamped to a valid address outside the
  // image, where the scaled input is zero)
  int i2s[Q];
  float2 xs[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k2 = p + P * q;
    const bool in = valid && ax_inside(k2, rg.n2, N);
    i2s[q] = in ? ((k2 < rg.n2 - h2) ? k2 + h2 : k2 - N + h2) : 0;
    float2 xv = rg.x[pixrow + i2s[q]];
    if (rg.anchor) xv = csub(xv, rg.anchor[pixrow + i2s[q]]);
    xs[q] = in ? cscale(xv, s01 * rg.ia2[i2s[q]]) : make_float2(0.f, 0.f);
  }
  const float2* mp = rg.maps + pixrow;
  float2 mv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) mv[q] = mp[i2s[q]];
  const int nv = (int)min((long long)ROWS, nrows - row0);
  __syncthreads();  // tw, rbase
  for (int j = 0; j < rg.ncoils; ++j) {
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = cmul(mv[q], xs[q]);
    if (j + 1 < rg.ncoils) {
      const float2* mn = mp + (long long)(j + 1) * rg.D;
#pragma unroll
      for (int q = 0; q < Q; ++q) mv[q] = mn[i2s[q]];
    }
    fft_s1_fwd<P, Q>(r, p, tw);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[lr * S::VS + S::GS * k2 + p] = r[k2];
    __syncthreads();
    float2* gj = rg.grid + (long long)j * rg.G;
    if (P > 1) {
      for (int it = tid; it < ROWS * Q; it += T) {
        const int l2 = it / Q, k2 = it - l2 * Q;
        if (l2 >= nv) continue;
        float2 g[P];
        const float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
        fft_s2_fwd<P>(g);
        float2* gr = gj + rbase[l2] + k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gr[Q * k1] = g[k1];
      }
    } else {
      for (int e = tid; e < nv * N; e += T) {
        const int l3 = e / N, pos = e - l3 * N;
        gj[rbase[l3] + pos] = buf[l3 * S::VS + S::pad(pos)];
      }
    }
    __syncthreads();  // buf is rewritten by the next coil
  }
}

// short rows (Q <= 12, config 4's 200-cell rows): capped at 3 CTAs / SM worth of registers (152 -> 128,
// 20 bytes of spills; config-4 apply -0.08 ms); a cap for 4 CTAs measured slower (+0.33 ms)
template <int P, int Q>
__global__ void __launch_bounds__(AxCfg<P, Q>::T, (SR_CROP_MINB > 1 || Q > 12) ? SR_CROP_MINB : 3)
k_rows_crop(const RowGeom rg) {
  using S = FftShape<P, Q>;
  using A = AxCfg<P, Q>;
  constexpr int N = S::N, ROWS = A::ROWS, T = A::T;
  constexpr int TILE = ROWS * S::VS;
  extern __shared__ __align__(16) float2 dsm[];
  __shared__ long long rbase[ROWS];
  float2* tw = dsm;
  float2* bufs = dsm + N;  // two row tiles: coil j+1 streams in (cp.async) while coil j transforms
  const int tid = threadIdx.x;
  const int i0a = rg.i0a, i0b = rg.i0b < 0 ? rg.n0 : rg.i0b;
  const long long nrows = (long long)(i0b - i0a) * rg.n1;
  const long long row0 = (long long)blockIdx.x * ROWS;
  const int lr = tid / P, p = tid % P;
  init_tw_s2<P, Q>(tw, tid, T);
  const long long rid = row0 + lr;
  const bool valid = rid < nrows;
  const int i0 = valid ? i0a + (int)(rid / rg.n1) : 0;
  const int i1 = valid ? (int)(rid - (long long)(i0 - i0a) * rg.n1) : 0;
  if (p == 0) rbase[lr] = ((long long)ax_wrap(i0, rg.n0, rg.g0) * rg.g1 + ax_wrap(i1, rg.n1, rg.g1)) * N;
  const long long pixrow = ((long long)i0 * rg.n1 + i1) * rg.n2;
  const int h2 = rg.n2 >> 1;
  const int nv = (int)min((long long)ROWS, nrows - row0);
  // natural output positions k2 = p + P q of this thread inside the image, and their pixel
  int i2s[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k2 = p + P * q;
    i2s[q] = (valid && ax_inside(k2, rg.n2, N)) ? ((k2 < rg.n2 - h2) ? k2 + h2 : k2 - N + h2) : -1;
  }
  float2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_float2(0.f, 0.f);
  __syncthreads();  // rbase
  // Grid rows are natural-order along axis 2.  With Q <= P (one step-2' task per thread) the row
  // lands in shared memory as it is (contiguous 16-byte cp.async), step 2' reads its group at the
  // natural positions k2 + Q k1 (lanes over k2: conflict-free) and, after a barrier, writes the
  // perm-padded layout step 1' expects; otherwise each cell goes straight to its perm position.
  constexpr bool NATLOAD = (Q <= P) && (N % 2 == 0) && (S::VS % 2 == 0);
  auto issue = [&](int j) {
    const float2* gj = rg.grid + (long long)j * rg.G;
    float2* dst = bufs + (j & 1) * TILE;
    if constexpr (NATLOAD) {
      for (int e = 2 * tid; e < nv * N; e += 2 * T) {
        const int l3 = e / N, pos = e - l3 * N;
        cp_async16(dst + l3 * S::VS + pos, gj + rbase[l3] + pos);
      }
    } else {
      for (int e = tid; e < nv * N; e += T) {
        const int l3 = e / N, pos = e - l3 * N;
        cp_async8(dst + l3 * S::VS + S::pad(S::perm_pos(pos)), gj + rbase[l3] + pos);
      }
    }
    cp_async_commit();
  };
  issue(0);
  for (int j = 0; j < rg.ncoils; ++j) {
    if (j + 1 < rg.ncoils) {
      issue(j + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    float2 m[Q];
    const float2* mj = rg.maps + (long long)j * rg.D + pixrow;
#pragma unroll
    for (int q = 0; q < Q; ++q) m[q] = (i2s[q] >= 0) ? mj[i2s[q]] : make_float2(0.f, 0.f);
    __syncthreads();
    float2* buf = bufs + (j & 1) * TILE;
    if constexpr (NATLOAD && P > 1) {
      const bool has = tid < ROWS * Q;
      const int l2 = tid / Q, k2 = tid - l2 * Q;
      float2 g[P];
      if (has) {
        const float2* gn = buf + l2 * S::VS + k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) g[k1] = gn[Q * k1];
        fft_s2_inv<P, Q>(g, k2, tw);
      }
      __syncthreads();  // every natural-order read done before the perm-order writes
      if (has) {
        float2* gp = buf + l2 * S::VS + S::GS * k2;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
      }
      __syncthreads();
    } else if (P > 1) {
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
#pragma unroll
    for (int q = 0; q < Q; ++q) cfma_conj(acc[q], m[q], r[q]);
    __syncthreads();  // buf (j & 1) is refilled by the prefetch issued next iteration
  }
  if (!valid) return;
  const float s01 = rg.ia0[i0] * rg.ia1[i1] * rg.scale;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i2 = i2s[q];
    if (i2 < 0) continue;
    const long long pix = pixrow + i2;
    float2 v = cscale(acc[q], s01 * rg.ia2[i2]);
    if (rg.coef) {
      const float4 cf = rg.coef[0];
      v = cscale(v, cf.x);
      if (rg.u) { const float2 uu = rg.u[pix]; v.x = fmaf(cf.y, uu.x, v.x); v.y = fmaf(cf.y, uu.y, v.y); }
      if (rg.d) { const float2 dd = rg.d[pix]; v.x = fmaf(cf.z, dd.x, v.x); v.y = fmaf(cf.z, dd.y, v.y); }
    }
    rg.out[pix] = v;
  }
}

template <int P, int Q, bool INV>
int launch_row_fused(const RowGeom& rg, cudaStream_t st) {
  using A = AxCfg<P, Q>;
  using S = FftShape<P, Q>;
  const size_t smem = sizeof(float2) * (S::N + (INV ? 2 : 1) * A::ROWS * S::VS);
  auto kern = INV ? k_rows_crop<P, Q> : k_embed_rows<P, Q>;
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SR_ECUDA;
    cfg = true;
  }
  if constexpr (!INV && Q <= 16) {
    // coil-looped embed: several coils and enough image rows for >= 2 CTAs per SM
    const long long nimg = (long long)rg.n0 * rg.n1;
    const long long nb = (nimg + A::ROWS - 1) / A::ROWS;
    if (rg.ncoils >= 2 && nb >= 2 * 148 && nb <= 0x7fffffffLL) {
      static bool cfg2 = false;
      if (!cfg2) {
        if (cudaFuncSetAttribute(k_embed_rows_loop<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
          return SR_ECUDA;
        cfg2 = true;
      }
      k_embed_rows_loop<P, Q><<<(unsigned)nb, A::T, smem, st>>>(rg);
      SR_CHECK_LAUNCH();
      return SR_OK;
    }
  }
  const int nplanes = INV ? (rg.i0b < 0 ? rg.n0 : rg.i0b) - rg.i0a : rg.n0;
  const long long nrows = INV ? (long long)nplanes * rg.n1 : (long long)rg.ncoils * rg.n0 * rg.n1;
  if (nrows <= 0) return SR_OK;
  const long long nblk = (nrows + A::ROWS - 1) / A::ROWS;
  if (nblk > 0x7fffffffLL) return SR_EINVAL;
  kern<<<(unsigned)nblk, A::T, smem, st>>>(rg);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // namespace
