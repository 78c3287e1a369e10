// Per-axis FFT kernels of the gridded NUFFT (contiguous rows and strided axes), shared by
// the size-bucket translation units fft_axis_inst_<k>.cu (nufft.cu chains the buckets).
#pragma once
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

}  // namespace
