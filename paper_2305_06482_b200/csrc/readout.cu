// K8: readout decoupling of 3-D Cartesian data (BASELINE config 2).
//
// 3-D Cartesian k-space sampled on a ky-kz mask broadcast over the fully sampled
// readout kx, stored (C, nkx, Nyz) in argwhere order (kx-major), becomes nkx
// independent 2-D problems after a centered unitary 1-D IFFT along kx: for every
// readout position x, out[x, c, :] equals the 2-D SENSE forward of slice x with
// maps[:, x] and the ky-kz mask (verified on the oracle).
// Centered IDFT (the reference convention, linops.py:300-313):
//   img[x] = n^-1/2 sum_k K[k] e^{2 pi i (k-h)(x-h)/n},  h = n // 2
//          = n^-1/2 e^{2 pi i h^2/n} e^{-2 pi i h x/n} * IDFT_unnorm( K[k] e^{-2 pi i k h/n} )[x]
// The kernel runs the two-level register FFT with natural-order input AND output
// (the perm -> natural reorder is folded into the copy-out) and writes the result
// slice-major: out[x][c][j], i.e. directly in the (slices, C, N) layout the batched
// reconstruction consumes.
#include "fft2step.cuh"

namespace {

template <int P, int Q>
struct RoCfg {
  static constexpr int CB = (P >= 16) ? 16 : (P >= 4 ? 32 : 64);
  static constexpr int T = CB * P;
  static constexpr int VSP = FftShape<P, Q>::VS0 | 1;
};

// in: (C, n, inner) natural; out: (n, C, inner); pre[k], post[x] complex phases (scale folded)
template <int P, int Q>
__global__ void __launch_bounds__(RoCfg<P, Q>::T)
k_readout_idft(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ pre,
               const float2* __restrict__ post, long long inner, int ncoils) {
  using S = FftShape<P, Q>;
  using R = RoCfg<P, Q>;
  constexpr int N = S::N, CB = R::CB, T = R::T, VSP = R::VSP;
  extern __shared__ __align__(16) float2 dsm[];
  float2* tw = dsm;  // W_N^{p k2} for the forward data flow; conjugated -> inverse transform
  float2* buf = dsm + N;
  const int tid = threadIdx.x;
  const long long c0 = (long long)blockIdx.x * CB;
  const int coil = blockIdx.y;
  const float2* src = in + (long long)coil * N * inner;
  const int ncols = (int)min((long long)CB, inner - c0);
  const int c = tid % CB, p = tid / CB;
  const bool cvalid = c < ncols;
  init_tw_s1<P, Q>(tw, tid, T);
  __syncthreads();
  // step 1 (inverse direction): DFT^-1_Q over q of v[p + P q], twiddle conj(W^{p k2})
  float2 r[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k = p + P * q;
    r[q] = cvalid ? cmul(src[(long long)k * inner + c0 + c], pre[k]) : make_float2(0.f, 0.f);
  }
  RegDFT<Q, true>::run(r);
  if (P > 1) {
#pragma unroll
    for (int k2 = 1; k2 < Q; ++k2) r[k2] = cmulc(tw[k2 * P + p], r[k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < Q; ++k2) buf[c * VSP + S::GS * k2 + p] = r[k2];
  __syncthreads();
  if (P > 1) {
    for (int it = tid; it < CB * Q; it += T) {
      const int cc = it % CB, k2 = it / CB;
      if (cc >= ncols) continue;
      float2 g[P];
      float2* gp = buf + cc * VSP + S::GS * k2;
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) g[k1] = gp[k1];
      RegDFT<P, true>::run(g);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) gp[k1] = g[k1];
    }
    __syncthreads();
  }
  // copy-out in natural order x: value of x sits at perm position P*(x % Q) + x / Q
  for (int e = tid; e < CB * N; e += T) {
    const int cc = e % CB, x = e / CB;
    if (cc >= ncols) continue;
    const float2 v = buf[cc * VSP + S::pad(S::perm_pos(x))];
    out[((long long)x * ncoils + coil) * inner + c0 + cc] = cmul(v, post[x]);
  }
}

template <int P, int Q>
int launch_readout(const float2* in, float2* out, const float2* pre, const float2* post, long long inner,
                   int ncoils, cudaStream_t st) {
  using R = RoCfg<P, Q>;
  const size_t smem = sizeof(float2) * (P * Q + R::CB * R::VSP);
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(k_readout_idft<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SR_ECUDA;
    cfg = true;
  }
  if (ncoils > 65535) return SR_EINVAL;
  dim3 grid((unsigned)((inner + R::CB - 1) / R::CB), ncoils);
  k_readout_idft<P, Q><<<grid, R::T, smem, st>>>(in, out, pre, post, inner, ncoils);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // namespace

extern "C" {

// in (ncoils, n, inner) -> out (n, ncoils, inner), centered unitary IDFT along n.
// pre/post: device phase vectors of length n (the host folds n^-1/2 and the
// centering phases into them).  in and out must not alias.
int sr_readout_idft(const sr_c64* in, sr_c64* out, const sr_c64* pre, const sr_c64* post, int ncoils, int n,
                    long long inner, void* stream) {
  if (ncoils < 1 || n < 2 || inner < 1 || (const void*)in == (const void*)out) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (n) {
#define X(N_, P_, Q_)                                                                                   \
  case N_:                                                                                             \
    return launch_readout<P_, Q_>((const float2*)in, (float2*)out, (const float2*)pre, (const float2*)post, \
                                  inner, ncoils, st);
    SR_FFT_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

}  // extern "C"
