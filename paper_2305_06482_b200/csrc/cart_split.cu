// K1 (split-column schedule): the Cartesian sketched normal operator for square images with the
// column transform split between the three passes, so that the middle pass needs no shared
// memory exchange and no barrier.
//
//   out_b = e( sum_j conj(c_bj) . F^H M'_b F (c_bj . (x_b - a_b)) )
//
// Reference: SenseOperator._forward/_adjoint (forward_model.py:168-180) over
// _CartesianMaskKernel (linops.py:344-364), called as adjoint(forward(.)) by the solvers
// (coil_sketch.py:126,133,197; solvers.py:175,248).
//
// Both axes have length N = P * Q and use the two-level split of fft2step.cuh.  Along y the
// row index is y = p + P q.  The column FFT's first step (DFT_Q over q for fixed p, times
// W_N^{p k2}) only combines the Q rows {p + P q}, so it is done by the pass that owns those
// rows anyway:
//   pass A (k_split_rowfwd, CTA = one p, its Q rows):  u = c_j (x - a); row FFTs (perm order
//          along x); per x position DFT_Q over the Q rows, twiddle W_N^{p k2}
//          -> workspace row P k2 + p
//   pass B (k_split_col, thread = (x position, k2)):     DFT_P over the P contiguous rows
//          P k2 + p, mask (perm order along y, unchanged), IDFT_P, twiddle conj W_N^{m1 k2}
//          -> workspace row P k2 + m1            (registers only: no shared memory, no barrier)
//   pass C (k_split_rowinv, CTA = one m1):              per x position IDFT_Q over the Q rows
//          P k2 + m1 -> rows m1 + P m2; row IFFTs; acc += conj(c_j) (.) ; epilogue
// The spectrum layout between A and B is the same perm order as cart.cu's, so the host mask
// tables (plan.py) are shared.  Traffic equals the three-pass schedule's; the arithmetic of the
// column transform moves from the issue-bound column pass to the HBM-bound row passes.
// Measured at config 1 (tools/sweep_k1.py --split): the middle pass drops from 250 to 202 us
// (HBM-bound, 6.0 TB/s), but the row passes, now with 16-row CTAs, three barriers per coil and
// ~25 % more arithmetic, take 251 + 252 us instead of 215 + 205 us: 0.72 ms per apply against
// 0.68 ms for cart.cu's schedule, which therefore stays the default (chunk 0).
#include "fft2step.cuh"

namespace {

template <int P, int Q>
struct SplitCfg {
  static constexpr int N = P * Q;
  static constexpr int T = N;  // threads: one per x position (column phases) = Q rows x P (row phases)
  using RS = RowShape<P, Q>;
  static constexpr int XS = N + ((((P % 16) - (N % 16)) % 16 + 16) % 16);  // x row stride = P (mod 16)
  static constexpr size_t SMEM_A = sizeof(float2) * (N + Q * RS::VS + Q * XS);
  static constexpr size_t SMEM_C = sizeof(float2) * (N + Q * RS::VS + Q * N);
  static constexpr bool OK = (N % 32) == 0 && N <= 1024 && P > 1 && (P % 4) == 0 && RS::VEC;
};

template <int P, int Q>
__global__ void __launch_bounds__(SplitCfg<P, Q>::T, 2)
k_split_rowfwd(const float2* __restrict__ x, const float2* __restrict__ anchor, const float2* __restrict__ maps,
               float2* __restrict__ ws, int ncoils, long long x_bstride, long long map_bstride, int jc) {
  using S = RowShape<P, Q>;
  using CF = SplitCfg<P, Q>;
  constexpr int N = CF::N, T = CF::T, XS = CF::XS;
  constexpr long long D = (long long)N * N;
  extern __shared__ __align__(16) float2 dsm[];
  float2* t1 = dsm;
  float2* buf = dsm + N;
  float2* xs = buf + Q * S::VS;
  const int tid = threadIdx.x;
  const int p = blockIdx.x, b = blockIdx.y;
  const int j0 = blockIdx.z * jc, j1 = min(ncoils, j0 + jc);  // coils of this CTA (smaller tail)
  const int lr = tid / P, px = tid % P;  // row phase: row p + P lr, x positions px + P qx
  init_tw_s1<P, Q>(t1, tid, T);
  const float2* mb = maps + b * map_bstride + (long long)(p + P * lr) * N + px;
  float2* wb = ws + (long long)b * ncoils * D + (long long)p * N + tid;
  float2 mcur[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) mcur[q] = __ldg(mb + j0 * D + P * q);
  {
    // u = x - a for the CTA's Q rows; thread tid loads position tid of every row (coalesced)
    const float2* xb = x + b * x_bstride + (long long)p * N + tid;
    const float2* ab = anchor ? anchor + b * x_bstride + (long long)p * N + tid : xb;
    float2 v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = __ldg(xb + (long long)P * i * N);
    if (anchor) {
#pragma unroll
      for (int i = 0; i < Q; ++i) v[i] = csub(v[i], __ldg(ab + (long long)P * i * N));
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) xs[i * XS + tid] = v[i];
  }
  __syncthreads();
  const float2* xr = xs + lr * XS + px;
  const int ppos = S::pad(tid);
  for (int j = j0; j < j1; ++j) {
    float2 r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = cmul(mcur[q], xr[P * q]);
    if (j + 1 < j1) {
      const float2* mn = mb + (j + 1) * D;
#pragma unroll
      for (int q = 0; q < Q; ++q) mcur[q] = __ldg(mn + P * q);
    }
    fft_s1_fwd<P, Q>(r, px, t1);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[lr * S::VS + S::GS * k2 + px] = r[k2];
    __syncthreads();
    for (int it = tid; it < Q * Q; it += T) {
      const int l2 = it / Q, k2 = it - l2 * Q;
      float2 g[P];
      float2* gp = buf + l2 * S::VS + S::GS * k2;
      lds_group<P, true>(g, gp);
      fft_s2_fwd<P>(g);
      sts_group<P, true>(gp, g);
    }
    __syncthreads();
    // column step 1 for x position tid: DFT_Q over the rows p + P q, twiddle W_N^{p k2}
    float2 v[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) v[q] = buf[q * S::VS + ppos];
    fft_s1_fwd<P, Q>(v, p, t1);
    float2* wj = wb + j * D;
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) wj[(long long)P * k2 * N] = v[k2];
    __syncthreads();  // buf is rewritten by the next coil
  }
}

// one thread per (x position, k2) of a slice; JC coils per CTA
template <int P, int Q>
__global__ void __launch_bounds__(SplitCfg<P, Q>::T, 3)
k_split_col(float2* __restrict__ ws, const uint8_t* __restrict__ maskT, long long mask_bstride, int ncoils,
            int jc) {
  using CF = SplitCfg<P, Q>;
  constexpr int N = CF::N;
  constexpr long long D = (long long)N * N;
  __shared__ float2 t2[P * Q];
  const int tid = threadIdx.x;
  const int k2 = blockIdx.x;
  const int j0 = blockIdx.y * jc, j1 = min(ncoils, j0 + jc);
  const int b = blockIdx.z;
  init_tw_s2<P, Q>(t2, tid, CF::T);
  uint32_t mw[P / 4];
  {
    const uint32_t* mk = reinterpret_cast<const uint32_t*>(maskT + b * mask_bstride + (long long)tid * N + P * k2);
#pragma unroll
    for (int w4 = 0; w4 < P / 4; ++w4) mw[w4] = __ldg(mk + w4);
  }
  __syncthreads();
  float2* img0 = ws + (long long)b * ncoils * D + (long long)P * k2 * N + tid;
  for (int j = j0; j < j1; ++j) {
    float2* img = img0 + j * D;
    float2 g[P];
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) g[k1] = img[(long long)k1 * N];
    fft_s2_fwd<P>(g);
#pragma unroll
    for (int w4 = 0; w4 < P / 4; ++w4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!((mw[w4] >> (8 * i)) & 0xffu)) g[4 * w4 + i] = make_float2(0.f, 0.f);
    }
    fft_s2_inv<P, Q>(g, k2, t2);
#pragma unroll
    for (int m1 = 0; m1 < P; ++m1) img[(long long)m1 * N] = g[m1];
  }
}

template <int P, int Q>
__global__ void __launch_bounds__(SplitCfg<P, Q>::T, 2)
k_split_rowinv(const float2* __restrict__ ws, const float2* __restrict__ maps, float2* __restrict__ out,
               int ncoils, long long x_bstride, long long map_bstride, const float4* __restrict__ coef,
               const float2* __restrict__ u, const float2* __restrict__ d, float oscale) {
  using S = RowShape<P, Q>;
  using CF = SplitCfg<P, Q>;
  constexpr int N = CF::N, T = CF::T;
  constexpr long long D = (long long)N * N;
  extern __shared__ __align__(16) float2 dsm[];
  float2* t2 = dsm;
  float2* buf = dsm + N;
  float2* stage = buf + Q * S::VS;  // [Q][N]: this thread's column values of the next coil (cp.async)
  const int tid = threadIdx.x;
  const int m1 = blockIdx.x, b = blockIdx.y;
  const int lr = tid / P, px = tid % P;  // row phase: output row m1 + P lr
  init_tw_s2<P, Q>(t2, tid, T);
  float2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_float2(0.f, 0.f);
  const long long rowoff = (long long)(m1 + P * lr) * N + px;
  const float2* mb = maps + b * map_bstride + rowoff;
  const float2* wb = ws + (long long)b * ncoils * D + (long long)m1 * N + tid;
  const int ppos = S::pad(tid);
  auto issue = [&](int j) {
    const float2* wj = wb + j * D;
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) cp_async8(stage + k2 * N + tid, wj + (long long)P * k2 * N);
    cp_async_commit();
  };
  issue(0);
  __syncthreads();
  for (int j = 0; j < ncoils; ++j) {
    // column step 1': IDFT_Q over the rows P k2 + m1 -> rows m1 + P m2
    float2 v[Q];
    cp_async_wait<0>();
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) v[k2] = stage[k2 * N + tid];
    if (j + 1 < ncoils) issue(j + 1);  // own slots only: no barrier needed
    fft_s1_inv<Q>(v);
#pragma unroll
    for (int m2 = 0; m2 < Q; ++m2) buf[m2 * S::VS + ppos] = v[m2];
    __syncthreads();
    for (int it = tid; it < Q * Q; it += T) {
      const int l2 = it / Q, k2 = it - l2 * Q;
      float2 g[P];
      float2* gp = buf + l2 * S::VS + S::GS * k2;
      lds_group<P, true>(g, gp);
      fft_s2_inv<P, Q>(g, k2, t2);
      sts_group<P, true>(gp, g);
    }
    __syncthreads();
    // this coil's map values are in flight during the row IFFT's last step
    float2 mreg[Q];
    const float2* mr = mb + j * D;
#pragma unroll
    for (int q = 0; q < Q; ++q) mreg[q] = __ldg(mr + P * q);
    float2 r[Q];
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) r[k2] = buf[lr * S::VS + S::GS * k2 + px];
    fft_s1_inv<Q>(r);
#pragma unroll
    for (int q = 0; q < Q; ++q) cfma_conj(acc[q], mreg[q], r[q]);
    __syncthreads();  // buf is rewritten by the next coil
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = cscale(acc[q], oscale);
  const long long off = b * x_bstride + rowoff;
  if (coef == nullptr) {
#pragma unroll
    for (int q = 0; q < Q; ++q) out[off + P * q] = acc[q];
  } else {
    const float4 c = coef[b];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      float2 v = cscale(acc[q], c.x);
      if (u) { const float2 uu = u[off + P * q]; v.x = fmaf(c.y, uu.x, v.x); v.y = fmaf(c.y, uu.y, v.y); }
      if (d) { const float2 dd = d[off + P * q]; v.x = fmaf(c.z, dd.x, v.x); v.y = fmaf(c.z, dd.y, v.y); }
      out[off + P * q] = v;
    }
  }
}

int g_split_jc = 4;   // coils per CTA of the middle pass
int g_split_ja = 2;   // coil ranges (CTAs) per row group of the first pass

template <int P, int Q>
int launch_split(const float2* x, const float2* anchor, const float2* maps, long long mbs, const uint8_t* maskT,
                 long long kbs, float2* out, float2* ws, int batch, int ncoils, const float4* coef,
                 const float2* u, const float2* d, cudaStream_t st) {
  using CF = SplitCfg<P, Q>;
  constexpr int N = CF::N;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(k_split_rowfwd<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)CF::SMEM_A) != cudaSuccess ||
        cudaFuncSetAttribute(k_split_rowinv<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)CF::SMEM_C) != cudaSuccess)
      return SR_ECUDA;
    configured = true;
  }
  const long long D = (long long)N * N;
  const int ja = g_split_ja < ncoils ? g_split_ja : ncoils, jca = (ncoils + ja - 1) / ja;
  k_split_rowfwd<P, Q><<<dim3(P, batch, (ncoils + jca - 1) / jca), CF::T, CF::SMEM_A, st>>>(x, anchor, maps, ws,
                                                                                          ncoils, D, mbs, jca);
  SR_CHECK_LAUNCH();
  const int jc = g_split_jc < ncoils ? g_split_jc : ncoils;
  k_split_col<P, Q><<<dim3(Q, (ncoils + jc - 1) / jc, batch), CF::T, 0, st>>>(ws, maskT, kbs, ncoils, jc);
  SR_CHECK_LAUNCH();
  k_split_rowinv<P, Q><<<dim3(P, batch), CF::T, CF::SMEM_C, st>>>(ws, maps, out, ncoils, D, mbs, coef, u, d,
                                                                  (float)(1.0 / (double)D));
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// instantiated square sizes (N, P, Q)
#define SR_SPLIT_SIZES(X) X(320, 20, 16) X(256, 16, 16) X(384, 24, 16) X(160, 16, 10)

}  // namespace

int sr_split_normal_supported_n(int n) {
  switch (n) {
#define X(N_, P_, Q_) \
  case N_: return SplitCfg<P_, Q_>::OK ? 1 : 0;
    SR_SPLIT_SIZES(X)
#undef X
    default: return 0;
  }
}

int sr_split_normal(const float2* x, const float2* anchor, const float2* maps, long long mbs,
                    const uint8_t* maskT, long long kbs, float2* out, float2* ws, int batch, int ncoils, int n,
                    const float4* coef, const float2* u, const float2* d, cudaStream_t st) {
  switch (n) {
#define X(N_, P_, Q_)                                                                                 \
  case N_:                                                                                            \
    if constexpr (SplitCfg<P_, Q_>::OK)                                                               \
      return launch_split<P_, Q_>(x, anchor, maps, mbs, maskT, kbs, out, ws, batch, ncoils, coef, u, d, st); \
    return SR_EUNSUPPORTED;
    SR_SPLIT_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

extern "C" int sr_split_tune(int jc, int ja) {
  if (jc < 1 || ja < 1) return SR_EINVAL;
  g_split_jc = jc;
  g_split_ja = ja;
  return SR_OK;
}
