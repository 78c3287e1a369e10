// K5: coil-dimension contraction  out[b, i, :] = sum_k S[b, i, k] * in[b, k, :]
//
// Serves two reference computations:
//   sketch_maps            /root/reference/pkg/src/sketchrecon/sketching.py:97-103   (S real, Chat x C)
//   coil_compress_svd rot  /root/reference/pkg/src/sketchrecon/forward_model.py:268-269 (comp complex)
// Bandwidth-bound: each thread owns one voxel, keeps up to 32 input coils in
// registers (coalesced complex64 loads across the warp) and emits every output
// coil from the coefficient matrix broadcast out of shared memory.
#include "common.cuh"

namespace {

constexpr int KCHUNK = 32;

__global__ void __launch_bounds__(256)
k_coil_contract(const float2* __restrict__ in, float2* __restrict__ out,
                const float2* __restrict__ S, long long s_bstride, int cout, int cin,
                long long D, long long in_bstride, long long out_bstride, int k0, int kn,
                int accumulate) {
  extern __shared__ float2 sS[];  // cout x kn slice of S
  const int b = blockIdx.y;
  const float2* Sb = S + b * s_bstride;
  for (int e = threadIdx.x; e < cout * kn; e += blockDim.x) {
    const int i = e / kn, k = e - i * kn;
    sS[e] = Sb[(long long)i * cin + k0 + k];
  }
  __syncthreads();
  const float2* ib = in + b * in_bstride + (long long)k0 * D;
  float2* ob = out + b * out_bstride;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < D;
       d += (long long)gridDim.x * blockDim.x) {
    float2 v[KCHUNK];
#pragma unroll
    for (int k = 0; k < KCHUNK; ++k) v[k] = (k < kn) ? __ldg(ib + k * D + d) : make_float2(0.f, 0.f);
    for (int i = 0; i < cout; ++i) {
      float2 acc = accumulate ? ob[i * D + d] : make_float2(0.f, 0.f);
      const float2* si = sS + i * kn;
#pragma unroll
      for (int k = 0; k < KCHUNK; ++k) {
        if (k < kn) {
          const float2 s = si[k];
          acc.x = fmaf(s.x, v[k].x, fmaf(-s.y, v[k].y, acc.x));
          acc.y = fmaf(s.x, v[k].y, fmaf(s.y, v[k].x, acc.y));
        }
      }
      ob[i * D + d] = acc;
    }
  }
}

// Real coefficient matrix (the sketch S~ of sketching.py:69-94 is real: identity rows and
// +-scale Rademacher rows): 2 FMAs per complex MAC instead of 4, two voxels per thread (16-byte
// loads / stores) so each broadcast coefficient serves 4 FMAs, and the input coils streamed in
// chunks of 8 with all CO outputs accumulated in registers.
template <int CO>
__global__ void __launch_bounds__(256)
k_coil_contract_real(const float4* __restrict__ in, float4* __restrict__ out, const float* __restrict__ S,
                     long long s_bstride, int cout, int cin, long long D2, long long in_bstride2,
                     long long out_bstride2) {
  extern __shared__ float sR[];  // cout x cin
  const int b = blockIdx.y;
  const float* Sb = S + b * s_bstride;
  for (int e = threadIdx.x; e < cout * cin; e += blockDim.x) sR[e] = Sb[e];
  __syncthreads();
  const float4* ib = in + b * in_bstride2;
  float4* ob = out + b * out_bstride2;
  constexpr int KC = 8;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < D2;
       d += (long long)gridDim.x * blockDim.x) {
    float4 acc[CO];
#pragma unroll
    for (int i = 0; i < CO; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < cin; k0 += KC) {
      float4 v[KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) v[k] = (k0 + k < cin) ? __ldg(ib + (long long)(k0 + k) * D2 + d) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < CO; ++i) {
        if (i >= cout) break;
        const float* si = sR + i * cin + k0;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          if (k0 + k < cin) {
            const float c = si[k];
            acc[i].x = fmaf(c, v[k].x, acc[i].x);
            acc[i].y = fmaf(c, v[k].y, acc[i].y);
            acc[i].z = fmaf(c, v[k].z, acc[i].z);
            acc[i].w = fmaf(c, v[k].w, acc[i].w);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CO; ++i) {
      if (i >= cout) break;
      ob[(long long)i * D2 + d] = acc[i];
    }
  }
}

}  // namespace

extern "C" {

// S: (batch or 1, cout, cin) float32 (a real coefficient matrix); s_bstride = 0 shares S.
// D must be even (two voxels per thread); in/out 16-byte aligned.
int sr_coil_contract_real(const sr_c64* in, sr_c64* out, const float* S, long long s_bstride, int batch, int cout,
                          int cin, long long D, long long in_bstride, long long out_bstride, void* stream) {
  if (batch < 1 || cout < 1 || cin < 1 || D < 2 || (D & 1) || (in_bstride & 1) || (out_bstride & 1))
    return SR_EINVAL;
  if ((const void*)in == (const void*)out) return SR_EINVAL;
  if ((((uintptr_t)in) | ((uintptr_t)out)) & 15) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  const long long D2 = D / 2;
  long long blocks = (D2 + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  dim3 grid((unsigned)blocks, batch);
  const size_t smem = sizeof(float) * cout * cin;
  if (smem > 48 * 1024) return SR_EINVAL;
#define SR_LAUNCH_CR(CO_)                                                                                     \
  k_coil_contract_real<CO_><<<grid, threads, smem, st>>>((const float4*)in, (float4*)out, S, s_bstride, cout, \
                                                         cin, D2, in_bstride / 2, out_bstride / 2)
  if (cout <= 8) SR_LAUNCH_CR(8);
  else if (cout <= 12) SR_LAUNCH_CR(12);
  else if (cout <= 16) SR_LAUNCH_CR(16);
  else if (cout <= 32) SR_LAUNCH_CR(32);
  else return SR_EUNSUPPORTED;
#undef SR_LAUNCH_CR
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// S: (batch or 1, cout, cin) complex64 (imag 0 for a real sketch); s_bstride = 0 shares S.
int sr_coil_contract(const sr_c64* in, sr_c64* out, const sr_c64* S, long long s_bstride,
                     int batch, int cout, int cin, long long D, long long in_bstride,
                     long long out_bstride, void* stream) {
  if (batch < 1 || cout < 1 || cin < 1 || D < 1) return SR_EINVAL;
  if ((const void*)in == (const void*)out) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  long long blocks = (D + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  dim3 grid((unsigned)blocks, batch);
  for (int k0 = 0; k0 < cin; k0 += KCHUNK) {
    const int kn = (cin - k0) < KCHUNK ? (cin - k0) : KCHUNK;
    const size_t smem = sizeof(float2) * cout * kn;
    if (smem > 48 * 1024) {
      if (cudaFuncSetAttribute(k_coil_contract, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess)
        return SR_ECUDA;
    }
    k_coil_contract<<<grid, threads, smem, st>>>((const float2*)in, (float2*)out,
                                                 (const float2*)S, s_bstride, cout, cin, D,
                                                 in_bstride, out_bstride, k0, kn, k0 > 0);
    SR_CHECK_LAUNCH();
  }
  return SR_OK;
}

}  // extern "C"
