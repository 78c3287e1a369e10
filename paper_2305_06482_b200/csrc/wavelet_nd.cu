// K6 (n-D): one axis of one level of the periodic DB4 wavelet, for 1-D and 3-D
// grids (2-D grids use the tiled kernels of wavelet.cu).  BASELINE config 4
// reconstructs a 256 x 256 x 160 volume, so its L1-wavelet prox is 3-D.
//
// Reference: _analysis_axis / _synthesis_axis (linops.py:619-651); WaveletOp
// applies the analysis along axes 0..d-1 on the low-pass corner of each level
// and the synthesis in reverse axis order (linops.py:677-702).  Each launch
// here is one axis over the (h0, h1, h2) corner of arrays shaped (n0, n1, n2)
// (leading 1s for lower dimensions); src and dst never alias.  The last axis of
// a level may apply the soft threshold to the detail sub-bands (and to the
// low-pass corner at the coarsest level) and collect sum |c| partials; the last
// synthesis launch may apply the FISTA momentum epilogue.
#include "common.cuh"

#ifndef SR_WAV_AXIS_GRID
#define SR_WAV_AXIS_GRID (148 * 16)
#endif

namespace {

struct AxisArgs {
  const float2* src;
  float2* dst;
  int h[3];         // region extent
  long long st[3];  // element strides of the full array
  long long bs;     // slice stride
  int axis;
  int inverse;
  const float* thresh;  // per-slice thresholds (device) or null
  float hthresh;        // host threshold (< 0: none)
  int thr_enable;       // apply threshold (last axis of an analysis level)
  int last_level;       // threshold the low-pass corner too
  double* l1part;       // (batch, gridDim.x) partial sums or null
  float2* zout;         // synthesis epilogue z = v + beta (v - xold)
  const float2* xold;
  float beta;
};

// periodic index j in [-p, 2p) (the common case) without an integer division
__device__ __forceinline__ int pwrap(int j, int p) {
  if (j >= p) j -= p;
  else if (j < 0) j += p;
  if ((unsigned)j >= (unsigned)p) {  // tiny levels: more than one period away
    j %= p;
    if (j < 0) j += p;
  }
  return j;
}

// filter taps as compile-time constants (hi[k] = (-1)^k lo[7 - k])
__device__ __forceinline__ constexpr float k_lo(int k) {
  return k == 0 ? -0.010597401785069032105f : k == 1 ? 0.032883011666885199735f
       : k == 2 ? 0.030841381835560763627f : k == 3 ? -0.18703481171909308408f
       : k == 4 ? -0.027983769416859854211f : k == 5 ? 0.63088076792985890788f
       : k == 6 ? 0.71484657055291564709f : 0.23037781330889650086f;
}
__device__ __forceinline__ constexpr float k_hi(int k) { return (k & 1) ? -k_lo(7 - k) : k_lo(7 - k); }

// One work item makes an output PAIR along the axis from shared loads: analysis item i reads the 8
// inputs 2i .. 2i + 7 once for the low-pass output i and the high-pass output hn + i; synthesis item j
// reads lo / hi at j, j - 1, j - 2, j - 3 once for the outputs 2j and 2j + 1 (taps 2t and 2t + 1).  The
// per-output form loaded 8 values per output and indexed the tap tables by the output's band / parity.
__global__ void __launch_bounds__(256) k_wav_axis(AxisArgs a) {
  const int b = blockIdx.y;
  const int ax = a.axis;
  const int n = a.h[ax], hn = n >> 1;
  // items: the level corner with the extent along `ax` halved (< 2^30, see sr_wavelet_axis)
  int hx[3] = {a.h[0], a.h[1], a.h[2]};
  hx[ax] = hn;
  const int total = hx[0] * hx[1] * hx[2];
  const long long sa = a.st[ax];
  const float2* src = a.src + b * a.bs;
  float2* dst = a.dst + b * a.bs;
  double part = 0.0;
  const float t = a.thresh ? a.thresh[b] : a.hthresh;
  const bool thr = a.thresh || a.hthresh >= 0.f;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int q = e / hx[2];
    const int i2 = e - q * hx[2];
    const int i0 = q / hx[1];
    const int i1 = q - i0 * hx[1];
    const int ii[3] = {i0, i1, i2};
    const int i = ii[ax];
    const long long line = i0 * a.st[0] + i1 * a.st[1] + i2 * a.st[2] - (long long)i * sa;  // start of the line along `ax`
    if (!a.inverse) {
      float2 lo = make_float2(0.f, 0.f), hi = lo;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 x = src[line + (long long)pwrap(2 * i + k, n) * sa];
        lo.x = fmaf(k_lo(k), x.x, lo.x);
        lo.y = fmaf(k_lo(k), x.y, lo.y);
        hi.x = fmaf(k_hi(k), x.x, hi.x);
        hi.y = fmaf(k_hi(k), x.y, hi.y);
      }
      if (a.thr_enable) {
        // the high-pass output is a detail coefficient; the low-pass one is final only outside the
        // low-pass corner of the other axes, or at the last level
        bool lowpass = true;
#pragma unroll
        for (int d = 0; d < 3; ++d)
          if (d != ax && a.h[d] > 1 && ii[d] >= (a.h[d] >> 1)) lowpass = false;
        const bool lo_final = !lowpass || a.last_level;
        if (thr) {
          const float mh = sqrtf(hi.x * hi.x + hi.y * hi.y);
          const float sh = (mh > t) ? (mh - t) / mh : 0.f;
          hi = make_float2(hi.x * sh, hi.y * sh);
          if (lo_final) {
            const float ml = sqrtf(lo.x * lo.x + lo.y * lo.y);
            const float sl = (ml > t) ? (ml - t) / ml : 0.f;
            lo = make_float2(lo.x * sl, lo.y * sl);
          }
        }
        if (a.l1part) {
          if (lo_final) part += sqrt((double)lo.x * lo.x + (double)lo.y * lo.y);
          part += sqrt((double)hi.x * hi.x + (double)hi.y * hi.y);
        }
      }
      dst[line + (long long)i * sa] = lo;
      dst[line + (long long)(hn + i) * sa] = hi;
    } else {
      const long long oe = line + (long long)(2 * i) * sa, oo = oe + sa;
      float2 xe = make_float2(0.f, 0.f), xo = xe;
      if (a.zout) {
        xe = a.xold[b * a.bs + oe];
        xo = a.xold[b * a.bs + oo];
      }
      float2 ve = make_float2(0.f, 0.f), vo = ve;
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const int p = pwrap(i - tt, hn);
        const float2 lo = src[line + (long long)p * sa];
        const float2 hi = src[line + (long long)(hn + p) * sa];
        ve.x = fmaf(k_lo(2 * tt), lo.x, fmaf(k_hi(2 * tt), hi.x, ve.x));
        ve.y = fmaf(k_lo(2 * tt), lo.y, fmaf(k_hi(2 * tt), hi.y, ve.y));
        vo.x = fmaf(k_lo(2 * tt + 1), lo.x, fmaf(k_hi(2 * tt + 1), hi.x, vo.x));
        vo.y = fmaf(k_lo(2 * tt + 1), lo.y, fmaf(k_hi(2 * tt + 1), hi.y, vo.y));
      }
      if (a.zout) {
        a.zout[b * a.bs + oe] = make_float2(fmaf(a.beta, ve.x - xe.x, ve.x), fmaf(a.beta, ve.y - xe.y, ve.y));
        a.zout[b * a.bs + oo] = make_float2(fmaf(a.beta, vo.x - xo.x, vo.x), fmaf(a.beta, vo.y - xo.y, vo.y));
      }
      dst[oe] = ve;
      dst[oo] = vo;
    }
  }
  if (a.l1part) {
    __shared__ double red[256];
    red[threadIdx.x] = part;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) a.l1part[(long long)b * gridDim.x + blockIdx.x] = red[0];
  }
}

}  // namespace

extern "C" {

int sr_wavelet_axis_nblocks(void) { return 148 * 4; }

// One axis of one level over the (h0, h1, h2) corner of (n0, n1, n2) arrays.
int sr_wavelet_axis(const sr_c64* src, sr_c64* dst, int h0, int h1, int h2, int n1, int n2, long long bs,
                    int batch, int axis, int inverse, const float* thresh, float hthresh, int thr_enable,
                    int last_level, double* l1part, sr_c64* zout, const sr_c64* xold, float beta,
                    void* stream) {
  if (batch < 1 || axis < 0 || axis > 2 || h0 < 1 || h1 < 1 || h2 < 1) return SR_EINVAL;
  const int h[3] = {h0, h1, h2};
  if (h[axis] < 2 || (h[axis] & 1)) return SR_EINVAL;
  if ((long long)h0 * h1 * h2 >= (1LL << 31)) return SR_EINVAL;
  if ((const void*)src == (const void*)dst) return SR_EINVAL;
  AxisArgs a;
  a.src = (const float2*)src;
  a.dst = (float2*)dst;
  a.h[0] = h0; a.h[1] = h1; a.h[2] = h2;
  a.st[0] = (long long)n1 * n2; a.st[1] = n2; a.st[2] = 1;
  a.bs = bs;
  a.axis = axis;
  a.inverse = inverse;
  a.thresh = thresh;
  a.hthresh = hthresh;
  a.thr_enable = thr_enable;
  a.last_level = last_level;
  a.l1part = l1part;
  a.zout = (float2*)zout;
  a.xold = (const float2*)xold;
  a.beta = beta;
  // without per-block partials the grid is 2368 blocks (config-4 prox with the pair kernel: 1184
  // blocks 0.663 ms, 2368 0.672, 4736 0.659 -- flat; the per-output kernel had measured 592 blocks
  // 1.17 ms, 2368 1.04, one element per thread 1.49 ms)
  const long long total = (long long)h0 * h1 * h2 / 2;  // one work item per output pair along the axis
  long long nb = l1part ? sr_wavelet_axis_nblocks() : min((total + 255) / 256, (long long)SR_WAV_AXIS_GRID);
  if (nb > 0x7fffffffLL) nb = 0x7fffffffLL;
  dim3 grid((unsigned)nb, batch);
  k_wav_axis<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // extern "C"
