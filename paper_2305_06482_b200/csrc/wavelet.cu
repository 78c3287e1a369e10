// K6: orthonormal Daubechies-4 (8-tap) multilevel periodic wavelet and the
// fused L1 prox  x = Psi^H soft(Psi v, t)  (+ FISTA momentum epilogue).
//
// Reference:
//   _DB4_LO/_DB4_HI                    /root/reference/pkg/src/sketchrecon/linops.py:593-606
//   _analysis_axis / _synthesis_axis   linops.py:619-651
//   WaveletOp._forward / _adjoint      linops.py:677-702  ([lo|hi] in place, recurse on lo corner)
//   prox_l1                            /root/reference/pkg/src/sketchrecon/solvers.py:129-135
//   Regularizer.prox (l1-wavelet)      solvers.py:78-80
//
// One kernel launch per level and direction.  Level l works on the top-left
// (n0>>l) x (n1>>l) [x (n2>>l)] corner.  Analysis level l reads its input
// from src_l and writes the four (eight in 3-D) subbands to buffer buf(l)
// (alternating between two coefficient buffers), so no launch reads what
// another block of the same launch writes.  Synthesis level l reads buf(l)
// and writes the reconstructed corner into buf(l-1)'s low-pass quadrant
// (already consumed by the analysis), or into the output for l = 0.
#include "common.cuh"

namespace {

__constant__ float c_lo[8] = {
    -0.010597401785069032105f, 0.032883011666885199735f, 0.030841381835560763627f,
    -0.18703481171909308408f, -0.027983769416859854211f, 0.63088076792985890788f,
    0.71484657055291564709f, 0.23037781330889650086f};
// hi = reverse(lo), odd taps negated
__constant__ float c_hi[8] = {
    0.23037781330889650086f, -0.71484657055291564709f, 0.63088076792985890788f,
    0.027983769416859854211f, -0.18703481171909308408f, -0.030841381835560763627f,
    0.032883011666885199735f, 0.010597401785069032105f};

// the same taps as compile-time constants (immediate operands where the tap index is known)
__device__ __forceinline__ constexpr float k_lo(int k) {
  return k == 0 ? -0.010597401785069032105f : k == 1 ? 0.032883011666885199735f
       : k == 2 ? 0.030841381835560763627f : k == 3 ? -0.18703481171909308408f
       : k == 4 ? -0.027983769416859854211f : k == 5 ? 0.63088076792985890788f
       : k == 6 ? 0.71484657055291564709f : 0.23037781330889650086f;
}
// hi[k] = (-1)^k lo[7 - k]
__device__ __forceinline__ constexpr float k_hi(int k) { return (k & 1) ? -k_lo(7 - k) : k_lo(7 - k); }

__device__ __forceinline__ float2 soft(float2 v, float t) {
  // v * max(|v| - t, 0) / |v|, zeros stay zero
  const float m = sqrtf(v.x * v.x + v.y * v.y);
  const float s = (m > t) ? (m - t) / m : 0.f;
  return make_float2(v.x * s, v.y * s);
}

__device__ __forceinline__ int wrap(int i, int n) {
  // periodic index; the tiles reach at most one period past either edge except on the smallest
  // levels, so the integer division is off the common path
  if ((unsigned)i < (unsigned)n) return i;
  if (i >= n && i < 2 * n) return i - n;
  if (i < 0 && i >= -n) return i + n;
  i %= n;
  return i < 0 ? i + n : i;
}

constexpr int TI = 16, TJ = 16;            // analysis output tile (per subband)
constexpr int AR = 2 * TI + 6, AC = 2 * TJ + 6;

// ---------------------------------------------------------------- 2-D analysis
// region h x w at the top-left of arrays with row stride ld, slice stride bs.
__global__ void __launch_bounds__(256)
k_wav_ana2(const float2* __restrict__ src, float2* __restrict__ dst, int h, int w, int ld,
           long long bs, const float* __restrict__ thresh, float hthresh, int last,
           double* __restrict__ l1part) {
  __shared__ float2 tin[AR][AC + 1];
  __shared__ float2 tlo[AR][TJ + 1], thi[AR][TJ + 1];
  const int b = blockIdx.z;
  const int hh = h >> 1, hw = w >> 1;
  const int i0 = blockIdx.y * TI, j0 = blockIdx.x * TJ;
  const float2* s = src + b * bs;
  float2* o = dst + b * bs;
  const int tid = threadIdx.y * TJ + threadIdx.x;
  if (2 * i0 + AR <= h && 2 * j0 + AC <= w && !(ld & 1) && !(reinterpret_cast<size_t>(s) & 15)) {
    // interior tile: no wrap, two pixels per 16-byte load (even column start and row stride)
    for (int e = tid; e < AR * (AC / 2); e += 256) {
      const int r = e / (AC / 2), c = 2 * (e - r * (AC / 2));
      const float4 v = *reinterpret_cast<const float4*>(s + (long long)(2 * i0 + r) * ld + 2 * j0 + c);
      tin[r][c] = make_float2(v.x, v.y);
      tin[r][c + 1] = make_float2(v.z, v.w);
    }
  } else {
    for (int e = tid; e < AR * AC; e += 256) {
      const int r = e / AC, c = e - r * AC;
      tin[r][c] = s[(long long)wrap(2 * i0 + r, h) * ld + wrap(2 * j0 + c, w)];
    }
  }
  __syncthreads();
  for (int e = tid; e < AR * TJ; e += 256) {
    const int r = e / TJ, j = e - r * TJ;
    float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 v = tin[r][2 * j + k];
      lo.x = fmaf(c_lo[k], v.x, lo.x); lo.y = fmaf(c_lo[k], v.y, lo.y);
      hi.x = fmaf(c_hi[k], v.x, hi.x); hi.y = fmaf(c_hi[k], v.y, hi.y);
    }
    tlo[r][j] = lo;
    thi[r][j] = hi;
  }
  __syncthreads();
  const int i = threadIdx.y, j = threadIdx.x;
  const int gi = i0 + i, gj = j0 + j;
  double part = 0.0;
  if (gi < hh && gj < hw) {
    float2 ll = make_float2(0.f, 0.f), lh = ll, hl = ll, hh2 = ll;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 a = tlo[2 * i + k][j], c = thi[2 * i + k][j];
      ll.x = fmaf(c_lo[k], a.x, ll.x); ll.y = fmaf(c_lo[k], a.y, ll.y);
      hl.x = fmaf(c_hi[k], a.x, hl.x); hl.y = fmaf(c_hi[k], a.y, hl.y);
      lh.x = fmaf(c_lo[k], c.x, lh.x); lh.y = fmaf(c_lo[k], c.y, lh.y);
      hh2.x = fmaf(c_hi[k], c.x, hh2.x); hh2.y = fmaf(c_hi[k], c.y, hh2.y);
    }
    const bool thr = (thresh != nullptr) || (hthresh >= 0.f);
    const float t = thresh ? thresh[b] : hthresh;
    if (thr) {
      lh = soft(lh, t); hl = soft(hl, t); hh2 = soft(hh2, t);
      if (last) ll = soft(ll, t);
    }
    if (l1part) {
      part = sqrt((double)lh.x * lh.x + (double)lh.y * lh.y) +
             sqrt((double)hl.x * hl.x + (double)hl.y * hl.y) +
             sqrt((double)hh2.x * hh2.x + (double)hh2.y * hh2.y);
      if (last) part += sqrt((double)ll.x * ll.x + (double)ll.y * ll.y);
    }
    o[(long long)gi * ld + gj] = ll;
    o[(long long)gi * ld + hw + gj] = lh;
    o[(long long)(hh + gi) * ld + gj] = hl;
    o[(long long)(hh + gi) * ld + hw + gj] = hh2;
  }
  if (l1part) {
    __shared__ double red[256];
    red[tid] = part;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
      if (tid < st) red[tid] += red[tid + st];
      __syncthreads();
    }
    if (tid == 0) {
      const long long blk = (long long)blockIdx.y * gridDim.x + blockIdx.x;
      l1part[(long long)b * gridDim.x * gridDim.y + blk] = red[0];
    }
  }
}

// --------------------------------------------------------------- 2-D synthesis
constexpr int SM = 32, SN = 32;                 // output tile
constexpr int SR_ = SM / 2 + 3, SC_ = SN / 2 + 3;  // coefficient tile per quadrant

// out[b] region h x w  <-  quadrants of coef[b] region h x w.
// Epilogue (final level): xnew = synth; if zout: z = xnew + beta (xnew - xold)
__global__ void __launch_bounds__(256)
k_wav_syn2(const float2* __restrict__ coef, float2* __restrict__ out, int h, int w, int ld,
           long long bs, float2* __restrict__ zout, const float2* __restrict__ xold,
           float beta) {
  __shared__ float2 q[4][SR_][SC_ + 1];
  __shared__ float2 ulo[SR_][SN + 1], uhi[SR_][SN + 1];
  const int b = blockIdx.z;
  const int hh = h >> 1, hw = w >> 1;
  const int m0 = blockIdx.y * SM, n0 = blockIdx.x * SN;
  const int ci0 = m0 / 2 - 3, cj0 = n0 / 2 - 3;
  const float2* cb = coef + b * bs;
  const int tid = threadIdx.x;
  const bool interior = ci0 >= 0 && ci0 + SR_ <= hh && cj0 >= 0 && cj0 + SC_ <= hw;
  if (interior && cj0 >= 1 && !(ld & 1) && !(hw & 1) && !(reinterpret_cast<size_t>(cb) & 15)) {
    // interior tile, even row stride and quadrant offset: rows of 20 cells from the even column
    // cj0 - 1 as ten 16-byte loads (the first cell is outside the tile)
    for (int e = tid; e < 4 * SR_ * 10; e += 256) {
      const int row = e / 10, pr = e - row * 10;
      const int qd = row / SR_, r = row - qd * SR_;
      const int oi = (qd & 2) ? hh : 0, oj = (qd & 1) ? hw : 0;
      const float4 v = *reinterpret_cast<const float4*>(cb + (long long)(oi + ci0 + r) * ld + oj + cj0 - 1 + 2 * pr);
      if (pr > 0) q[qd][r][2 * pr - 1] = make_float2(v.x, v.y);
      q[qd][r][2 * pr] = make_float2(v.z, v.w);
    }
  } else
  for (int e = tid; e < 4 * SR_ * SC_; e += 256) {
    const int qd = e / (SR_ * SC_);
    const int rem = e - qd * SR_ * SC_;
    const int r = rem / SC_, c = rem - r * SC_;
    const int gi = interior ? ci0 + r : wrap(ci0 + r, hh), gj = interior ? cj0 + c : wrap(cj0 + c, hw);
    const int oi = (qd & 2) ? hh : 0, oj = (qd & 1) ? hw : 0;
    q[qd][r][c] = cb[(long long)(oi + gi) * ld + oj + gj];
  }
  __syncthreads();
  // Each task makes the two outputs of a pair (even, odd position): they read the same four
  // coefficients per band (position j + 3 - t of the tile for taps k = 2t and 2t + 1), so the loads are
  // shared and every filter tap is a compile-time constant (the per-output form indexed the
  // coefficient tables by the output's parity).  Accumulation order per output as before.
  // undo axis 1: u_lo0[r][n] from (LL, LH); u_hi0[r][n] from (HL, HH)
  for (int e = tid; e < SR_ * (SN / 2); e += 256) {
    const int r = e / (SN / 2), jp = e - r * (SN / 2);
    float2 ae = make_float2(0.f, 0.f), ce = ae, ao = ae, co = ae;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = jp + 3 - t;  // ((n0 + 2 jp [+ 1]) - k) / 2 - cj0
      const float2 ll = q[0][r][jj], lh = q[1][r][jj], hl = q[2][r][jj], h2 = q[3][r][jj];
      ae.x = fmaf(k_lo(2 * t), ll.x, fmaf(k_hi(2 * t), lh.x, ae.x));
      ae.y = fmaf(k_lo(2 * t), ll.y, fmaf(k_hi(2 * t), lh.y, ae.y));
      ce.x = fmaf(k_lo(2 * t), hl.x, fmaf(k_hi(2 * t), h2.x, ce.x));
      ce.y = fmaf(k_lo(2 * t), hl.y, fmaf(k_hi(2 * t), h2.y, ce.y));
      ao.x = fmaf(k_lo(2 * t + 1), ll.x, fmaf(k_hi(2 * t + 1), lh.x, ao.x));
      ao.y = fmaf(k_lo(2 * t + 1), ll.y, fmaf(k_hi(2 * t + 1), lh.y, ao.y));
      co.x = fmaf(k_lo(2 * t + 1), hl.x, fmaf(k_hi(2 * t + 1), h2.x, co.x));
      co.y = fmaf(k_lo(2 * t + 1), hl.y, fmaf(k_hi(2 * t + 1), h2.y, co.y));
    }
    ulo[r][2 * jp] = ae;
    ulo[r][2 * jp + 1] = ao;
    uhi[r][2 * jp] = ce;
    uhi[r][2 * jp + 1] = co;
  }
  __syncthreads();
  float2* ob = out + b * bs;
  for (int e = tid; e < (SM / 2) * SN; e += 256) {
    const int ip = e / SN, nn = e - ip * SN;
    const int m = m0 + 2 * ip, n = n0 + nn;
    if (m >= h || n >= w) continue;  // h even: row m + 1 is inside with row m
    const long long off = (long long)m * ld + n;
    float2 xe = make_float2(0.f, 0.f), xo = xe;
    if (zout) {  // issued before the taps: the loads are in flight while they run
      xe = xold[b * bs + off];
      xo = xold[b * bs + off + ld];
    }
    float2 ve = make_float2(0.f, 0.f), vo = ve;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int ii = ip + 3 - t;
      const float2 a = ulo[ii][nn], c = uhi[ii][nn];
      ve.x = fmaf(k_lo(2 * t), a.x, fmaf(k_hi(2 * t), c.x, ve.x));
      ve.y = fmaf(k_lo(2 * t), a.y, fmaf(k_hi(2 * t), c.y, ve.y));
      vo.x = fmaf(k_lo(2 * t + 1), a.x, fmaf(k_hi(2 * t + 1), c.x, vo.x));
      vo.y = fmaf(k_lo(2 * t + 1), a.y, fmaf(k_hi(2 * t + 1), c.y, vo.y));
    }
    if (zout) {
      zout[b * bs + off] = make_float2(fmaf(beta, ve.x - xe.x, ve.x), fmaf(beta, ve.y - xe.y, ve.y));
      zout[b * bs + off + ld] = make_float2(fmaf(beta, vo.x - xo.x, vo.x), fmaf(beta, vo.y - xo.y, vo.y));
    }
    ob[off] = ve;
    ob[off + ld] = vo;
  }
}

}  // namespace

extern "C" {

int sr_wavelet_levels_max(void) { return 8; }

// One analysis level (2-D).  thresh: device per-slice thresholds or NULL; if
// NULL and hthresh >= 0 a host threshold is used; both absent -> no prox.
// l1part: NULL or (batch, nblocks) doubles of sum |c| over the final coefficients.
int sr_wavelet_ana2(const sr_c64* src, sr_c64* dst, int h, int w, int ld, long long bs,
                    int batch, const float* thresh, float hthresh, int last, double* l1part,
                    void* stream) {
  if (h < 2 || w < 2 || (h & 1) || (w & 1) || batch < 1) return SR_EINVAL;
  if ((const void*)src == (const void*)dst) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid(((w >> 1) + TJ - 1) / TJ, ((h >> 1) + TI - 1) / TI, batch);
  k_wav_ana2<<<grid, dim3(TJ, TI), 0, st>>>((const float2*)src, (float2*)dst, h, w, ld, bs,
                                             thresh, hthresh, last, l1part);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_wavelet_ana2_nblocks(int h, int w) {
  return (((w >> 1) + TJ - 1) / TJ) * (((h >> 1) + TI - 1) / TI);
}

int sr_wavelet_syn2(const sr_c64* coef, sr_c64* out, int h, int w, int ld, long long bs,
                    int batch, sr_c64* zout, const sr_c64* xold, float beta, void* stream) {
  if (h < 2 || w < 2 || (h & 1) || (w & 1) || batch < 1) return SR_EINVAL;
  if ((const void*)coef == (const void*)out) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((w + SN - 1) / SN, (h + SM - 1) / SM, batch);
  k_wav_syn2<<<grid, 256, 0, st>>>((const float2*)coef, (float2*)out, h, w, ld, bs,
                                   (float2*)zout, (const float2*)xold, beta);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// The whole 2-D prox of Regularizer.prox (solvers.py:71-81) in one call: `levels` analysis levels
// (v -> buf0/buf1 ping-pong, soft threshold on every detail band and on the last low-pass corner)
// and the synthesis back into out with the FISTA momentum epilogue zout = out + beta (out - xold)
// on level 0 -- the launches of WaveletEngine.prox issued from C (one host call per prox).
int sr_wavelet_prox2(const sr_c64* v, sr_c64* out, sr_c64* buf0, sr_c64* buf1, int ny, int nx, long long bs,
                     int batch, int levels, const float* thresh, float hthresh, sr_c64* zout, const sr_c64* xold,
                     float beta, void* stream) {
  if (levels < 1 || levels > 8 || !v || !out || !buf0 || !buf1) return SR_EINVAL;
  sr_c64* bufs[2] = {buf0, buf1};
  const sr_c64* src = v;
  for (int l = 0; l < levels; ++l) {
    const int rc = sr_wavelet_ana2(src, bufs[l % 2], ny >> l, nx >> l, nx, bs, batch, thresh, hthresh,
                                   l == levels - 1, nullptr, stream);
    if (rc) return rc;
    src = bufs[l % 2];
  }
  for (int l = levels - 1; l >= 0; --l) {
    sr_c64* dst = (l == 0) ? out : bufs[(l - 1) % 2];
    const int rc = (l == 0) ? sr_wavelet_syn2(bufs[0], dst, ny, nx, nx, bs, batch, zout, xold, beta, stream)
                            : sr_wavelet_syn2(bufs[l % 2], dst, ny >> l, nx >> l, nx, bs, batch, nullptr, nullptr,
                                              0.f, stream);
    if (rc) return rc;
  }
  return SR_OK;
}

}  // extern "C"
