// Batched tall-skinny Householder QR, R factor only (complex128), for the PCA coil compression
// of many slices (config 2: 256 blocks of 5119 x 32).
//
// Reference: coil_compress_svd (forward_model.py:245-272) takes U of np.linalg.svd(Y); for a wide
// C x N matrix LAPACK (zgesdd) first reduces Y by an LQ factorisation, so svd(Y).U equals the
// U of svd(L) with L = R^H from the Householder QR of Y^H (parallel_recon.slice_compression).
// This kernel computes that R with LAPACK's zgeqr2 / zlarfg conventions (real beta =
// -sign(Re alpha) * ||(alpha, x)||, tau = ((beta - Re alpha) / beta, -Im alpha / beta),
// v = x / (alpha - beta), H^H = I - conj(tau) v v^H applied to the trailing columns), one CTA per
// block: per column a norm reduction, then the trailing columns' v^H A products (register
// partials + warp shuffles + a small shared-memory tree) and the rank-1 update, which also
// accumulates the next column's squared norm.  Replaces a loop of cuSOLVER geqrf calls
// (105 ms -> a few ms at config 2).
#include "common.cuh"

namespace {

constexpr int TS_THREADS = 256;
constexpr int TS_MAXC = 32;

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconjmul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// block-wide sum of nv <= TS_MAXC complex values per thread (red: [NW][TS_MAXC] double2); the
// loops are fully unrolled so the per-thread values stay in registers
template <int NW>
__device__ __forceinline__ void block_sum(const double2 (&v)[TS_MAXC], int nv, double2* red, double2* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < TS_MAXC; ++j) {
    if (j < nv) {
      double2 s = v[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) red[warp * TS_MAXC + j] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      s.x += red[w * TS_MAXC + threadIdx.x].x;
      s.y += red[w * TS_MAXC + threadIdx.x].y;
    }
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(TS_THREADS)
k_tsqr_r(double2* __restrict__ A, long long N, int C, long long a_bstride, double2* __restrict__ R) {
  constexpr int NW = TS_THREADS / 32;
  __shared__ double2 red[NW * TS_MAXC];
  __shared__ double2 wsum[TS_MAXC];
  __shared__ double2 s_par[3];  // (scale = 1/(alpha - beta), conj(tau), beta)
  __shared__ double s_nrm;
  double2* a = A + blockIdx.x * a_bstride;
  double2* r = R + (long long)blockIdx.x * C * C;
  const int tid = threadIdx.x;
  for (int e = tid; e < C * C; e += TS_THREADS) r[e] = make_double2(0.0, 0.0);
  // ||A[1:, 0]||^2 for the first reflector
  double part = 0.0;
  for (long long i = 1 + tid; i < N; i += TS_THREADS) {
    const double2 v = a[i * C];
    part += v.x * v.x + v.y * v.y;
  }
  double2 tmp[TS_MAXC];
  for (int k = 0; k < C; ++k) {
    // column k's squared norm below the diagonal -> reflector (zlarfg)
    tmp[0] = make_double2(part, 0.0);
    block_sum<NW>(tmp, 1, red, wsum);
    if (tid == 0) {
      const double xnorm = sqrt(wsum[0].x);
      const double2 alpha = a[(long long)k * C + k];
      if (xnorm == 0.0 && alpha.y == 0.0) {
        s_par[0] = make_double2(0.0, 0.0);
        s_par[1] = make_double2(0.0, 0.0);
        s_par[2] = alpha;
      } else {
        // dlapy3(alphr, alphi, xnorm)
        const double ax = fabs(alpha.x), ay = fabs(alpha.y), az = xnorm;
        const double wmax = fmax(fmax(ax, ay), az);
        const double nrm = wmax == 0.0 ? ax + ay + az
                                       : wmax * sqrt((ax / wmax) * (ax / wmax) + (ay / wmax) * (ay / wmax) +
                                                     (az / wmax) * (az / wmax));
        const double beta = signbit(alpha.x) ? nrm : -nrm;  // -SIGN(nrm, alphr), Fortran sign bit
        const double2 tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
        // zladiv(1, alpha - beta)
        const double2 den = make_double2(alpha.x - beta, alpha.y);
        const double dd = den.x * den.x + den.y * den.y;
        s_par[0] = make_double2(den.x / dd, -den.y / dd);
        s_par[1] = make_double2(tau.x, -tau.y);  // conj(tau)
        s_par[2] = make_double2(beta, 0.0);
      }
      s_nrm = 0.0;
    }
    __syncthreads();
    const double2 scale = s_par[0], ctau = s_par[1];
    const bool reflect = !(ctau.x == 0.0 && ctau.y == 0.0);
    // v = x * scale below the diagonal (v_k = 1), kept in column k
    if (reflect)
      for (long long i = k + 1 + tid; i < N; i += TS_THREADS) a[i * C + k] = zmul(a[i * C + k], scale);
    __syncthreads();
    const int nt = C - k - 1;  // trailing columns
    if (reflect && nt > 0) {
      // w_j = sum_i conj(v_i) A[i, j]
#pragma unroll
      for (int j = 0; j < TS_MAXC; ++j) tmp[j] = make_double2(0.0, 0.0);
      for (long long i = k + tid; i < N; i += TS_THREADS) {
        const double2 vi = (i == k) ? make_double2(1.0, 0.0) : a[i * C + k];
        const double2* row = a + i * C + k + 1;
#pragma unroll
        for (int j = 0; j < TS_MAXC; ++j) {
          if (j < nt) {
            const double2 p = zconjmul(vi, row[j]);
            tmp[j].x += p.x;
            tmp[j].y += p.y;
          }
        }
      }
      block_sum<NW>(tmp, nt, red, wsum);
      // A[i, j] -= conj(tau) v_i w_j; the next column's squared norm below the next diagonal
      part = 0.0;
      for (long long i = k + tid; i < N; i += TS_THREADS) {
        const double2 vi = (i == k) ? make_double2(1.0, 0.0) : a[i * C + k];
        const double2 cv = zmul(ctau, vi);
        double2* row = a + i * C + k + 1;
#pragma unroll 4
        for (int j = 0; j < nt; ++j) {
          const double2 p = zmul(cv, wsum[j]);
          double2 x = row[j];
          x.x -= p.x;
          x.y -= p.y;
          row[j] = x;
          if (j == 0 && i > k + 1) part += x.x * x.x + x.y * x.y;
        }
      }
    } else {
      part = 0.0;
      if (nt > 0)
        for (long long i = k + 2 + tid; i < N; i += TS_THREADS) {
          const double2 x = a[i * C + k + 1];
          part += x.x * x.x + x.y * x.y;
        }
    }
    __syncthreads();
    // row k of R: beta on the diagonal, the updated A[k, k+1:] to its right
    if (tid == 0) r[(long long)k * C + k] = s_par[2];
    for (int j = k + 1 + tid; j < C; j += TS_THREADS) r[(long long)k * C + j] = a[(long long)k * C + j];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ one block, many CTAs
// The same zgeqr2 / zlarfg sequence for a single tall block (the single-slice compression of
// coil_sketching_recon: config 0 is 16.4 K x 16, config 3 81.9 K x 16), spread over G CTAs that
// each own a contiguous row range of A (A stays L2-resident: 4-21 MB).  Per column: partial
// squared norms -> grid barrier -> every CTA sums the G partials in the same fixed order (so all
// agree bit for bit on beta / tau) -> v and partial v^H A products -> grid barrier -> fixed-order
// sums -> rank-1 update of the own rows.  Rows 0..C-1 lie in CTA 0, which writes R.  One CTA per
// block took 4.6 ms at config 0 (latency-bound); this runs in ~0.1 ms.
constexpr int TG_MAXCTA = 148;
__device__ double2 g_tg_part[2][TG_MAXCTA][TS_MAXC];
__device__ unsigned g_tg_bar[2];

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// sense-free grid barrier: arrivals counted monotonically, generation published by the last CTA
__device__ __forceinline__ void grid_barrier(unsigned G, unsigned& gen) {
  __syncthreads();
  ++gen;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&g_tg_bar[0], 1u) + 1u;
    if (arrived == G * gen) {
      __threadfence();
      atomicExch(&g_tg_bar[1], gen);
    } else {
      while (ld_acquire_u32(&g_tg_bar[1]) < gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(TS_THREADS)
k_tsqr_r_grid(double2* __restrict__ A, long long N, int C, double2* __restrict__ R) {
  constexpr int NW = TS_THREADS / 32;
  __shared__ double2 red[NW * TS_MAXC];
  __shared__ double2 wsum[TS_MAXC];
  __shared__ double s_x2;
  const unsigned G = gridDim.x;
  const int cta = blockIdx.x, tid = threadIdx.x;
  const long long per = (N + G - 1) / G;
  const long long i0 = (long long)cta * per, i1 = min(N, i0 + per);
  unsigned gen = 0;
  if (cta == 0)
    for (int e = tid; e < C * C; e += TS_THREADS) R[e] = make_double2(0.0, 0.0);
  double part = 0.0;
  for (long long i = max(i0, 1LL) + tid; i < i1; i += TS_THREADS) {
    const double2 v = A[i * C];
    part += v.x * v.x + v.y * v.y;
  }
  double2 tmp[TS_MAXC];
  for (int k = 0; k < C; ++k) {
    tmp[0] = make_double2(part, 0.0);
    block_sum<NW>(tmp, 1, red, wsum);
    if (tid == 0) g_tg_part[0][cta][0] = wsum[0];
    grid_barrier(G, gen);
    if (tid == 0) {
      double x2 = 0.0;
      for (unsigned c = 0; c < G; ++c) x2 += g_tg_part[0][c][0].x;
      s_x2 = x2;
    }
    __syncthreads();
    // zlarfg, identically in every CTA (alpha = A[k, k] written by CTA 0 before the barrier)
    const double xnorm = sqrt(s_x2);
    const double2 alpha = A[(long long)k * C + k];
    double2 scale, ctau, beta2;
    if (xnorm == 0.0 && alpha.y == 0.0) {
      scale = make_double2(0.0, 0.0);
      ctau = make_double2(0.0, 0.0);
      beta2 = alpha;
    } else {
      const double ax = fabs(alpha.x), ay = fabs(alpha.y), az = xnorm;
      const double wmax = fmax(fmax(ax, ay), az);
      const double nrm = wmax == 0.0 ? ax + ay + az
                                     : wmax * sqrt((ax / wmax) * (ax / wmax) + (ay / wmax) * (ay / wmax) +
                                                   (az / wmax) * (az / wmax));
      const double beta = signbit(alpha.x) ? nrm : -nrm;
      const double2 den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
      ctau = make_double2((beta - alpha.x) / beta, alpha.y / beta);  // conj(tau)
      beta2 = make_double2(beta, 0.0);
    }
    const bool reflect = !(ctau.x == 0.0 && ctau.y == 0.0);
    const int nt = C - k - 1;
    if (reflect)
      for (long long i = max(i0, (long long)k + 1) + tid; i < i1; i += TS_THREADS) A[i * C + k] = zmul(A[i * C + k], scale);
    __syncthreads();
    if (reflect && nt > 0) {
#pragma unroll
      for (int j = 0; j < TS_MAXC; ++j) tmp[j] = make_double2(0.0, 0.0);
      for (long long i = max(i0, (long long)k) + tid; i < i1; i += TS_THREADS) {
        const double2 vi = (i == k) ? make_double2(1.0, 0.0) : A[i * C + k];
        const double2* row = A + i * C + k + 1;
#pragma unroll
        for (int j = 0; j < TS_MAXC; ++j) {
          if (j < nt) {
            const double2 pz = zconjmul(vi, row[j]);
            tmp[j].x += pz.x;
            tmp[j].y += pz.y;
          }
        }
      }
      block_sum<NW>(tmp, nt, red, wsum);
      if (tid < nt) g_tg_part[1][cta][tid] = wsum[tid];
    }
    grid_barrier(G, gen);
    if (reflect && nt > 0) {
      if (tid < nt) {
        double2 w = make_double2(0.0, 0.0);
        for (unsigned c = 0; c < G; ++c) {
          w.x += g_tg_part[1][c][tid].x;
          w.y += g_tg_part[1][c][tid].y;
        }
        wsum[tid] = w;
      }
      __syncthreads();
      part = 0.0;
      for (long long i = max(i0, (long long)k) + tid; i < i1; i += TS_THREADS) {
        const double2 vi = (i == k) ? make_double2(1.0, 0.0) : A[i * C + k];
        const double2 cv = zmul(ctau, vi);
        double2* row = A + i * C + k + 1;
#pragma unroll 4
        for (int j = 0; j < nt; ++j) {
          const double2 pz = zmul(cv, wsum[j]);
          double2 x = row[j];
          x.x -= pz.x;
          x.y -= pz.y;
          row[j] = x;
          if (j == 0 && i > k + 1) part += x.x * x.x + x.y * x.y;
        }
      }
    } else {
      part = 0.0;
      if (nt > 0)
        for (long long i = max(i0, (long long)k + 2) + tid; i < i1; i += TS_THREADS) {
          const double2 x = A[i * C + k + 1];
          part += x.x * x.x + x.y * x.y;
        }
    }
    __syncthreads();
    if (cta == 0) {
      if (tid == 0) R[(long long)k * C + k] = beta2;
      for (int j = k + 1 + tid; j < C; j += TS_THREADS) R[(long long)k * C + j] = A[(long long)k * C + j];
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

// A: (batch, N, C) complex128 row-major (Y^H of each block), overwritten (Householder vectors);
// R: (batch, C, C) complex128 upper triangular, LAPACK zgeqrf conventions.  C <= 32.
// A single large block runs on many CTAs with grid barriers (k_tsqr_r_grid; not re-entrant across
// concurrent streams: it uses one static barrier), batches on one CTA per block.
int sr_tsqr_r(void* A, long long N, int C, long long a_bstride, int batch, void* R, void* stream) {
  if (!A || !R || batch < 1 || C < 1 || C > TS_MAXC || N < C || a_bstride < N * C) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (batch == 1 && N >= 64LL * TS_MAXC) {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return SR_ECUDA;
    // every CTA co-resident (one per SM at most), each owning >= 64 rows (so rows 0..C-1 sit in CTA 0)
    long long G = N / 64;
    if (G > nsm) G = nsm;
    if (G > TG_MAXCTA) G = TG_MAXCTA;
    void* bar = nullptr;
    if (cudaGetSymbolAddress(&bar, g_tg_bar) != cudaSuccess) return SR_ECUDA;
    if (cudaMemsetAsync(bar, 0, sizeof(unsigned) * 2, st) != cudaSuccess) return SR_ECUDA;
    k_tsqr_r_grid<<<(unsigned)G, TS_THREADS, 0, st>>>((double2*)A, N, C, (double2*)R);
    SR_CHECK_LAUNCH();
    return SR_OK;
  }
  k_tsqr_r<<<batch, TS_THREADS, 0, st>>>((double2*)A, N, C, a_bstride, (double2*)R);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // extern "C"
