// K7: solver vector kernels -- per-slice linear combinations and deterministic
// fixed-order reductions (no atomics, so results are bit-reproducible).
//
// Reference loops these serve:
//   fista            /root/reference/pkg/src/sketchrecon/solvers.py:290-297
//   _cg_loop         /root/reference/pkg/src/sketchrecon/solvers.py:206-229
//   max_eig_power    /root/reference/pkg/src/sketchrecon/linops.py:766-782
// All scalars stay on the device (per-slice arrays) so an inner loop never
// synchronises with the host.
#include "common.cuh"

namespace {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 64;  // partial sums per slice (fixed => deterministic)

enum { RED_NORM2 = 0, RED_DOT = 1, RED_ABS = 2, RED_DIFF2 = 3 };

// result[b] = (re, im) of the reduction of slice b.
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_partial(int mode, const float2* __restrict__ a, const float2* __restrict__ bv,
                 long long n, long long bstride, double2* __restrict__ partial) {
  const int b = blockIdx.y;
  const float2* ab = a + b * bstride;
  const float2* bb = bv ? bv + b * bstride : nullptr;
  // contiguous chunk per block
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk;
  const long long hi = min(n, lo + chunk);
  double sr = 0.0, si = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float2 x = ab[i];
    if (mode == RED_NORM2) {
      sr += (double)x.x * x.x + (double)x.y * x.y;
    } else if (mode == RED_DOT) {  // sum conj(a) * b
      const float2 y = bb[i];
      sr += (double)x.x * y.x + (double)x.y * y.y;
      si += (double)x.x * y.y - (double)x.y * y.x;
    } else if (mode == RED_ABS) {
      sr += sqrt((double)x.x * x.x + (double)x.y * x.y);
    } else {  // RED_DIFF2
      const float2 y = bb[i];
      const double dx = (double)x.x - y.x, dy = (double)x.y - y.y;
      sr += dx * dx + dy * dy;
    }
  }
  __shared__ double rr[RED_THREADS], ri[RED_THREADS];
  rr[threadIdx.x] = sr;
  ri[threadIdx.x] = si;
  __syncthreads();
  for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rr[threadIdx.x] += rr[threadIdx.x + s];
      ri[threadIdx.x] += ri[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(long long)b * gridDim.x + blockIdx.x] = make_double2(rr[0], ri[0]);
}

__global__ void k_reduce_final(const double2* __restrict__ partial, int nparts, int batch,
                               double2* __restrict__ result) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double sr = 0.0, si = 0.0;
  for (int k = 0; k < nparts; ++k) {
    sr += partial[(long long)b * nparts + k].x;
    si += partial[(long long)b * nparts + k].y;
  }
  result[b] = make_double2(sr, si);
}

// out = c.x * X + c.y * Y + c.z * Z  (per-slice real coefficients; Y/Z nullable)
__global__ void k_lincomb(float2* __restrict__ out, const float2* __restrict__ X,
                          const float2* __restrict__ Y, const float2* __restrict__ Z,
                          const float4* __restrict__ coef, float4 hcoef, long long n,
                          long long bstride) {
  const int b = blockIdx.y;
  const float4 c = coef ? coef[b] : hcoef;
  const long long o = b * bstride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float2 x = X[o + i];
    float2 v = make_float2(c.x * x.x, c.x * x.y);
    if (Y) { const float2 y = Y[o + i]; v.x = fmaf(c.y, y.x, v.x); v.y = fmaf(c.y, y.y, v.y); }
    if (Z) { const float2 z = Z[o + i]; v.x = fmaf(c.z, z.x, v.x); v.y = fmaf(c.z, z.y, v.y); }
    out[o + i] = v;
  }
}

// Scalar bookkeeping kernels (one thread per slice) -------------------------
enum {
  SC_POWER = 0,     // in0 = (|w|^2, .), in1 = <v, w>: lam = Re in1; coef = (1/|w|, 0, 0); flag |w| == 0
  SC_CG_ALPHA = 1,  // in0 = rs (re), in1 = <p, Mp>: alpha = rs / denom; coefX = (1, alpha, 0), coefR = (1, -alpha, 0)
  SC_CG_BETA = 2,   // in0 = rs_new, state.rs_old: beta = rs_new / rs_old; coef = (1, beta, 0)
};

__global__ void k_scalar(int op, const double2* __restrict__ in0, const double2* __restrict__ in1,
                         double* __restrict__ state, float4* __restrict__ coefA,
                         float4* __restrict__ coefB, int* __restrict__ flags, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  if (op == SC_POWER) {
    const double nw = sqrt(in0[b].x);
    if (nw == 0.0) {
      flags[b] = 1;
      state[b] = 0.0;
      coefA[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (!flags[b]) {
      state[b] = in1[b].x;  // lam = Re <v, w>
      coefA[b] = make_float4((float)(1.0 / nw), 0.f, 0.f, 0.f);
    } else {
      coefA[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (op == SC_CG_ALPHA) {
    // state layout per slice: [rs, active]
    const double rs = state[2 * b];
    const double denom = in1[b].x;
    const bool active = state[2 * b + 1] != 0.0 && denom > 0.0;
    if (!active) state[2 * b + 1] = 0.0;
    const double alpha = active ? rs / denom : 0.0;
    coefA[b] = make_float4(1.f, (float)alpha, 0.f, 0.f);
    coefB[b] = make_float4(1.f, (float)(-alpha), 0.f, 0.f);
  } else if (op == SC_CG_BETA) {
    const double rs_new = in0[b].x;
    const double rs = state[2 * b];
    const bool active = state[2 * b + 1] != 0.0;
    const double beta = (active && rs != 0.0) ? rs_new / rs : 0.0;
    if (active) state[2 * b] = rs_new;
    // p = r + beta p (inactive slices keep p: coef (0, 1))
    coefA[b] = active ? make_float4(1.f, (float)beta, 0.f, 0.f) : make_float4(0.f, 1.f, 0.f, 0.f);
  }
}

}  // namespace

extern "C" {

int sr_reduce_nparts(void) { return RED_BLOCKS; }

// partial: (batch, RED_BLOCKS) double2 workspace; result: (batch,) double2
int sr_reduce(int mode, const sr_c64* a, const sr_c64* b, long long n, long long bstride,
              int batch, double* partial, double* result, void* stream) {
  if (n < 0 || batch < 1 || mode < 0 || mode > 3) return SR_EINVAL;
  if ((mode == RED_DOT || mode == RED_DIFF2) && b == nullptr) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid(RED_BLOCKS, batch);
  k_reduce_partial<<<grid, RED_THREADS, 0, st>>>(mode, (const float2*)a, (const float2*)b, n,
                                                 bstride, (double2*)partial);
  SR_CHECK_LAUNCH();
  k_reduce_final<<<(batch + 127) / 128, 128, 0, st>>>((const double2*)partial, RED_BLOCKS, batch,
                                                      (double2*)result);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

// coef: device (batch, 4) floats or NULL -> host coefficients (cx, cy, cz) for every slice
int sr_lincomb(sr_c64* out, const sr_c64* X, const sr_c64* Y, const sr_c64* Z,
               const float* coef, float cx, float cy, float cz, long long n,
               long long bstride, int batch, void* stream) {
  if (n < 0 || batch < 1) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  dim3 grid((unsigned)blocks, batch);
  k_lincomb<<<grid, 256, 0, st>>>((float2*)out, (const float2*)X, (const float2*)Y,
                                  (const float2*)Z, (const float4*)coef,
                                  make_float4(cx, cy, cz, 0.f), n, bstride);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

int sr_scalar_op(int op, const double* in0, const double* in1, double* state, float* coefA,
                 float* coefB, int* flags, int batch, void* stream) {
  if (batch < 1 || op < 0 || op > 2) return SR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  k_scalar<<<(batch + 127) / 128, 128, 0, st>>>(op, (const double2*)in0, (const double2*)in1,
                                                state, (float4*)coefA, (float4*)coefB, flags,
                                                batch);
  SR_CHECK_LAUNCH();
  return SR_OK;
}

}  // extern "C"
