// Size bucket SR_BUCKET_ID of the Cartesian kernels: dispatchers for the sizes in
// SR_BUCKET_SIZES only (cart.cu chains the buckets).  Generated wrappers cart_inst_<k>.cu
// define both macros and include this file.
#include "cart_kernels.cuh"

#define SR_CAT2(a, b) a##b
#define SR_CAT(a, b) SR_CAT2(a, b)

int SR_CAT(sr_dispatch_rowfwd_b, SR_BUCKET_ID)(int nx, const float2* x, const float2* anchor, const float2* maps,
                                               float2* ws, int batch, int ncoils, int ny, long long xbs,
                                               long long mbs, cudaStream_t st) {
  switch (nx) {
#define X(N, P, Q) \
  case N: return launch_rowfwd<P, Q>(x, anchor, maps, ws, batch, ncoils, ny, xbs, mbs, st);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

int SR_CAT(sr_dispatch_rowinv_b, SR_BUCKET_ID)(int nx, const float2* ws, const float2* maps, float2* out,
                                               int batch, int ncoils, int ny, long long xbs, long long mbs,
                                               const float4* coef, const float2* u, const float2* d,
                                               float oscale, cudaStream_t st) {
  switch (nx) {
#define X(N, P, Q)                                                                      \
  case N:                                                                               \
    return launch_rowinv<P, Q>(ws, maps, out, batch, ncoils, ny, xbs, mbs, coef, u, d, \
                               oscale, st);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

int SR_CAT(sr_dispatch_colpass_b, SR_BUCKET_ID)(int ny, float2* ws, const uint8_t* maskT, long long mbs,
                                                float mscale, int mode, int batch, int ncoils, int nx,
                                                cudaStream_t st, const SampleIO* sio) {
  switch (ny) {
#define X(N, P, Q) \
  case N: return launch_colpass<P, Q>(ws, maskT, mbs, mscale, mode, batch, ncoils, nx, st, sio);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

int SR_CAT(sr_dispatch_colblock_b, SR_BUCKET_ID)(int ny) {
  switch (ny) {
#define X(N, P, Q) \
  case N: return ColCfg<P, Q>::CB;
    SR_BUCKET_SIZES(X)
#undef X
    default: return 0;
  }
}
