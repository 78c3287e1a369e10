// Size bucket SR_BUCKET_ID of the per-axis NUFFT FFT kernels (see fft_axis.cuh); the
// generated wrappers fft_axis_inst_<k>.cu define SR_BUCKET_ID / SR_BUCKET_SIZES.
#include "fft_axis.cuh"

#define SR_CAT2(a, b) a##b
#define SR_CAT(a, b) SR_CAT2(a, b)

int SR_CAT(sr_fft_axis_b, SR_BUCKET_ID)(float2* data, long long outer, int n, long long inner, int inv,
                                       cudaStream_t st) {
  if (inner == 1) {
    switch (n) {
#define X(N_, P_, Q_) case N_: return launch_rows<P_, Q_>(data, outer, inv, st);
      SR_BUCKET_SIZES(X)
#undef X
      default: return SR_EUNSUPPORTED;
    }
  }
  switch (n) {
#define X(N_, P_, Q_) case N_: return launch_strided<P_, Q_>(data, outer, inner, inv, st);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

// contiguous rows whose frequency side is in natural order (grid rows of the NUFFT pipeline)
int SR_CAT(sr_fft_rows_nat_b, SR_BUCKET_ID)(float2* data, long long nrows, int n, int inv, cudaStream_t st) {
  switch (n) {
#define X(N_, P_, Q_) case N_: return launch_rows<P_, Q_>(data, nrows, inv, st, 1);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

int SR_CAT(sr_fft_axis_pruned_b, SR_BUCKET_ID)(float2* data, long long outer, int n, long long inner, int inv,
                                              AxPrune pr, cudaStream_t st) {
  switch (n) {
#define X(N_, P_, Q_) case N_: return launch_strided<P_, Q_>(data, outer, inner, inv, st, pr);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}

int SR_CAT(sr_nufft_row_fused_b, SR_BUCKET_ID)(const RowGeom& rg, int inv, cudaStream_t st) {
  switch (rg.g2) {
#define X(N_, P_, Q_) \
  case N_: return inv ? launch_row_fused<P_, Q_, true>(rg, st) : launch_row_fused<P_, Q_, false>(rg, st);
    SR_BUCKET_SIZES(X)
#undef X
    default: return SR_EUNSUPPORTED;
  }
}
