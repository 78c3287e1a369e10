// Two-level (four-step) in-CTA FFT building blocks.
//
// A length N = P*Q transform is split as natural index m = p + P*q
// (p < P, q < Q).  Frequencies k = k2 + Q*k1 (k2 < Q, k1 < P).
//
//   forward step 1 (per p, in registers):  Y[p][k2] = DFT_Q over q of x[p + P q],
//                                           then *= W_N^{p k2}; stored at pos P*k2 + p
//   forward step 2 (per k2, in registers): X[k2 + Q k1] = DFT_P over p of Y[p][k2];
//                                           stored at pos P*k2 + k1      ("perm order")
//   inverse step 2' (per k2): DFT^-1_P over k1 of the perm-order group, *= conj W_N^{m1 k2}
//   inverse step 1' (per m1): DFT^-1_Q over k2 -> x[m1 + P m2] in natural order.
//
// The forward output is left in perm order and the inverse consumes perm
// order, so forward -> (pointwise op) -> inverse never reorders data; the
// pointwise op (the undersampling mask) is stored in perm order by the host.
//
// Shared-memory layout: one vector of N float2 occupies Q groups of P
// elements, each group padded by one element (stride P+1) so that both the
// strided step-1 access and the contiguous step-2 access are bank-conflict
// free for P in {8, 16, 32}.
#pragma once
#include "common.cuh"
#include "dft_gen.cuh"
#include "tw_gen.cuh"

template <int P_, int Q_>
struct FftShape {
  static constexpr int P = P_;
  static constexpr int Q = Q_;
  static constexpr int N = P_ * Q_;
  static constexpr int GS = (P_ == 1) ? 1 : P_ + 1;  // padded group stride
  // padded vector stride, VS = P (mod 16): rows of a CTA then interleave in the
  // 32 banks exactly like contiguous data (conflict-free step-1 stores)
  static constexpr int VS0 = Q_ * GS;
  static constexpr int VS = VS0 + ((((P_ % 16) - (VS0 % 16)) % 16 + 16) % 16);
  __device__ __forceinline__ static int pad(int pos) { return (P_ == 1) ? pos : pos + pos / P_; }
  // perm position of frequency k (forward output layout)
  __host__ __device__ __forceinline__ static int perm_pos(int k) { return P_ * (k % Q_) + k / Q_; }
};

// Twiddle tables, copied into shared memory from the generated constants of
// tw_gen.cuh (float64 -> float32, correctly rounded):
//   t1[k2*P + p] = W_N^{p k2}   (forward step 1; lanes vary p  -> conflict-free)
//   t2[m1*Q + k2] = W_N^{m1 k2} (inverse step 2'; lanes vary k2 -> conflict-free)
template <int P, int Q>
__device__ __forceinline__ void init_tw_s1(float2* t1, int tid, int nthreads) {
  if constexpr (P > 1) {
    const float2* src = TwTab<P, Q>::t1();
    for (int e = tid; e < P * Q; e += nthreads) t1[e] = __ldg(src + e);
  }
}
template <int P, int Q>
__device__ __forceinline__ void init_tw_s2(float2* t2, int tid, int nthreads) {
  if constexpr (P > 1) {
    const float2* src = TwTab<P, Q>::t2();
    for (int e = tid; e < P * Q; e += nthreads) t2[e] = __ldg(src + e);
  }
}

// forward step 1: r[q] = x[p + P q]  ->  r[k2] = W_N^{p k2} * DFT_Q(r)[k2]
template <int P, int Q>
__device__ __forceinline__ void fft_s1_fwd(float2* r, int p, const float2* t1) {
  RegDFT<Q, false>::run(r);
  if (P > 1) {
#pragma unroll
    for (int k2 = 1; k2 < Q; ++k2) r[k2] = cmul(r[k2], t1[k2 * P + p]);
  }
}

// forward step 2: group of P values (index p) -> DFT_P (index k1)
template <int P>
__device__ __forceinline__ void fft_s2_fwd(float2* g) { RegDFT<P, false>::run(g); }

// inverse step 2': group (index k1) -> IDFT_P (index m1), then *= conj(W_N^{m1 k2})
template <int P, int Q>
__device__ __forceinline__ void fft_s2_inv(float2* g, int k2, const float2* t2) {
  RegDFT<P, true>::run(g);
  if (Q > 1) {
#pragma unroll
    for (int m1 = 1; m1 < P; ++m1) g[m1] = cmulc(t2[m1 * Q + k2], g[m1]);
  }
}

// inverse step 1': r[k2] -> IDFT_Q -> r[m2] = x[m1 + P m2]
template <int Q>
__device__ __forceinline__ void fft_s1_inv(float2* r) { RegDFT<Q, true>::run(r); }

// Row-tile layout of the row passes: groups of P padded by 2 (P even) so every
// group starts 16-byte aligned -> the step-2 group moves and the tile copies are
// 128-bit (LDS/STS/LDG/STG.128, cp.async 16 B).  Group stride GS/2 is odd in
// 16-byte units, so the 8-lane phases of the 128-bit step-2 accesses are
// conflict-free; VS = P (mod 16) keeps the 64-bit step-1 stores conflict-free.
template <int P_, int Q_>
struct RowShape {
  static constexpr int P = P_, Q = Q_, N = P_ * Q_;
  static constexpr bool VEC = (P_ % 2 == 0) && (P_ > 1);
  static constexpr int GS = VEC ? P_ + 2 : (P_ == 1 ? 1 : P_ + 1);
  static constexpr int VS0 = Q_ * GS;
  static constexpr int VS = VS0 + ((((P_ % 16) - (VS0 % 16)) % 16 + 16) % 16);
  __device__ __forceinline__ static int pad(int pos) { return (P_ == 1) ? pos : pos + (GS - P_) * (pos / P_); }
};

// Row tiles without group padding (groups of P back to back, rows padded to VS = P (mod 16)):
// a whole row is contiguous in shared memory, so one bulk-async copy moves it (k_rowinv).
// With P = 20 the 128-bit group loads see 2-way bank conflicts, which the DRAM-bound row IFFT
// pass absorbs.
template <int P_, int Q_>
struct RowShapeNP {
  static constexpr int P = P_, Q = Q_, N = P_ * Q_;
  static constexpr bool VEC = (P_ % 2 == 0) && (P_ > 1);
  static constexpr int GS = P_;
  static constexpr int VS0 = N;
  static constexpr int VS = VS0 + ((((P_ % 16) - (VS0 % 16)) % 16 + 16) % 16);
  __device__ __forceinline__ static int pad(int pos) { return pos; }
};

template <int P, bool VEC>
__device__ __forceinline__ void lds_group(float2* g, const float2* gp) {
  if constexpr (VEC) {
#pragma unroll
    for (int i = 0; i < P / 2; ++i) {
      const float4 v = reinterpret_cast<const float4*>(gp)[i];
      g[2 * i] = make_float2(v.x, v.y);
      g[2 * i + 1] = make_float2(v.z, v.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < P; ++i) g[i] = gp[i];
  }
}
template <int P, bool VEC>
__device__ __forceinline__ void sts_group(float2* gp, const float2* g) {
  if constexpr (VEC) {
#pragma unroll
    for (int i = 0; i < P / 2; ++i)
      reinterpret_cast<float4*>(gp)[i] = make_float4(g[2 * i].x, g[2 * i].y, g[2 * i + 1].x, g[2 * i + 1].y);
  } else {
#pragma unroll
    for (int i = 0; i < P; ++i) gp[i] = g[i];
  }
}

// ---------------------------------------------------------------------------
// Supported lengths and their (P, Q) split.  X(N, P, Q)
#define SR_FFT_SIZES(X)                                                          \
  X(1, 1, 1) X(2, 1, 2) X(3, 1, 3) X(4, 1, 4) X(5, 1, 5) X(6, 1, 6) X(8, 1, 8)             \
  X(9, 1, 9) X(10, 1, 10) X(12, 1, 12) X(15, 1, 15) X(16, 1, 16) X(18, 1, 18)   \
  X(20, 1, 20) X(24, 1, 24) X(25, 1, 25) X(30, 1, 30)                          \
  X(32, 16, 2) X(36, 12, 3) X(40, 8, 5) X(48, 16, 3) X(50, 10, 5) X(60, 12, 5)  \
  X(64, 16, 4) X(72, 12, 6) X(80, 16, 5) X(90, 10, 9) X(96, 16, 6)             \
  X(100, 10, 10) X(120, 12, 10) X(128, 16, 8) X(144, 12, 12) X(150, 25, 6)     \
  X(160, 16, 10) X(180, 20, 9) X(192, 16, 12) X(200, 20, 10) X(240, 20, 12)    \
  X(250, 25, 10) X(256, 16, 16) X(270, 30, 9) X(288, 24, 12) X(300, 20, 15)    \
  X(320, 20, 16) X(360, 24, 15) X(384, 24, 16) X(400, 20, 20) X(450, 30, 15)   \
  X(480, 24, 20) X(500, 25, 20) X(512, 32, 16) X(540, 30, 18) X(576, 24, 24)   \
  X(600, 24, 25) X(640, 32, 20) X(720, 30, 24) X(750, 30, 25) X(768, 32, 24)   \
  X(800, 32, 25) X(900, 30, 30) X(960, 32, 30) X(1024, 32, 32)
