// In-register FFT building blocks shared by the line-pass kernels (fft.cu)
// and the cluster-fused 2-D transforms (fft2d.cu).
#pragma once

#include "tbt_internal.cuh"

namespace tbt {
namespace fftreg {

// cos(2*pi*t/16) for any integer t.
__host__ __device__ constexpr double cos16(int t) {
  t &= 15;
  if (t > 8) t = 16 - t;
  switch (t) {
    case 0: return 1.0;
    case 1: return 0.92387953251128675613;
    case 2: return 0.70710678118654752440;
    case 3: return 0.38268343236508977173;
    case 4: return 0.0;
    case 5: return -0.38268343236508977173;
    case 6: return -0.70710678118654752440;
    case 7: return -0.92387953251128675613;
    default: return -1.0;
  }
}

// b * exp(sign * 2*pi*i * t / 16), sign = +1 for the inverse.
template <bool INV>
__device__ __forceinline__ double2 twiddle16(double2 b, int t) {
  if (t == 0) return b;
  if (t == 4) return INV ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
  const double c = cos16(t);
  const double s = INV ? cos16(t + 12) : -cos16(t + 12);
  return make_double2(b.x * c - b.y * s, b.x * s + b.y * c);
}

template <int R>
__host__ __device__ constexpr int log2c() {
  return R <= 1 ? 0 : 1 + log2c<R / 2>();
}
__host__ __device__ constexpr int bitrev(int v, int bits) {
  int r = 0;
  for (int k = 0; k < bits; ++k) r |= ((v >> k) & 1) << (bits - 1 - k);
  return r;
}

// In-register radix-2 DIT transform of R <= 16 points. Stages and the
// bit-reversal are expanded by template recursion so every array index is
// a compile-time constant (the array stays in registers).
template <int R, int K>
__device__ __forceinline__ void bitrevPermute(double2 (&u)[R]) {
  if constexpr (K < R) {
    constexpr int J = bitrev(K, log2c<R>());
    if constexpr (K < J) {
      const double2 t = u[K];
      u[K] = u[J];
      u[J] = t;
    }
    bitrevPermute<R, K + 1>(u);
  }
}

template <int R, bool INV, int LEN, int IDX>
__device__ __forceinline__ void butterflies(double2 (&u)[R]) {
  // IDX enumerates (base, k) pairs of this stage: base = (IDX / HALF) * LEN.
  constexpr int HALF = LEN / 2;
  if constexpr (IDX < R / 2) {
    constexpr int BASE = (IDX / HALF) * LEN, K = IDX % HALF;
    const double2 b = twiddle16<INV>(u[BASE + K + HALF], K * (16 / LEN));
    const double2 a = u[BASE + K];
    u[BASE + K] = cadd(a, b);
    u[BASE + K + HALF] = csub(a, b);
    butterflies<R, INV, LEN, IDX + 1>(u);
  }
}

template <int R, bool INV, int LEN>
__device__ __forceinline__ void stages(double2 (&u)[R]) {
  if constexpr (LEN <= R) {
    butterflies<R, INV, LEN, 0>(u);
    stages<R, INV, LEN * 2>(u);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void fftReg(double2 (&u)[R]) {
  static_assert(R >= 1 && R <= 16 && (R & (R - 1)) == 0, "radix");
  bitrevPermute<R, 0>(u);
  stages<R, INV, 2>(u);
}


// Radix split of a transform length: N = R1 * R2 with R1, R2 <= 16.
template <int N>
struct Split {
  static constexpr int R1 = N <= 16 ? N : (N == 32 ? 4 : (N == 64 ? 8 : (N == 128 ? 8 : 16)));
  static constexpr int R2 = N / R1;
  static constexpr int LANES = R1 > R2 ? R1 : R2;  // butterfly lanes per batch entry
  static_assert(R1 * R2 == N && R2 <= 16, "unsupported FFT length");
};

}  // namespace fftreg
}  // namespace tbt
