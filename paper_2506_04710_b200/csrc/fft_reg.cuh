// In-register FFT building blocks shared by the line-pass kernels (fft.cu)
// and the cluster-fused 2-D transforms (fft2d.cu).
#pragma once

#include <type_traits>
#include <utility>

#include "tbt_internal.cuh"
#include "twiddle144.cuh"

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


// ---- mixed radix (2, 3 and their products up to 16) ---------------------

template <int... Is, class F>
__device__ __forceinline__ void staticForImpl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
// f(std::integral_constant<int, i>) for i = 0 .. N-1, fully expanded.
template <int N, class F>
__device__ __forceinline__ void staticFor(F&& f) {
  staticForImpl(std::make_integer_sequence<int, N>{}, f);
}

// b * exp(sign 2 pi i K / R) (sign = +1 for the inverse), R | 144.
template <bool INV, int K, int R>
__device__ __forceinline__ double2 twMul(double2 b) {
  constexpr int idx = (((K % R) + R) % R) * (144 / R);
  if constexpr (idx == 0) {
    return b;
  } else if constexpr (idx == 72) {
    return make_double2(-b.x, -b.y);
  } else if constexpr (idx == 36) {
    return INV ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
  } else if constexpr (idx == 108) {
    return INV ? make_double2(b.y, -b.x) : make_double2(-b.y, b.x);
  } else {
    constexpr double c = cos144(idx);
    constexpr double sn = cos144(idx - 36);  // sin(2 pi idx / 144)
    constexpr double sg = INV ? sn : -sn;
    return make_double2(b.x * c - b.y * sg, b.x * sg + b.y * c);
  }
}

// In-register DFT of R points, natural order in and out, for R in
// {1,2,3,4,6,8,9,12,16}: powers of two by fftReg, radix 3 explicitly, the
// rest by one decimation-in-time split R = P*Q (P = 3 or 2) with constant
// twiddles from the 144-entry table.
template <int R, bool INV>
__device__ __forceinline__ void dftReg(double2 (&u)[R]) {
  if constexpr (R == 1) {
  } else if constexpr ((R & (R - 1)) == 0) {
    fftReg<R, INV>(u);
  } else if constexpr (R == 3) {
    constexpr double h = 0.86602540378443864676;  // sqrt(3)/2
    const double2 t1 = cadd(u[1], u[2]);
    const double2 t2 = make_double2(u[0].x - 0.5 * t1.x, u[0].y - 0.5 * t1.y);
    const double2 d = csub(u[1], u[2]);
    const double2 t3 = INV ? make_double2(-d.y * h, d.x * h) : make_double2(d.y * h, -d.x * h);
    u[0] = cadd(u[0], t1);
    u[1] = cadd(t2, t3);
    u[2] = csub(t2, t3);
  } else {
    constexpr int P = (R % 3 == 0) ? 3 : 2;
    constexpr int Q = R / P;
    double2 a[P][Q];
    staticFor<P>([&](auto p) {
      constexpr int pp = decltype(p)::value;
      staticFor<Q>([&](auto q) { a[pp][decltype(q)::value] = u[decltype(q)::value * P + pp]; });
      dftReg<Q, INV>(a[pp]);
    });
    staticFor<Q>([&](auto k) {
      constexpr int kk = decltype(k)::value;
      double2 t[P];
      staticFor<P>([&](auto p) {
        constexpr int pp = decltype(p)::value;
        t[pp] = twMul<INV, pp * kk, R>(a[pp][kk]);
      });
      dftReg<P, INV>(t);
      staticFor<P>([&](auto s2) { u[kk + Q * decltype(s2)::value] = t[decltype(s2)::value]; });
    });
  }
}

// Radix split of a transform length: N = R1 * R2 with R1, R2 <= 16 from
// {1,2,3,4,6,8,9,12,16}; LANES = butterfly lanes per batch entry.
template <int N>
struct Split {
  static constexpr int R1 =
      (N <= 16 && N != 5 && N != 7 && N != 10 && N != 11 && N != 13 && N != 14 && N != 15) ? N
      : N == 18 ? 3 : N == 24 ? 4 : N == 32 ? 4 : N == 36 ? 6 : N == 48 ? 6 : N == 64 ? 8 : N == 72 ? 8
      : N == 96 ? 8 : N == 128 ? 8 : N == 144 ? 12 : N == 192 ? 12 : N == 256 ? 16 : 0;
  static constexpr int R2 = R1 ? N / R1 : 0;
  static constexpr int LANES = R1 > R2 ? R1 : R2;
  static_assert(R1 > 0 && R1 * R2 == N && R2 <= 16, "unsupported FFT length");
};

}  // namespace fftreg
}  // namespace tbt
