// Batched shared-memory FFT line passes (kernels K2 / K4 and the K1
// precompute transform).
//
// Replaces the reference's fftInPlace (proj/src/fft.cpp:28-53) as used by
// fft2 (proj/src/linsolve.cpp:229-237). Same transform (forward sign -1,
// unscaled inverse, fft.hpp:27-28), different algorithm: a Stockham
// autosort over N = R1*R2 with each radix-R step done in registers with
// exact constant twiddles and the inter-step twiddles from an exact table,
// batched over the basis index (contiguous in memory, so every load and
// store is coalesced) instead of one scalar line at a time.
#include <algorithm>
#include <cstdio>

#include "tbt_internal.cuh"

namespace tbt {
namespace {

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

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

template <int R1, int R2, int BC, bool INV>
__global__ void __launch_bounds__(BC*(R1 > R2 ? R1 : R2))
fftPassKernel(FftPass p) {
  constexpr int N = R1 * R2;
  extern __shared__ double2 sbuf[];
  const int line = blockIdx.x;
  const int b = threadIdx.x % BC;
  const int i = threadIdx.x / BC;
  const int bg = blockIdx.y * BC + b;
  const bool bok = bg < p.batch;
  const double2* in = p.in + line * p.in_line_stride + bg;
  double2* out = p.out + line * p.out_line_stride + bg;
  const double2 zero = make_double2(0.0, 0.0);

  if constexpr (R2 == 1) {
    if (i != 0) return;
    double2 u[R1];
#pragma unroll
    for (int r = 0; r < R1; ++r) u[r] = (bok && r < p.n_in) ? ldg2(in + r * p.in_point_stride) : zero;
    fftReg<R1, INV>(u);
#pragma unroll
    for (int r = 0; r < R1; ++r)
      if (bok && r < p.n_out) out[r * p.out_point_stride] = cscale(u[r], p.scale);
    return;
  } else {
    // Step 1 (span 1): radix-R1 butterflies over points i + r*R2.
    if (i < R2) {
      double2 u[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        const int pt = i + r * R2;
        u[r] = (bok && pt < p.n_in) ? ldg2(in + (long long)pt * p.in_point_stride) : zero;
      }
      fftReg<R1, INV>(u);
#pragma unroll
      for (int r = 0; r < R1; ++r) sbuf[(i * R1 + r) * BC + b] = u[r];
    }
    __syncthreads();
    // Step 2 (span R1): twiddle w_N^{r*i}, radix-R2 butterflies, natural order out.
    if (i < R1) {
      double2 u[R2];
#pragma unroll
      for (int r = 0; r < R2; ++r) u[r] = sbuf[(i + r * R1) * BC + b];
#pragma unroll
      for (int r = 1; r < R2; ++r) {
        double2 w = __ldg(p.tw + r * i);  // r*i < N
        if (INV) w.y = -w.y;
        u[r] = cmul(u[r], w);
      }
      fftReg<R2, INV>(u);
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        const int pt = i + r * R1;
        if (bok && pt < p.n_out) out[(long long)pt * p.out_point_stride] = cscale(u[r], p.scale);
      }
    }
  }
  (void)N;
}

template <int R1, int R2, int BC>
void launchT(const FftPass& p, cudaStream_t s) {
  constexpr int NT = BC * (R1 > R2 ? R1 : R2);
  const size_t sm = (R2 > 1) ? sizeof(double2) * R1 * R2 * BC : 0;
  dim3 grid(p.lines, (p.batch + BC - 1) / BC);
  if (p.inverse)
    fftPassKernel<R1, R2, BC, true><<<grid, NT, sm, s>>>(p);
  else
    fftPassKernel<R1, R2, BC, false><<<grid, NT, sm, s>>>(p);
}

template <int BC>
void launchN(const FftPass& p, cudaStream_t s) {
  switch (p.n) {
    case 1: launchT<1, 1, BC>(p, s); break;
    case 2: launchT<2, 1, BC>(p, s); break;
    case 4: launchT<4, 1, BC>(p, s); break;
    case 8: launchT<8, 1, BC>(p, s); break;
    case 16: launchT<16, 1, BC>(p, s); break;
    case 32: launchT<4, 8, BC>(p, s); break;
    case 64: launchT<8, 8, BC>(p, s); break;
    case 128: launchT<8, 16, BC>(p, s); break;
    case 256: launchT<16, 16, BC>(p, s); break;
    default:
      throw Error{TBT_USER_ERROR, "FFT length " + std::to_string(p.n) +
                                      " not supported (powers of two up to 256)"};
  }
}

}  // namespace

void launchFftPass(const FftPass& p, cudaStream_t s) {
  if (p.lines == 0 || p.batch == 0) return;
  if (p.batch % 16 == 0 || p.batch >= 64)
    launchN<16>(p, s);
  else
    launchN<8>(p, s);
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
