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

#include "fft_reg.cuh"
#include "tbt_internal.cuh"

namespace tbt {
namespace {

using fftreg::dftReg;

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
    dftReg<R1, INV>(u);
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
      dftReg<R1, INV>(u);
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
      dftReg<R2, INV>(u);
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        const int pt = i + r * R1;
        if (bok && pt < p.n_out) out[(long long)pt * p.out_point_stride] = cscale(u[r], p.scale);
      }
    }
  }
  (void)N;
}

// One thread per (line, batch entry): consecutive threads take consecutive
// batch entries, so every point's load / store is one contiguous 16-byte-
// per-lane run (512 B per warp), and a thread keeps all n_in loads of its
// line in flight. The N = R1 * R2 transform runs in registers: R2 radix-R1
// DFTs over the decimated inputs, the twiddles w_N^(n2 k1) (table), then R1
// radix-R2 DFTs; natural order in and out. No shared memory, no barriers.
// CROP (inverse passes that keep n_out <= ceil(N/2) points, i.e. every
// embedding's crop): the unused outputs and their arithmetic drop out at
// compile time, and the registers they held carry the correction values.
template <int N, bool INV, bool CROP>
__global__ void __launch_bounds__(128, (N >= 48 ? 1 : N >= 24 ? 3 : 4)) regLineKernel(FftPass p) {
  using S = fftreg::Split<N>;
  constexpr int R1 = S::R1, R2 = S::R2;
  const int bg = blockIdx.x * blockDim.x + threadIdx.x;
  if (bg >= p.batch) return;
  const int line = blockIdx.y;
  const long long userBase = p.userM ? static_cast<long long>(bg / p.userM) * p.userN + bg % p.userM : 0;
  const double2* in = p.inUser ? p.in + userBase + static_cast<long long>(line) * p.userNx * p.userM
                               : p.in + line * p.in_line_stride + bg;
  const long long inStride = p.inUser ? p.userM : p.in_point_stride;
  double2 t[R2][R1];  // t[n2][n1] = x[R2 * n1 + n2]
#pragma unroll
  for (int n1 = 0; n1 < R1; ++n1)
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      const int pt = R2 * n1 + n2;
      t[n2][n1] = pt < p.n_in ? ldg2(in + static_cast<long long>(pt) * inStride) : make_double2(0.0, 0.0);
    }
  // Which output points carry correction terms (a mask for this line), read
  // while the line's own loads are in flight.
  unsigned long long targets = 0;
  if (p.ycorr)
    for (int pt = 0; pt < p.n_out && pt < 64; ++pt) {
      const int e = line * p.corrNx + pt;
      if (__ldg(p.tPtr + e) != __ldg(p.tPtr + e + 1)) targets |= 1ull << pt;
    }
#pragma unroll
  for (int n2 = 0; n2 < R2; ++n2) dftReg<R1, INV>(t[n2]);  // -> t[n2][k1]
#pragma unroll
  for (int n2 = 1; n2 < R2; ++n2)
#pragma unroll
    for (int k1 = 1; k1 < R1; ++k1) {
      double2 w = __ldg(p.tw + n2 * k1);  // n2 * k1 < N
      if (INV) w.y = -w.y;
      t[n2][k1] = cmul(t[n2][k1], w);
    }
  double2* out = p.outUser ? p.out + userBase + static_cast<long long>(line) * p.userNx * p.userM
                           : p.out + line * p.out_line_stride + bg;
  const long long outStride = p.outUser ? p.userM : p.out_point_stride;
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    double2 v[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) v[n2] = t[n2][k1];
    if constexpr (R2 > 1) dftReg<R2, INV>(v);
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) t[n2][k1] = v[n2];  // t[k2][k1] = X[k1 + R1 k2]
  }
  // ycorr is internal [e][B]: e * B + bg = line * out_line_stride + pt * out_point_stride + bg
  constexpr int NC = (N + 1) / 2;
  const double2* yc = p.ycorr ? p.ycorr + line * p.out_line_stride + bg : nullptr;  // read only where targets != 0
  if constexpr (CROP) {
    // Every correction load of the thread goes out before the first store
    // (read-only loads, so the stores do not order them; one at a time they
    // were 18 serial latencies per thread, half of the last pass's time in
    // ncu's stall samples).
    double2 cv[NC];
#pragma unroll
    for (int pt = 0; pt < NC; ++pt)
      cv[pt] = (targets >> pt) & 1ull ? ldg2(yc + static_cast<long long>(pt) * p.out_point_stride) : make_double2(0.0, 0.0);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2)
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const int pt = k1 + R1 * k2;
        if (pt < NC && pt < p.n_out) out[static_cast<long long>(pt) * outStride] = cadd(cscale(t[k2][k1], p.scale), cv[pt]);
      }
  } else {
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2)
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const int pt = k1 + R1 * k2;
        if (pt < p.n_out) {
          double2 o = cscale(t[k2][k1], p.scale);
          if ((targets >> pt) & 1ull) o = cadd(o, ldg2(yc + static_cast<long long>(pt) * p.out_point_stride));
          out[static_cast<long long>(pt) * outStride] = o;
        }
      }
  }
}

template <int N>
void launchReg(const FftPass& p, cudaStream_t s) {
  dim3 grid((p.batch + 127) / 128, p.lines);
  if (!p.inverse)
    regLineKernel<N, false, false><<<grid, 128, 0, s>>>(p);
  else if (p.n_out <= (N + 1) / 2)
    regLineKernel<N, true, true><<<grid, 128, 0, s>>>(p);
  else
    regLineKernel<N, true, false><<<grid, 128, 0, s>>>(p);
}

template <int R1, int R2, int BC>
void launchT(const FftPass& p, cudaStream_t s) {
  constexpr int NT = BC * (R1 > R2 ? R1 : R2);
  const size_t sm = (R2 > 1) ? sizeof(double2) * R1 * R2 * BC : 0;
  dim3 grid(p.lines, (p.batch + BC - 1) / BC);
  if (sm > 48 * 1024) {  // opt in above the default dynamic shared-memory limit
    static std::atomic<unsigned long long> done[2] = {{0}, {0}};
    oncePerDevice(done[p.inverse ? 1 : 0], [&] {
      const void* fn = p.inverse ? reinterpret_cast<const void*>(fftPassKernel<R1, R2, BC, true>)
                                 : reinterpret_cast<const void*>(fftPassKernel<R1, R2, BC, false>);
      TBT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    });
  }
  if (p.inverse)
    fftPassKernel<R1, R2, BC, true><<<grid, NT, sm, s>>>(p);
  else
    fftPassKernel<R1, R2, BC, false><<<grid, NT, sm, s>>>(p);
}

template <int BC>
void launchN(const FftPass& p, cudaStream_t s) {
  switch (p.n) {
#define TBT_CASE(N) \
  case N: launchT<fftreg::Split<N>::R1, fftreg::Split<N>::R2, BC>(p, s); break;
    TBT_CASE(1) TBT_CASE(2) TBT_CASE(3) TBT_CASE(4) TBT_CASE(6) TBT_CASE(8) TBT_CASE(9) TBT_CASE(12)
    TBT_CASE(16) TBT_CASE(18) TBT_CASE(24) TBT_CASE(32) TBT_CASE(36) TBT_CASE(48) TBT_CASE(64) TBT_CASE(72)
    TBT_CASE(96) TBT_CASE(128) TBT_CASE(144) TBT_CASE(192) TBT_CASE(256)
#undef TBT_CASE
    default:
      throw Error{TBT_USER_ERROR, "FFT length " + std::to_string(p.n) + " not supported"};
  }
}

}  // namespace

bool launchFftPassReg(const FftPass& p, cudaStream_t s) {
  if (p.lines == 0 || p.batch == 0) return true;
  if (p.batch < 512 || p.lines > 65535) return false;
  switch (p.n) {
    case 8: launchReg<8>(p, s); break;
    case 9: launchReg<9>(p, s); break;
    case 12: launchReg<12>(p, s); break;
    case 16: launchReg<16>(p, s); break;
    case 18: launchReg<18>(p, s); break;
    case 24: launchReg<24>(p, s); break;
    case 32: launchReg<32>(p, s); break;
    case 36: launchReg<36>(p, s); break;
    case 48: launchReg<48>(p, s); break;
    case 64: launchReg<64>(p, s); break;
    default: return false;
  }
  TBT_CUDA_CHECK(cudaGetLastError());
  return true;
}

void launchFftPass(const FftPass& p, cudaStream_t s) {
  if (p.lines == 0 || p.batch == 0) return;
  if (p.batch % 16 == 0 || p.batch >= 64)
    launchN<16>(p, s);
  else
    launchN<8>(p, s);
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
