// Cluster-fused 2-D transforms (kernels K2 and K4).
//
// One thread-block cluster owns a chunk of BC batch entries (basis index x
// right-hand side) of the whole L1 x L0 grid. The two 1-D passes of fft2
// (proj/src/linsolve.cpp:229-237) run in one kernel: the first pass writes
// its lines straight into the shared memory of the CTA that owns them for
// the second pass (distributed shared memory, cluster-wide barrier in
// between), so the intermediate never goes to global memory and the
// transform costs one launch instead of two.
//
//   forward (K2): rows r < ny of x (only nx non-zero points each) along
//                 level 0  ->  DSMEM transpose  ->  columns along level 1
//                 (ny non-zero points)  ->  xhat[s1][s0][b]
//   inverse (K4): columns of yhat along level 1, keeping the ny element rows
//                 ->  DSMEM transpose  ->  rows along level 0, keeping nx
//                 points, times 1/L, plus the edge/corner correction
//                 (correction.cu) in the store epilogue  ->  y[e][b]
// Line ownership is cyclic: CTA k of the cluster owns rows r = k + CL*i and
// columns s0 = k + CL*j.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fft_reg.cuh"
#include "ptx.cuh"
#include "tbt_internal.cuh"

namespace cg = cooperative_groups;

namespace tbt {
namespace {

using fftreg::dftReg;
using fftreg::Split;

// One line of length N for one batch entry per thread (ii = butterfly
// lane). All threads of the line group call it: the group synchronises on
// its own named barrier (bar, nthr threads), so line groups of a CTA do not
// wait for each other; `act` masks the work of lanes without a line.
template <int N, int BC, bool INV, class Src, class Snk>
__device__ __forceinline__ void lineFft(double2* st, int ii, int b, bool act, const double2* tw, int bar, int nthr,
                                        Src src, Snk snk) {
  using S = Split<N>;
  if constexpr (S::R2 == 1) {
    if (act && ii == 0) {
      double2 u[S::R1];
#pragma unroll
      for (int r = 0; r < S::R1; ++r) u[r] = src(r);
      dftReg<S::R1, INV>(u);
#pragma unroll
      for (int r = 0; r < S::R1; ++r) snk(r, u[r]);
    }
  } else {
    if (act && ii < S::R2) {
      double2 u[S::R1];
#pragma unroll
      for (int r = 0; r < S::R1; ++r) u[r] = src(ii + r * S::R2);
      dftReg<S::R1, INV>(u);
#pragma unroll
      for (int r = 0; r < S::R1; ++r) st[(ii * S::R1 + r) * BC + b] = u[r];
    }
    if (nthr > 0)
      namedBarrier(bar, nthr);
    else
      __syncthreads();
    if (act && ii < S::R1) {
      double2 u[S::R2];
#pragma unroll
      for (int r = 0; r < S::R2; ++r) u[r] = st[(ii + r * S::R1) * BC + b];
#pragma unroll
      for (int r = 1; r < S::R2; ++r) {
        double2 w = __ldg(tw + r * ii);
        if (INV) w.y = -w.y;
        u[r] = cmul(u[r], w);
      }
      dftReg<S::R2, INV>(u);
#pragma unroll
      for (int r = 0; r < S::R2; ++r) snk(ii + r * S::R1, u[r]);
    }
    if (nthr > 0)
      namedBarrier(bar, nthr);
    else
      __syncthreads();
  }
}

template <int N0, int N1, int BC>
struct Fft2dCfg {
  static constexpr int NTL = Split<N0>::LANES > Split<N1>::LANES ? Split<N0>::LANES : Split<N1>::LANES;
  static constexpr int TPL = NTL * BC;  // threads per line group
  static constexpr int LPAR = (256 / TPL) < 1 ? 1 : ((256 / TPL) > 8 ? 8 : 256 / TPL);
  static constexpr int NT = LPAR * TPL;
  static constexpr int NMAX = N0 > N1 ? N0 : N1;
  static constexpr int STAGE = NMAX * BC;  // double2 per line group
};

template <int N0, int N1, int BC, bool INV>
__global__ void __launch_bounds__(Fft2dCfg<N0, N1, BC>::NT) fft2dKernel(Fft2dArgs a) {
  using C = Fft2dCfg<N0, N1, BC>;
  extern __shared__ __align__(16) double2 sm2[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = static_cast<int>(cl.num_blocks());
  const int k = static_cast<int>(cl.block_rank());
  const int g = threadIdx.x / C::TPL;
  const int rem = threadIdx.x % C::TPL;
  const int b = rem % BC, ii = rem / BC;
  const int bg = (blockIdx.x / CL) * BC + b;
  const bool bok = bg < a.B;
  double2* st = sm2 + g * C::STAGE;
  double2* xbuf = sm2 + C::LPAR * C::STAGE;
  const double2 zero = make_double2(0.0, 0.0);
  const long long B = a.B;
  const int rowsLocal = (a.ny + CL - 1) / CL;
  const int colsLocal = a.L0 / CL;

  if constexpr (!INV) {
    // Rows along level 0 -> column owners' buffers [j][r][b].
    for (int base = 0; base < rowsLocal; base += C::LPAR) {
      const int i = base + g, r = k + CL * i;
      const bool act = bok && i < rowsLocal && r < a.ny;
      lineFft<N0, BC, false>(
          st, ii, b, act, a.tw0, 1 + g, C::TPL % 32 == 0 ? C::TPL : 0,
          [&](int c) { return c < a.nx ? a.in[(static_cast<long long>(r) * a.nx + c) * B + bg] : zero; },
          [&](int s0, double2 v) {
            double2* dst = cl.map_shared_rank(xbuf, s0 % CL);
            dst[(static_cast<long long>(s0 / CL) * a.ny + r) * BC + b] = v;
          });
    }
    cl.sync();
    // Columns along level 1 -> xhat[s1][s0][b].
    for (int base = 0; base < colsLocal; base += C::LPAR) {
      const int j = base + g, s0 = k + CL * j;
      const bool act = bok && j < colsLocal;
      lineFft<N1, BC, false>(
          st, ii, b, act, a.tw1, 1 + g, C::TPL % 32 == 0 ? C::TPL : 0,
          [&](int r) { return r < a.ny ? xbuf[(static_cast<long long>(j) * a.ny + r) * BC + b] : zero; },
          [&](int s1, double2 v) { a.out[(static_cast<long long>(s1) * a.L0 + s0) * B + bg] = v; });
    }
  } else {
    // Columns along level 1 (inverse), keep the ny element rows -> row
    // owners' buffers [i][s0][b].
    for (int base = 0; base < colsLocal; base += C::LPAR) {
      const int j = base + g, s0 = k + CL * j;
      const bool act = bok && j < colsLocal;
      lineFft<N1, BC, true>(
          st, ii, b, act, a.tw1, 1 + g, C::TPL % 32 == 0 ? C::TPL : 0,
          [&](int s1) { return a.in[(static_cast<long long>(s1) * a.L0 + s0) * B + bg]; },
          [&](int r, double2 v) {
            if (r < a.ny) {
              double2* dst = cl.map_shared_rank(xbuf, r % CL);
              dst[(static_cast<long long>(r / CL) * a.L0 + s0) * BC + b] = v;
            }
          });
    }
    cl.sync();
    // Rows along level 0 (inverse), keep nx points, scale, correction.
    for (int base = 0; base < rowsLocal; base += C::LPAR) {
      const int i = base + g, r = k + CL * i;
      const bool act = bok && i < rowsLocal && r < a.ny;
      lineFft<N0, BC, true>(
          st, ii, b, act, a.tw0, 1 + g, C::TPL % 32 == 0 ? C::TPL : 0,
          [&](int s0) { return xbuf[(static_cast<long long>(i) * a.L0 + s0) * BC + b]; },
          [&](int c, double2 v) {
            if (c < a.nx) {
              const int e = r * a.nx + c;
              double2 out = cscale(v, a.scale);
              if (a.corr && a.tPtr[e] != a.tPtr[e + 1]) out = cadd(out, a.ycorr[static_cast<long long>(e) * B + bg]);
              a.out[static_cast<long long>(e) * B + bg] = out;
            }
          });
    }
  }
}

template <int N0, int N1, int BC>
bool launch2d(const Fft2dArgs& a, int CL, bool inverse, cudaStream_t s) {
  using C = Fft2dCfg<N0, N1, BC>;
  const int rowsLocal = (a.ny + CL - 1) / CL;
  const size_t xbuf = inverse ? static_cast<size_t>(rowsLocal) * a.L0 * BC
                              : static_cast<size_t>(a.L0 / CL) * a.ny * BC;
  const size_t smem = (static_cast<size_t>(C::LPAR) * C::STAGE + xbuf) * sizeof(double2);
  if (smem > 200 * 1024) return false;
  const void* fn = inverse ? reinterpret_cast<const void*>(fft2dKernel<N0, N1, BC, true>)
                           : reinterpret_cast<const void*>(fft2dKernel<N0, N1, BC, false>);
  TBT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg = {};
  const int chunks = (a.B + BC - 1) / BC;
  cfg.gridDim = dim3(CL * chunks);
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Fft2dArgs arg = a;
  if (inverse)
    TBT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft2dKernel<N0, N1, BC, true>, arg));
  else
    TBT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft2dKernel<N0, N1, BC, false>, arg));
  return true;
}

template <int N0, int N1>
bool launchBC(const Fft2dArgs& a, int CL, int BC, bool inverse, cudaStream_t s) {
  switch (BC) {
    case 16: return launch2d<N0, N1, 16>(a, CL, inverse, s);
    case 8: return launch2d<N0, N1, 8>(a, CL, inverse, s);
    case 4: return launch2d<N0, N1, 4>(a, CL, inverse, s);
    case 2: return launch2d<N0, N1, 2>(a, CL, inverse, s);
    default: return false;
  }
}

}  // namespace

bool fft2dSupported(int L0, int L1) {
  const int key = L0 * 1000 + L1;
  switch (key) {
    case 8008: case 16016: case 32032: case 64064: case 128128: case 256256: case 64032: case 16008:
    case 36018:
      return true;
    default:
      return false;
  }
}

// Cluster size and batch chunk: >= ~1 CTA per SM, transpose buffer within
// shared memory.
void fft2dPlan(int L0, int L1, int nx, int ny, int B, int sms, int* CL, int* BC) {
  (void)L1;
  (void)nx;
  int cl = 8;
  while (cl > 1 && (L0 % cl != 0 || cl > ny)) cl /= 2;  // columns split evenly, rows keep CTAs busy
  if (cl < 1) cl = 1;
  int bc = 16;
  auto xbufBytes = [&](int c) {
    const size_t rows = (ny + cl - 1) / cl;
    return std::max(static_cast<size_t>(L0 / cl) * ny, rows * L0) * c * 16;
  };
  while (bc > 2 && (static_cast<long long>(cl) * ((B + bc - 1) / bc) < sms || xbufBytes(bc) > 160 * 1024)) bc /= 2;
  *CL = cl;
  *BC = bc;
  // Tuning override "CL,BC" (CL must divide L0).
  if (const char* e = getenv("TBT_FFT2D")) {
    int c2 = 0, b2 = 0;
    if (sscanf(e, "%d,%d", &c2, &b2) == 2 && c2 >= 1 && c2 <= 8 && L0 % c2 == 0 && (b2 == 2 || b2 == 4 || b2 == 8 || b2 == 16)) {
      *CL = c2;
      *BC = b2;
    }
  }
}

bool launchFft2d(const Fft2dArgs& a, int CL, int BC, bool inverse, cudaStream_t s) {
  const int key = a.L0 * 1000 + a.L1;
  switch (key) {
    case 8008: return launchBC<8, 8>(a, CL, BC, inverse, s);
    case 16016: return launchBC<16, 16>(a, CL, BC, inverse, s);
    case 32032: return launchBC<32, 32>(a, CL, BC, inverse, s);
    case 64064: return launchBC<64, 64>(a, CL, BC, inverse, s);
    case 128128: return launchBC<128, 128>(a, CL, BC, inverse, s);
    case 256256: return launchBC<256, 256>(a, CL, BC, inverse, s);
    case 64032: return launchBC<64, 32>(a, CL, BC, inverse, s);
    case 16008: return launchBC<16, 8>(a, CL, BC, inverse, s);
    case 36018: return launchBC<36, 18>(a, CL, BC, inverse, s);
    default: return false;
  }
}

}  // namespace tbt
