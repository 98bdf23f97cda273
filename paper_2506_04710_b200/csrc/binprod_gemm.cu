// K3 for many right-hand sides (C3: 162 port excitations): the bin-pair
// product becomes two complex GEMMs per stored block,
//     Yhat_f = Ahat X_f,      Yhat_g = Ahat^T X_g      (X: m x nrhs),
// computed on the FP64 tensor path (mma.sync.m8n8k4.f64, "DMMA": on B200 it
// runs at the FP64 peak with one instruction per 256 FMAs). A complex
// 8x8x4 block is THREE real DMMAs (3M / Gauss): S1 += Ar Br, S2 += Ai Bi,
// S3 += (Ar + Ai)(Br + Bi); Re = S1 - S2, Im = S3 - S1 - S2 at the end. The
// kernel is DMMA-bound, so this removes a quarter of its work; the extra
// rounding is a few ulps of |A||X| (the matvec parity bound is 1e-11).
// TBT_GEMM=4m selects the 4M form (Re += Ar Br + (-Ai) Bi, Im += Ar Bi +
// Ai Br: four DMMAs, two accumulator sets) for comparison.
// The reference re-streams every block once per column
// (linsolve.cpp:276-282, 572).
//
// Two CTA shapes. binprodGemm (m = 64, and m = 128 under TBT_GEMM=wide|4m):
// all M rows x NTILE right-hand sides of one (pair, transpose) item; 8 warps,
// warp w owns rows [w*M/8, (w+1)*M/8). K advances in chunks of 32 through a
// cp.async double buffer: the A chunk (M x 32 for A, or the 32 contiguous
// rows of A for A^T) and the X chunk (32 x NTILE). binprodGemm2 (the m = 128
// default, below): 64-row tiles on 4-warp CTAs, two per SM.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tbt_internal.cuh"

namespace tbt {
namespace {

constexpr int NT = 256;
constexpr int KC = 32;     // K chunk
constexpr int NTILE = 56;  // right-hand sides per CTA tile (7 n-blocks of 8)
constexpr int NB = NTILE / 8;
constexpr int PADC = 4;    // complex padding per smem row (bank spread)

__device__ __forceinline__ void cpAsync16(void* dst, const void* src, bool pred) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpCommit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpWait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int M>
struct GemmCfg {
  static constexpr int MW = M / 8;   // rows per warp
  static constexpr int MB = MW / 8;  // m-blocks per warp
  // A chunk: non-transposed [M][KC+PADC]; transposed [KC][M] (rows of A).
  static constexpr int A_ELEMS = M * (KC + PADC) > KC * M ? M * (KC + PADC) : KC * M;
  static constexpr int B_ELEMS = NTILE * (KC + PADC);
  static constexpr int STAGE = A_ELEMS + B_ELEMS;  // double2
  static constexpr size_t SMEM = 2 * STAGE * sizeof(double2);
};

// item = ((p * 2 + t) * nTiles + tile); t = 1 is the transposed product.
template <int M, int MODE>
__global__ void __launch_bounds__(NT, 1)
binprodGemm(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
            long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int nrhs) {
  using C = GemmCfg<M>;
  extern __shared__ __align__(16) double2 gsm[];
  const int nTiles = (nrhs + NTILE - 1) / NTILE;
  const long long items = npairs * 2 * nTiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const long long B = static_cast<long long>(nrhs) * M;

  for (long long item = blockIdx.x; item < items; item += gridDim.x) {
    const int tile = static_cast<int>(item % nTiles);
    const int t = static_cast<int>((item / nTiles) & 1);
    const long long p = item / (2 * nTiles);
    const int f = pairF[p], g = pairG[p];
    if (t == 1 && f == g) continue;  // self-paired bin: one product only
    const int bin = t == 0 ? f : g;
    const double2* A = S + p * M * M;
    const double2* X = xhat + static_cast<long long>(bin) * B;  // column n at X + n*M
    double2* Y = yhat + static_cast<long long>(bin) * B;
    const int n0 = tile * NTILE;

    constexpr bool FOURM = MODE == 1;
    constexpr int NACC = FOURM ? 2 : 3;
    double acc[C::MB][NB][NACC][2];  // [mblock][nblock][S1/S2/S3 or Re/Im][c0/c1]
#pragma unroll
    for (int a = 0; a < C::MB; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < NACC; ++q) acc[a][b][q][0] = acc[a][b][q][1] = 0.0;

    auto load = [&](int kc, int stage) {
      double2* sA = gsm + stage * C::STAGE;
      double2* sB = sA + C::A_ELEMS;
      const int k0 = kc * KC;
      if (t == 0) {  // sA[i][k] = A[i][k0 + k]
        for (int q = threadIdx.x; q < M * KC; q += NT) {
          const int i = q / KC, k = q % KC;
          cpAsync16(sA + i * (KC + PADC) + k, A + static_cast<long long>(i) * M + k0 + k, true);
        }
      } else {  // sA[k][i] = A[k0 + k][i]  (contiguous rows)
        for (int q = threadIdx.x; q < KC * M; q += NT) cpAsync16(sA + q, A + static_cast<long long>(k0) * M + q, true);
      }
      for (int q = threadIdx.x; q < NTILE * KC; q += NT) {  // sB[n][k] = X[n0+n][k0+k]
        const int n = q / KC, k = q % KC;
        const bool ok = n0 + n < nrhs;
        cpAsync16(sB + n * (KC + PADC) + k, X + static_cast<long long>(ok ? n0 + n : 0) * M + k0 + k, ok);
      }
      cpCommit();
    };

    constexpr int NKC = M / KC;
    load(0, 0);
    for (int kc = 0; kc < NKC; ++kc) {
      if (kc + 1 < NKC) {
        load(kc + 1, (kc + 1) & 1);
        cpWait<1>();
      } else {
        cpWait<0>();
      }
      __syncthreads();
      const double2* sA = gsm + (kc & 1) * C::STAGE;
      const double2* sB = sA + C::A_ELEMS;
#pragma unroll
      for (int kk = 0; kk < KC; kk += 4) {
        double ar[C::MB], ai[C::MB], as[C::MB], br[NB], bi[NB], bs[NB];
#pragma unroll
        for (int a = 0; a < C::MB; ++a) {
          const int i = warp * C::MW + a * 8 + gid;
          const double2 v = t == 0 ? sA[i * (KC + PADC) + kk + tig] : sA[(kk + tig) * M + i];
          ar[a] = v.x;
          ai[a] = v.y;
          as[a] = FOURM ? -v.y : v.x + v.y;  // 4M: the negated imaginary part
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const double2 v = sB[(b * 8 + gid) * (KC + PADC) + kk + tig];
          br[b] = v.x;
          bi[b] = v.y;
          if (!FOURM) bs[b] = v.x + v.y;
        }
#pragma unroll
        for (int a = 0; a < C::MB; ++a) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (FOURM) {
              dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
              dmma(acc[a][b][1][0], acc[a][b][1][1], ar[a], bi[b]);
              dmma(acc[a][b][0][0], acc[a][b][0][1], as[a], bi[b]);
              dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], br[b]);
            } else {
              dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
              dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
              dmma(acc[a][b][2][0], acc[a][b][2][1], as[a], bs[b]);
            }
          }
        }
      }
      __syncthreads();
    }
    // D fragment: row gid, columns 2*tig + {0,1}; Y[n][i] (column n contiguous).
#pragma unroll
    for (int a = 0; a < C::MB; ++a) {
      const int i = warp * C::MW + a * 8 + gid;
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = n0 + b * 8 + 2 * tig + h;
          if (n >= nrhs) continue;
          if (FOURM) {
            Y[static_cast<long long>(n) * M + i] = make_double2(acc[a][b][0][h], acc[a][b][1][h]);
          } else {
            const double s1 = acc[a][b][0][h], s2 = acc[a][b][1][h], s3 = acc[a][b][NACC - 1][h];
            Y[static_cast<long long>(n) * M + i] = make_double2(s1 - s2, s3 - s1 - s2);
          }
        }
    }
  }
}

template <int M, int MODE>
void launchGemm(Ctx& c, int nrhs) {
  using C = GemmCfg<M>;
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodGemm<M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(C::SMEM)));
  });
  const int nTiles = (nrhs + NTILE - 1) / NTILE;
  const long long items = c.npairs * 2 * nTiles;
  const int grid = static_cast<int>(std::min<long long>(items, 16LL * smCount(c.device)));
  binprodGemm<M, MODE>
      <<<grid, NT, C::SMEM, c.stream>>>(c.dSpectra, c.dPairF, c.dPairG, c.npairs, c.dXhat, c.dYhat, nrhs);
}

// Second shape of the same product: a CTA of 4 warps owns 64 rows x NTILE
// right-hand sides of one (pair, transpose) item, K in chunks of 16 through
// an NST-stage cp.async ring with ONE barrier per chunk. At 77-115 KB of
// shared memory and 128 threads two CTAs share an SM, so one CTA's
// prologue (first chunks in flight, nothing to multiply yet) and epilogue
// (stores draining, CTA exit, the next CTA's launch) run under the other
// CTA's DMMA stream; with one 8-warp CTA per SM the pipe idled there (ncu:
// 18 % of the warp samples outside the chunk loop).
constexpr int NT2 = 128;
constexpr int KC2 = 16;
constexpr int RC2 = 64;   // rows per CTA: 4 warps x 2 m-blocks x 8
constexpr int PADT = 2;   // transposed A chunk [k][RC2 + PADT]: the four tig rows hit distinct banks

template <int NST>
struct Gemm2Cfg {
  static constexpr int A_ELEMS = RC2 * (KC2 + PADC) > KC2 * (RC2 + PADT) ? RC2 * (KC2 + PADC) : KC2 * (RC2 + PADT);
  static constexpr int B_ELEMS = NTILE * (KC2 + PADC);
  static constexpr int STAGE = A_ELEMS + B_ELEMS;  // double2
  static constexpr size_t SMEM = NST * STAGE * sizeof(double2);
};

// item = (((p * 2 + t) * nTiles + tile) * (M / RC2) + h); h selects the 64-row part.
template <int M, int NST, bool LATE>
__global__ void __launch_bounds__(NT2, 2)
binprodGemm2(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
             long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int nrhs) {
  using C = Gemm2Cfg<NST>;
  constexpr int NH = M / RC2;
  constexpr int MB = 2;
  extern __shared__ __align__(16) double2 gsm[];
  const int nTiles = (nrhs + NTILE - 1) / NTILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const long long B = static_cast<long long>(nrhs) * M;

  long long item = blockIdx.x;
  const int h = static_cast<int>(item % NH);
  item /= NH;
  const int tile = static_cast<int>(item % nTiles);
  const int t = static_cast<int>((item / nTiles) & 1);
  const long long p = item / (2 * nTiles);
  const int f = pairF[p], g = pairG[p];
  if (t == 1 && f == g) return;  // self-paired bin: one product only
  const int bin = t == 0 ? f : g;
  const int i0 = h * RC2;
  const double2* A = S + p * M * M;
  const double2* X = xhat + static_cast<long long>(bin) * B;  // column n at X + n*M
  double2* Y = yhat + static_cast<long long>(bin) * B;
  const int n0 = tile * NTILE;

  double acc[MB][NB][3][2];  // [mblock][nblock][S1/S2/S3][c0/c1]
#pragma unroll
  for (int a = 0; a < MB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[a][b][q][0] = acc[a][b][q][1] = 0.0;

  auto loadA = [&](int kc) {
    double2* sA = gsm + (kc % NST) * C::STAGE;
    const int k0 = kc * KC2;
    if (t == 0) {  // sA[i][k] = A[i0 + i][k0 + k]
#pragma unroll
      for (int q = threadIdx.x; q < RC2 * KC2; q += NT2) {
        const int i = q / KC2, k = q % KC2;
        cpAsync16(sA + i * (KC2 + PADC) + k, A + static_cast<long long>(i0 + i) * M + k0 + k, true);
      }
    } else {  // sA[k][i] = A[k0 + k][i0 + i]  (contiguous runs of RC2)
#pragma unroll
      for (int q = threadIdx.x; q < KC2 * RC2; q += NT2) {
        const int k = q / RC2, i = q % RC2;
        cpAsync16(sA + k * (RC2 + PADT) + i, A + static_cast<long long>(k0 + k) * M + i0 + i, true);
      }
    }
  };
  auto loadB = [&](int kc) {
    double2* sB = gsm + (kc % NST) * C::STAGE + C::A_ELEMS;
    const int k0 = kc * KC2;
#pragma unroll
    for (int q = threadIdx.x; q < NTILE * KC2; q += NT2) {  // sB[n][k] = X[n0+n][k0+k]
      const int n = q / KC2, k = q % KC2;
      const bool ok = n0 + n < nrhs;
      cpAsync16(sB + n * (KC2 + PADC) + k, X + static_cast<long long>(ok ? n0 + n : 0) * M + k0 + k, ok);
    }
  };

  constexpr int NKC = M / KC2;
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) {
    loadA(q);
    loadB(q);
    cpCommit();
  }
  for (int kc = 0; kc < NKC; ++kc) {
    cpWait<NST - 2>();  // this thread's pieces of chunk kc have landed
    __syncthreads();    // everyone's have, and everyone is done with chunk kc - 1
    // Chunk kc + NST - 1 goes into chunk kc - 1's buffer. LATE: its cp.async
    // pieces and their address arithmetic are issued between this chunk's
    // DMMA groups (A after the first k step, X after the second) instead of
    // ahead of them, where every warp of the CTA did that work with the pipe
    // idle right after the barrier.
    const bool more = kc + NST - 1 < NKC;
    if (!LATE) {
      if (more) {
        loadA(kc + NST - 1);
        loadB(kc + NST - 1);
      }
      cpCommit();  // (an empty group keeps the wait count uniform)
    }
    const double2* sA = gsm + (kc % NST) * C::STAGE;
    const double2* sB = sA + C::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < KC2; kk += 4) {
      double ar[MB], ai[MB], as[MB], br[NB], bi[NB], bs[NB];
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        const int i = warp * (MB * 8) + a * 8 + gid;
        const double2 v = t == 0 ? sA[i * (KC2 + PADC) + kk + tig] : sA[(kk + tig) * (RC2 + PADT) + i];
        ar[a] = v.x;
        ai[a] = v.y;
        as[a] = v.x + v.y;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const double2 v = sB[(b * 8 + gid) * (KC2 + PADC) + kk + tig];
        br[b] = v.x;
        bi[b] = v.y;
        bs[b] = v.x + v.y;
      }
#pragma unroll
      for (int a = 0; a < MB; ++a) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
          dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
          dmma(acc[a][b][2][0], acc[a][b][2][1], as[a], bs[b]);
        }
      }
      if (LATE && kk == 0 && more) loadA(kc + NST - 1);
      if (LATE && kk == 4) {
        if (more) loadB(kc + NST - 1);
        cpCommit();
      }
    }
  }
  // D fragment: row gid, columns 2*tig + {0,1}; Y[n][i] (column n contiguous).
#pragma unroll
  for (int a = 0; a < MB; ++a) {
    const int i = i0 + warp * (MB * 8) + a * 8 + gid;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int n = n0 + b * 8 + 2 * tig + hh;
        if (n >= nrhs) continue;
        const double s1 = acc[a][b][0][hh], s2 = acc[a][b][1][hh], s3 = acc[a][b][2][hh];
        Y[static_cast<long long>(n) * M + i] = make_double2(s1 - s2, s3 - s1 - s2);
      }
  }
}

template <int M, int NST, bool LATE>
void launchGemm2(Ctx& c, int nrhs) {
  using C = Gemm2Cfg<NST>;
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodGemm2<M, NST, LATE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(C::SMEM)));
    TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodGemm2<M, NST, LATE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));
  });
  const int nTiles = (nrhs + NTILE - 1) / NTILE;
  const long long items = c.npairs * 2 * nTiles * (M / RC2);
  binprodGemm2<M, NST, LATE><<<static_cast<unsigned>(items), NT2, C::SMEM, c.stream>>>(c.dSpectra, c.dPairF, c.dPairG,
                                                                                c.npairs, c.dXhat, c.dYhat, nrhs);
}

// TBT_GEMM: "4m" the 4M form; "wide" the one-CTA-per-SM 3M kernel; default
// for m = 128 the two-CTAs-per-SM kernel, 2-stage ring, late cp.async issue
// ("late3": 3-stage ring; "pair2" / "pair3": loads issued ahead of the chunk).
int gemmShape() {
  static const int v = [] {
    const char* e = getenv("TBT_GEMM");
    if (e && strcmp(e, "wide") == 0) return 0;
    if (e && strcmp(e, "pair2") == 0) return 2;
    if (e && strcmp(e, "pair3") == 0) return 3;
    if (e && strcmp(e, "late3") == 0) return 13;
    return 12;
  }();
  return v;
}

int gemm4m() {
  static const int on = [] {
    const char* e = getenv("TBT_GEMM");
    return e && strcmp(e, "4m") == 0 ? 1 : 0;
  }();
  return on;
}

}  // namespace

bool launchBinProductGemm(Ctx& c, int nrhs) {
  const int four = gemm4m();
  if (c.m == 64 && !four && gemmShape()) {
    launchGemm2<64, 2, true>(c, nrhs);
    TBT_CUDA_CHECK(cudaGetLastError());
    return true;
  }
  if (c.m == 128 && !four && gemmShape()) {
    switch (gemmShape()) {
      case 2: launchGemm2<128, 2, false>(c, nrhs); break;
      case 3: launchGemm2<128, 3, false>(c, nrhs); break;
      case 13: launchGemm2<128, 3, true>(c, nrhs); break;
      default: launchGemm2<128, 2, true>(c, nrhs);
    }
    TBT_CUDA_CHECK(cudaGetLastError());
    return true;
  }
  switch (c.m) {
    case 64: four ? launchGemm<64, 1>(c, nrhs) : launchGemm<64, 0>(c, nrhs); break;
    case 128: four ? launchGemm<128, 1>(c, nrhs) : launchGemm<128, 0>(c, nrhs); break;
    default: return false;
  }
  TBT_CUDA_CHECK(cudaGetLastError());
  return true;
}

}  // namespace tbt
