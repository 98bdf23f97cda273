// Kernel K3: per-frequency-bin block product, the dominant HBM stream.
//
// Replaces applyA's per-bin loop (proj/src/linsolve.cpp:276-282), which
// streams the whole spectrum set once per column:
//     acc[f] += ahat[(m*e5+n)*L + f] * xhat[n*L + f].
// Here each stored block Ahat_p (bin pair {f, g = -f}, see spectra.cu) is
// read from HBM exactly once per apply and used twice:
//     yhat_f = Ahat_p    xhat_f
//     yhat_g = Ahat_p^T  xhat_g          (skipped when g == f)
// so the HBM traffic of the dominant stream is half the reference's.
//
// Thread mapping (256 threads, TC lanes across columns, 256/TC row groups):
// each thread owns an RPT x CPT register tile of the current row chunk;
// the row products reduce over the TC column lanes with warp shuffles, the
// column products accumulate in registers across chunks and reduce over
// the row groups once per block. Every spectrum element is loaded once
// (16-byte streaming loads, evict-first) and feeds 2 complex MACs.
#include <algorithm>

#include "ptx.cuh"
#include "tbt_internal.cuh"

namespace tbt {
namespace {

__device__ __forceinline__ double2 shflXor(double2 v, int off) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, off);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, off);
  return v;
}

template <int M, int TC, int RCH>
__global__ void __launch_bounds__(256, 2)
binprodTile(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
            long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int nrhs) {
  constexpr int NT = 256;
  constexpr int TRN = NT / TC;
  constexpr int CPT = M / TC;
  constexpr int RPT = RCH / TRN;
  constexpr int NCH = M / RCH;
  static_assert(M % TC == 0 && RCH % TRN == 0 && M % RCH == 0, "tile");
  __shared__ double2 sxg[M];
  __shared__ double2 sred[NT / 32][M];
  const int tc = threadIdx.x % TC, tr = threadIdx.x / TC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long B = static_cast<long long>(nrhs) * M;

  for (long long p = blockIdx.x; p < npairs; p += gridDim.x) {
    const int f = pairF[p], g = pairG[p];
    const double2* A = S + p * M * M;
    for (int rhs = 0; rhs < nrhs; ++rhs) {
      const double2* xf = xhat + f * B + rhs * M;
      const double2* xg = xhat + g * B + rhs * M;
      double2* yf = yhat + f * B + rhs * M;
      double2* yg = yhat + g * B + rhs * M;
      __syncthreads();
      for (int q = threadIdx.x; q < M; q += NT) sxg[q] = xg[q];
      double2 xfr[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) xfr[j] = xf[tc + TC * j];
      double2 yga[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) yga[j] = make_double2(0.0, 0.0);
      __syncthreads();
#pragma unroll 1
      for (int ch = 0; ch < NCH; ++ch) {
        double2 a[RPT][CPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int j = 0; j < CPT; ++j)
            a[i][j] = __ldcs(A + static_cast<long long>(ch * RCH + tr + TRN * i) * M + tc + TC * j);
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          double2 s = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < CPT; ++j) cfma(s, a[i][j], xfr[j]);
#pragma unroll
          for (int off = TC / 2; off >= 1; off >>= 1) s = cadd(s, shflXor(s, off));
          if (tc == 0) yf[ch * RCH + tr + TRN * i] = s;
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const double2 xv = sxg[ch * RCH + tr + TRN * i];
#pragma unroll
          for (int j = 0; j < CPT; ++j) cfma(yga[j], a[i][j], xv);
        }
      }
      if (TC == 16) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) yga[j] = cadd(yga[j], shflXor(yga[j], 16));
      }
      if (lane < TC) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) sred[warp][tc + TC * j] = yga[j];
      }
      __syncthreads();
      if (f != g) {
        for (int q = threadIdx.x; q < M; q += NT) {
          double2 s = sred[0][q];
#pragma unroll
          for (int w = 1; w < NT / 32; ++w) s = cadd(s, sred[w][q]);
          yg[q] = s;
        }
      }
    }
  }
}

// Any m: one CTA per pair; row products by row-owner threads, column
// products by column-owner threads (second sweep hits L1/L2).
__global__ void __launch_bounds__(128)
binprodGeneric(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
               long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int m,
               int nrhs, int acc = 0, double sg = 1.0) {
  const long long B = static_cast<long long>(nrhs) * m;
  for (long long p = blockIdx.x; p < npairs; p += gridDim.x) {
    const int f = pairF[p], g = pairG[p];
    const double2* A = S + p * m * m;
    for (int rhs = 0; rhs < nrhs; ++rhs) {
      const double2* xf = xhat + f * B + rhs * m;
      const double2* xg = xhat + g * B + rhs * m;
      for (int a = threadIdx.x; a < m; a += blockDim.x) {
        double2 s = make_double2(0.0, 0.0);
        for (int b = 0; b < m; ++b) cfma(s, A[static_cast<long long>(a) * m + b], xf[b]);
        double2& yo = yhat[f * B + rhs * m + a];
        yo = acc ? cadd(yo, s) : s;
      }
      if (f != g)
        for (int b = threadIdx.x; b < m; b += blockDim.x) {
          double2 s = make_double2(0.0, 0.0);
          for (int a = 0; a < m; ++a) cfma(s, A[static_cast<long long>(a) * m + b], xg[a]);
          double2& yo = yhat[g * B + rhs * m + b];
          const double2 v = make_double2(sg * s.x, sg * s.y);
          yo = acc ? cadd(yo, v) : v;
        }
    }
  }
}

// Any m <= 64, any nrhs: CTA per (pair, chunk of kMultiRc right-hand sides).
// The m x m block (row stride ld = m | 1, odd, so a warp's row-owner reads
// and column-owner reads both spread over the bank groups) and the chunk's
// xhat_f / xhat_g columns are staged in shared memory; thread per output.
constexpr int kMultiRc = 8;
__global__ void __launch_bounds__(256)
binprodMulti(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
             long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int m, int nrhs) {
  extern __shared__ double2 smb[];
  const int ld = m | 1;
  double2* sA = smb;                      // [m][ld]
  double2* sxf = sA + m * ld;             // [RC][m]
  double2* sxg = sxf + kMultiRc * m;      // [RC][m]
  const int nch = (nrhs + kMultiRc - 1) / kMultiRc;
  const long long B = static_cast<long long>(nrhs) * m;
  for (long long item = blockIdx.x; item < npairs * nch; item += gridDim.x) {
    const long long p = item / nch;
    const int r0 = static_cast<int>(item % nch) * kMultiRc, rc = min(kMultiRc, nrhs - r0);
    const long long f = pairF[p], g = pairG[p];
    const double2* A = S + p * m * m;
    __syncthreads();  // previous item's readers are done
    for (int q = threadIdx.x; q < m * m; q += blockDim.x) sA[(q / m) * ld + q % m] = A[q];
    for (int q = threadIdx.x; q < rc * m; q += blockDim.x) {
      sxf[q] = xhat[f * B + static_cast<long long>(r0) * m + q];
      sxg[q] = xhat[g * B + static_cast<long long>(r0) * m + q];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < rc * m; o += blockDim.x) {  // yhat_f = A xhat_f
      const int rhs = o / m, a = o % m;
      double2 acc = make_double2(0.0, 0.0);
      for (int b = 0; b < m; ++b) cfma(acc, sA[a * ld + b], sxf[rhs * m + b]);
      yhat[f * B + static_cast<long long>(r0) * m + o] = acc;
    }
    if (f != g)
      for (int o = threadIdx.x; o < rc * m; o += blockDim.x) {  // yhat_g = A^T xhat_g
        const int rhs = o / m, b = o % m;
        double2 acc = make_double2(0.0, 0.0);
        for (int a = 0; a < m; ++a) cfma(acc, sA[a * ld + b], sxg[rhs * m + a]);
        yhat[g * B + static_cast<long long>(r0) * m + o] = acc;
      }
  }
}

// ---------------------------------------------------------------------------
// K3 v2 (single RHS): persistent, warp-specialised, TMA-engine ring.
// One producer warp streams each (pair, row-chunk) of the spectrum plus the
// matching xhat segments into a STAGES-deep shared-memory ring with
// cp.async.bulk (evict-first L2 policy for the spectrum, evict-last for the
// vectors); eight consumer warps compute from shared memory and release the
// slot as soon as their operands are in registers. One CTA per SM.
template <int M, int TC, int RCH, int STAGES>
struct RingCfg {
  static constexpr int NT = 256;
  static constexpr int TRN = NT / TC;
  static constexpr int CPT = M / TC;
  static constexpr int RPT = RCH / TRN;
  static constexpr int NCH = M / RCH;
  static constexpr uint32_t CHUNK = RCH * M * 16;
  static constexpr uint32_t XF = M * 16;
  static constexpr uint32_t XG = RCH * 16;
  static constexpr uint32_t STAGE = CHUNK + XF + XG;
  static constexpr uint32_t RED = 2 * (NT / 32) * M * 16;
  static constexpr uint32_t SMEM = STAGES * STAGE + RED + 2 * STAGES * 8;
  static_assert(M % TC == 0 && RCH % TRN == 0 && M % RCH == 0 && STAGE % 16 == 0, "ring tile");
};

template <int M, int TC, int RCH, int STAGES>
__global__ void __launch_bounds__(288, 1)
binprodRing(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
            long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat) {
  using C = RingCfg<M, TC, RCH, STAGES>;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* red = reinterpret_cast<double2*>(smem + STAGES * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE + C::RED);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbarInit(full + s, 1);
      mbarInit(empty + s, C::NT / 32);
    }
    fenceBarrierInit();
  }
  __syncthreads();
  if (blockIdx.x >= npairs) return;
  const long long mine = (npairs - 1 - blockIdx.x) / gridDim.x + 1;
  const long long total = mine * C::NCH;

  if (warp == C::NT / 32) {  // producer warp
    if (lane == 0) {
      const uint64_t polS = policyEvictFirst();
      const uint64_t polX = policyEvictLast();
      for (long long it = 0; it < total; ++it) {
        const int s = static_cast<int>(it % STAGES);
        const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
        const long long p = blockIdx.x + (it / C::NCH) * gridDim.x;
        const int ch = static_cast<int>(it % C::NCH);
        const long long f = pairF[p], g = pairG[p];
        mbarWait(empty + s, ph ^ 1u);
        unsigned char* st = smem + s * C::STAGE;
        mbarArriveExpectTx(full + s, C::STAGE);
        bulkG2S(st, S + p * M * M + static_cast<long long>(ch) * RCH * M, C::CHUNK, full + s, polS);
        bulkG2S(st + C::CHUNK, xhat + f * M, C::XF, full + s, polX);
        bulkG2S(st + C::CHUNK + C::XF, xhat + g * M + ch * RCH, C::XG, full + s, polX);
      }
    }
    return;
  }

  const int tc = threadIdx.x % TC, tr = threadIdx.x / TC;
  double2 yga[C::CPT];
  for (long long it = 0; it < total; ++it) {
    const int s = static_cast<int>(it % STAGES);
    const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
    const long long pi = it / C::NCH;
    const int ch = static_cast<int>(it % C::NCH);
    const long long p = blockIdx.x + pi * gridDim.x;
    if (ch == 0) {
#pragma unroll
      for (int j = 0; j < C::CPT; ++j) yga[j] = make_double2(0.0, 0.0);
    }
    mbarWait(full + s, ph);
    const double2* A = reinterpret_cast<const double2*>(smem + s * C::STAGE);
    const double2* xf = A + RCH * M;
    const double2* xg = xf + M;
    double2 a[C::RPT][C::CPT], xfr[C::CPT], xgv[C::RPT];
#pragma unroll
    for (int j = 0; j < C::CPT; ++j) xfr[j] = xf[tc + TC * j];
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      xgv[i] = xg[tr + C::TRN * i];
#pragma unroll
      for (int j = 0; j < C::CPT; ++j) a[i][j] = A[(tr + C::TRN * i) * M + tc + TC * j];
    }
    __syncwarp();
    if (lane == 0) mbarArrive(empty + s);  // slot free: operands are in registers

    const long long f = pairF[p], g = pairG[p];
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < C::CPT; ++j) cfma(acc, a[i][j], xfr[j]);
#pragma unroll
      for (int off = TC / 2; off >= 1; off >>= 1) acc = cadd(acc, shflXor(acc, off));
      if (tc == 0) yhat[f * M + ch * RCH + tr + C::TRN * i] = acc;
    }
#pragma unroll
    for (int i = 0; i < C::RPT; ++i)
#pragma unroll
      for (int j = 0; j < C::CPT; ++j) cfma(yga[j], a[i][j], xgv[i]);

    if (ch == C::NCH - 1) {
      if (TC == 16) {
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) yga[j] = cadd(yga[j], shflXor(yga[j], 16));
      }
      double2* rb = red + (pi & 1) * (C::NT / 32) * M;
      if (lane < TC) {
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) rb[warp * M + tc + TC * j] = yga[j];
      }
      namedBarrier(1, C::NT);
      if (f != g) {
        for (int q = threadIdx.x; q < M; q += C::NT) {
          double2 acc = rb[q];
#pragma unroll
          for (int w = 1; w < C::NT / 32; ++w) acc = cadd(acc, rb[w * M + q]);
          yhat[g * M + q] = acc;
        }
      }
    }
  }
}

template <int M, int TC, int RCH, int STAGES>
void launchRing(Ctx& c) {
  using C = RingCfg<M, TC, RCH, STAGES>;
  static std::atomic<unsigned long long> attrSet{0};
  oncePerDevice(attrSet, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodRing<M, TC, RCH, STAGES>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  const int sms = smCount(c.device);
  const int grid = static_cast<int>(std::min<long long>(c.npairs, sms));
  binprodRing<M, TC, RCH, STAGES><<<grid, C::NT + 32, C::SMEM, c.stream>>>(c.dSpectra, c.dPairF, c.dPairG, c.npairs,
                                                                          c.dXhat, c.dYhat);
}

// ---------------------------------------------------------------------------
// K3 for one right-hand side and ANY m up to 256 (the tuned ring kernels
// above are instantiated for m = 64, 128, 192): the same warp-specialised
// cp.async.bulk ring and register tiling with m a run-time value. Chunks
// are 16 contiguous rows of the block (the last one may be partial); warp w
// owns rows w and w + 8 of a chunk, lane l columns l + 32 j (j < CPT, CPT =
// ceil(m / 32) a template parameter; columns >= m are predicated off). A
// warp loads its operands into registers and releases the slot before
// computing; column products accumulate in registers across the pair's
// chunks and meet across the warps in shared memory once per pair.
constexpr uint32_t kAnyStages = 6;
constexpr int kAnyRows = 16;

template <int CPT>
__global__ void __launch_bounds__(288, 1)
binprodRingAny(const double2* __restrict__ S, const int* __restrict__ pairF, const int* __restrict__ pairG,
               long long npairs, const double2* __restrict__ xhat, double2* __restrict__ yhat, int m,
               uint32_t stageBytes, int nst, int accum, double sg) {
  constexpr int NT = 256, RPT = kAnyRows / (NT / 32);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stageBytes);
  uint64_t* empty = full + nst;
  double2* red = reinterpret_cast<double2*>(smem + nst * stageBytes + 2 * nst * 8);  // [2][8][m]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbarInit(full + s, 1);
      mbarInit(empty + s, NT / 32);
    }
    fenceBarrierInit();
  }
  __syncthreads();
  if (blockIdx.x >= npairs) return;
  const int nch = (m + kAnyRows - 1) / kAnyRows;
  const long long mine = (npairs - 1 - blockIdx.x) / gridDim.x + 1;
  const long long total = mine * nch;
  const long long mm = static_cast<long long>(m) * m;
  const uint32_t xfOff = static_cast<uint32_t>(kAnyRows) * m * 16;

  if (warp == NT / 32) {  // producer
    if (lane == 0) {
      const uint64_t polS = policyEvictFirst();
      const uint64_t polX = policyEvictLast();
      for (long long it = 0; it < total; ++it) {
        const int s = static_cast<int>(it % nst);
        const uint32_t ph = static_cast<uint32_t>((it / nst) & 1);
        const long long p = blockIdx.x + (it / nch) * gridDim.x;
        const int ch = static_cast<int>(it % nch);
        const int rr = min(kAnyRows, m - ch * kAnyRows);
        const long long f = pairF[p], g = pairG[p];
        const uint32_t chunk = static_cast<uint32_t>(rr) * m * 16, xf = static_cast<uint32_t>(m) * 16;
        mbarWait(empty + s, ph ^ 1u);
        unsigned char* st = smem + s * stageBytes;
        mbarArriveExpectTx(full + s, chunk + xf + static_cast<uint32_t>(rr) * 16);
        bulkG2S(st, S + p * mm + static_cast<long long>(ch) * kAnyRows * m, chunk, full + s, polS);
        bulkG2S(st + xfOff, xhat + f * m, xf, full + s, polX);
        bulkG2S(st + xfOff + xf, xhat + g * m + static_cast<long long>(ch) * kAnyRows, static_cast<uint32_t>(rr) * 16,
                full + s, polX);
      }
    }
    return;
  }

  double2 yga[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) yga[j] = make_double2(0.0, 0.0);
  for (long long it = 0; it < total; ++it) {
    const int s = static_cast<int>(it % nst);
    const uint32_t ph = static_cast<uint32_t>((it / nst) & 1);
    const long long pi = it / nch;
    const long long p = blockIdx.x + pi * gridDim.x;
    const int ch = static_cast<int>(it % nch);
    const int rr = min(kAnyRows, m - ch * kAnyRows);
    mbarWait(full + s, ph);
    const double2* A = reinterpret_cast<const double2*>(smem + s * stageBytes);
    const double2* xf = A + kAnyRows * m;
    const double2* xg = xf + m;
    double2 a[RPT][CPT], xfr[CPT], xgv[RPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = lane + 32 * j;
      xfr[j] = c < m ? xf[c] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = warp + (NT / 32) * i;
      const bool rok = r < rr;
      xgv[i] = rok ? xg[r] : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = lane + 32 * j;
        a[i][j] = rok && c < m ? A[r * m + c] : make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    if (lane == 0) mbarArrive(empty + s);  // slot free: operands are in registers

    const long long f = pairF[p], g = pairG[p];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = warp + (NT / 32) * i;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < CPT; ++j) cfma(acc, a[i][j], xfr[j]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) acc = cadd(acc, shflXor(acc, off));
      if (lane == 0 && r < rr) {
        double2& yo = yhat[f * m + static_cast<long long>(ch) * kAnyRows + r];
        yo = accum ? cadd(yo, acc) : acc;
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int j = 0; j < CPT; ++j) cfma(yga[j], a[i][j], xgv[i]);

    if (ch == nch - 1) {
      double2* rb = red + (pi & 1) * (NT / 32) * m;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = lane + 32 * j;
        if (c < m) rb[warp * m + c] = yga[j];
        yga[j] = make_double2(0.0, 0.0);
      }
      namedBarrier(1, NT);
      if (f != g)
        for (int q = threadIdx.x; q < m; q += NT) {
          double2 acc = rb[q];
#pragma unroll
          for (int w = 1; w < NT / 32; ++w) acc = cadd(acc, rb[w * m + q]);
          const double2 v = make_double2(sg * acc.x, sg * acc.y);
          yhat[g * m + q] = accum ? cadd(yhat[g * m + q], v) : v;
        }
    }
  }
}

template <int CPT>
void launchRingAny(Ctx& c, const double2* S, int accum, double sg) {
  const int m = c.m;
  const uint32_t stage =
      static_cast<uint32_t>((static_cast<size_t>(kAnyRows) * m * 16 + m * 16 + kAnyRows * 16 + 127) / 128 * 128);
  // ~150 KB of chunks in flight per SM (2..6 stages; C2 / C4 measured best
  // around 128 KB for this stream).
  const int nst = static_cast<int>(std::max<uint32_t>(2, std::min<uint32_t>(kAnyStages, 150u * 1024 / stage)));
  const size_t smem = nst * static_cast<size_t>(stage) + 2 * nst * 8 + 2 * 8 * static_cast<size_t>(m) * sizeof(double2);
  static std::atomic<unsigned long long> attrSet{0};
  oncePerDevice(attrSet, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodRingAny<CPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
  });
  const int grid = static_cast<int>(std::min<long long>(c.npairs, smCount(c.device)));
  binprodRingAny<CPT><<<grid, 288, smem, c.stream>>>(S, c.dPairF, c.dPairG, c.npairs, c.dXhat, c.dYhat, m, stage,
                                                     nst, accum, sg);
}

void launchStream(Ctx& c, const double2* S, int accum = 0, double sg = 1.0) {
  switch ((c.m + 31) / 32) {
    case 1: launchRingAny<1>(c, S, accum, sg); break;
    case 2: launchRingAny<2>(c, S, accum, sg); break;
    case 3: launchRingAny<3>(c, S, accum, sg); break;
    case 4: launchRingAny<4>(c, S, accum, sg); break;
    case 5: launchRingAny<5>(c, S, accum, sg); break;
    case 6: launchRingAny<6>(c, S, accum, sg); break;
    case 7: launchRingAny<7>(c, S, accum, sg); break;
    default: launchRingAny<8>(c, S, accum, sg); break;
  }
}

template <int M, int TC, int RCH>
void launchTile(Ctx& c, int nrhs) {
  const int sms = smCount(c.device);
  const long long grid = std::min<long long>(c.npairs, 2LL * sms);
  binprodTile<M, TC, RCH><<<static_cast<int>(grid), 256, 0, c.stream>>>(
      c.dSpectra, c.dPairF, c.dPairG, c.npairs, c.dXhat, c.dYhat, nrhs);
}

}  // namespace

int binprodVariant(int m) {
  switch (m) {
    case 64: return 1;
    case 128: return 2;
    case 192: return 3;
    default: return 0;
  }
}

void launchBinProduct(Ctx& c, int nrhs) {
  if (nrhs >= kGemmMinRhs && launchBinProductGemm(c, nrhs)) return;
  if (nrhs == 1 && c.binprodKernel >= 11) {
    switch (c.binprodKernel) {
      case 11: launchRing<64, 16, 64, 3>(c); break;
      case 12: launchRing<128, 32, 16, 4>(c); break;
      case 13: launchRing<192, 32, 16, 3>(c); break;
    }
    TBT_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (nrhs == 1 && binprodVariant(c.m) == 0 && c.m <= 256) {
    launchStream(c, c.dSpectra);
    TBT_CUDA_CHECK(cudaGetLastError());
    return;
  }
  switch (binprodVariant(c.m)) {
    case 1: launchTile<64, 16, 64>(c, nrhs); break;
    case 2: launchTile<128, 32, 32>(c, nrhs); break;
    case 3: launchTile<192, 32, 16>(c, nrhs); break;
    default: {
      const int sms = smCount(c.device);
      if (c.m <= 64) {
        const int ld = c.m | 1;
        const size_t smem = (static_cast<size_t>(c.m) * ld + 2 * kMultiRc * c.m) * sizeof(double2);
        static std::atomic<unsigned long long> attr{0};
        oncePerDevice(attr, [] {
          TBT_CUDA_CHECK(cudaFuncSetAttribute(binprodMulti, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        });
        const long long items = c.npairs * ((nrhs + kMultiRc - 1) / kMultiRc);
        const long long grid = std::min<long long>(items, 16LL * sms);
        binprodMulti<<<static_cast<int>(grid), 256, smem, c.stream>>>(c.dSpectra, c.dPairF, c.dPairG, c.npairs,
                                                                      c.dXhat, c.dYhat, c.m, nrhs);
        break;
      }
      const long long grid = std::min<long long>(c.npairs, 4LL * sms);
      binprodGeneric<<<static_cast<int>(grid), 128, 0, c.stream>>>(c.dSpectra, c.dPairF, c.dPairG, c.npairs,
                                                                  c.dXhat, c.dYhat, c.m, nrhs);
    }
  }
  TBT_CUDA_CHECK(cudaGetLastError());
}

// FULL generators: yhat += A_a xhat with the anti-reciprocal part's half
// spectrum (the partner product negated: Ahat_a(-f) = -Ahat_a(f)^T).
void launchBinProductAnti(Ctx& c, int nrhs) {
  if (!c.fullMode || !c.dSpectraAnti) return;
  if (nrhs == 1 && c.m <= 256) {
    launchStream(c, c.dSpectraAnti, 1, -1.0);
  } else {
    const long long grid = std::min<long long>(c.npairs, 4LL * smCount(c.device));
    binprodGeneric<<<static_cast<int>(std::max<long long>(grid, 1)), 128, 0, c.stream>>>(
        c.dSpectraAnti, c.dPairF, c.dPairG, c.npairs, c.dXhat, c.dYhat, c.m, nrhs, 1, -1.0);
  }
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
