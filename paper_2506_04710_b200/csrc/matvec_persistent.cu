// The whole single-RHS operator application as ONE persistent cooperative
// kernel (one CTA per SM), replacing the K2 -> K3 -> K4 launch chain of
// apply.cu for the sizes it is instantiated for:
//
//   phase A1  row FFTs along level 0 of x (nx non-zero points per row)
//   --- grid barrier ---
//   phase A2  column FFTs along level 1 (ny non-zero points)  -> xhat
//   --- grid barrier ---
//   phase B   bin-pair products (K3): producer warp streams the spectrum
//             through a cp.async.bulk ring; its first STAGES chunks are
//             issued at kernel start, i.e. the HBM stream ramps up while
//             phase A is still transforming x; meanwhile two auxiliary
//             warps per CTA build the edge/corner correction's term vectors
//   --- grid barrier ---
//   phase C1  inverse column FFTs, keep ny rows (aux warps: correction sums)
//   --- grid barrier ---
//   phase C2  inverse row FFTs, keep nx points, 1/L, + correction -> y
//
// FFT lines are warp-level work items (Stockham in registers, the
// inter-step exchange through a warp-private shared-memory slab, __syncwarp
// only), so the transform phases need no CTA-wide synchronisation.
// Restates applyA + apply (proj/src/linsolve.cpp:260-290,373-388).
#include <algorithm>
#include <cstdlib>

#include "fft_reg.cuh"
#include "gmres_dev.cuh"
#include "grid_sync.cuh"
#include "ptx.cuh"
#include "tbt_internal.cuh"

namespace tbt {
namespace {

using fftreg::dftReg;
using fftreg::Split;

constexpr int kConsumers = 256;
constexpr int kAux = 2;                                   // auxiliary warps
constexpr int kThreadsP = kConsumers + 32 + 32 * kAux;  // + producer warp + auxiliary warps

struct PArgs {
  const double2* S;
  const int* pairF;
  const int* pairG;
  long long npairs;
  const double2* x;
  double2* y;
  double2* xStage;   // zero-copy x (host memory): A1 also writes it here
  const double2* xc; // x as the correction terms read it (xStage or x)
  double2* xhat;
  double2* yhat;
  double2* T;  // [ny][L0][m] intermediate
  const double2* tw0;
  const double2* tw1;
  int nx, ny, L0, L1;
  double scale;
  unsigned* bar;
  unsigned long long* barFlags;  // monotonic grid-barrier arrival counter
  // correction
  int corr;
  const int* tInfo;
  const int* targetList;
  const int* targetPtr;
  int nTargets;
  const int* elemPtr;
  const double2* D;
  const double2* U;
  const double2* V;
  int rank;
  int nTerms;
  int nPairs;
  const int* pInfo;       // [pair][4] {target, source, code0, code1}, code = slot*2+trans or -1
  const int* pTargetPtr;  // [nTargets+1] CSR of pairs by target (same order as targetList)
  double2* tvec;          // [nPairs][M] pair vectors
  double2* ycorr;
  int prefetchAt;               // phase at which the spectrum ring is primed (0 = kernel start)
  long long l2Chunks;           // spectrum chunks per CTA bulk-prefetched into L2 (zero-copy x only)
  int l2At;                     // ... at kernel start (0) or after grid barrier 0 (1)
  const int* skip;              // optional: the whole launch is a no-op when *skip != 0
  int pdl;                      // launched with programmatic stream serialization
  int ctaMajor;                 // CTA-major transform items in every phase (zero-copy launches)
  int rev;                      // phase B walks this CTA's bin pairs last-to-first
  // Optional GMRES epilogue: the low-synchronisation Arnoldi step on y
  // (gmres_dev.cuh), so one cooperative launch is one GMRES iteration.
  int arnoldi;
  GmresArgs gm;
  double2* lsS;
  double2* lsDots;
  double2* lsPart;
  unsigned long long* phaseNs;  // optional: globaltimer at phase boundaries (CTA 0)
  unsigned long long* cta;      // optional (TBT_CTATRACE): per-CTA event times [16][256] of this launch
};

// Per-CTA trace (TBT_CTATRACE=1): 0 start, 1 after the PDL wait, 2+k / 6+k
// arrival at / release from grid barrier k, 10 end of C2, 11 = %smid,
// fused GMRES step: 12 after the y barrier, 13 after the LS dot barrier
// (CTA-local time at which the reduce starts), 14 end of the step.
__device__ __forceinline__ void trace(const PArgs& a, int ev) {
  if (a.cta && threadIdx.x == 0) {
    unsigned long long t;
    if (ev == 11) {
      unsigned s;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
      t = s;
    } else {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    }
    a.cta[ev * kCtaTraceMaxGrid + blockIdx.x] = t;
  }
}

__device__ __forceinline__ void stamp(const PArgs& a, int k) {
  if (a.phaseNs && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.phaseNs[k] = t;
  }
}

// Grid barrier (grid_sync.cuh); with phase timing armed it also records the
// earliest / latest CTA arrival of barrier k (ns) at phaseNs[16+k] / phaseNs[8+k].
__device__ __forceinline__ void gridSync(unsigned long long* counter, const PArgs& a, int k) {
  __syncthreads();
  if (k < 4) trace(a, 2 + k);
  if (threadIdx.x == 0) {
    if (a.phaseNs) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(a.phaseNs + 8 + k, t);
      atomicMin(a.phaseNs + 16 + k, t);
    }
    gridArriveWait(counter);
  }
  if (k < 4) trace(a, 6 + k);
  __syncthreads();
}

__device__ __forceinline__ double2 shflXorP(double2 v, int off) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, off);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, off);
  return v;
}

// Warp-level batched line FFT: WB batch entries per warp, LANES butterfly
// lanes per entry (LANES * WB == 32). For N <= 16 each lane owns a line.
// The slab between the two radix steps is padded: row ii1 of the first step
// starts at ii1 * STR with STR = WB (mod 8), so a warp's first-step stores
// (lanes over ii1 and b) fall into distinct 16-byte bank groups instead of
// one group per ii1 (16-way conflicts at N = 128, 256 unpadded); the second
// step's loads stay contiguous.
template <int N>
struct WarpFft {
  using S = Split<N>;
  static constexpr int LANES = S::R2 == 1 ? 1 : S::LANES;
  static constexpr int WB = 32 / LANES;
  static constexpr int STR =
      WB >= 8 ? S::R1 * WB : S::R1 * WB + ((WB - (S::R1 * WB) % 8) % 8 + 8) % 8;  // padded row stride
  static constexpr int SLAB = S::R2 == 1 ? 0 : S::R2 * STR;  // double2 per warp
};

template <int N, bool INV, class Src, class Snk>
__device__ __forceinline__ void warpLineFft(double2* slab, const double2* tw, Src src, Snk snk) {
  using S = Split<N>;
  using W = WarpFft<N>;
  const int lane = threadIdx.x & 31;
  const int b = lane % W::WB, ii = lane / W::WB;
  if constexpr (S::R2 == 1) {
    double2 u[S::R1];
#pragma unroll
    for (int r = 0; r < S::R1; ++r) u[r] = src(r, b);
    dftReg<S::R1, INV>(u);
#pragma unroll
    for (int r = 0; r < S::R1; ++r) snk(r, b, u[r], r);
  } else {
    if (ii < S::R2) {
      double2 u[S::R1];
#pragma unroll
      for (int r = 0; r < S::R1; ++r) u[r] = src(ii + r * S::R2, b);
      dftReg<S::R1, INV>(u);
#pragma unroll
      for (int r = 0; r < S::R1; ++r) slab[ii * W::STR + r * W::WB + b] = u[r];
    }
    __syncwarp();
    if (ii < S::R1) {
      double2 u[S::R2];
#pragma unroll
      for (int r = 0; r < S::R2; ++r) u[r] = slab[r * W::STR + ii * W::WB + b];
#pragma unroll
      for (int r = 1; r < S::R2; ++r) {
        double2 w = __ldg(tw + r * ii);
        if (INV) w.y = -w.y;
        u[r] = cmul(u[r], w);
      }
      dftReg<S::R2, INV>(u);
#pragma unroll
      for (int r = 0; r < S::R2; ++r) snk(ii + r * S::R1, b, u[r], r);
    }
    __syncwarp();
  }
}

// Output point of register r for the calling lane (matches warpLineFft).
template <int N>
__device__ __forceinline__ int outPoint(int r) {
  using S = Split<N>;
  using W = WarpFft<N>;
  if constexpr (S::R2 == 1) return r;
  const int ii = (threadIdx.x & 31) / W::WB;
  return ii + r * S::R1;
}
template <int N>
__device__ __forceinline__ bool outActive() {
  using S = Split<N>;
  using W = WarpFft<N>;
  if constexpr (S::R2 == 1) return true;
  return (threadIdx.x & 31) / W::WB < S::R1;
}

// Correction, one latency round per phase:
// A1: one warp per term t computes the whole term vector
//       tvec[t] = diag(d) x_src + W2 (W^T x_src)
//     (projections reduced across the warp, then expanded in registers);
// A2: one warp per target element sums its terms' vectors into ycorr[e];
// C2: the inverse-row pass adds ycorr (prefetched before the transform).
// One (target, source) pair: up to two terms sharing x_src (P of the
// target's relation and P^T of the source's relation back, or P and P^T of a
// self relation), tvec[pair] = sum_terms diag(d) x_src + W2 (W^T x_src).
// Runs on the auxiliary warp during phase B, off the critical path.
template <int M>
__device__ void termItem(const PArgs& a, const double2* xc, int p) {
  constexpr int KPL = (M + 31) / 32;
  constexpr int QB = 8;  // projections loaded / reduced per batch
  const int lane = threadIdx.x & 31;
  const int4 info = *reinterpret_cast<const int4*>(a.pInfo + 4 * p);
  const double2* xs = xc + static_cast<long long>(info.y) * M;
  double2 xv[KPL], acc[KPL];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int kk = lane + 32 * k;
    xv[k] = kk < M ? __ldcg(xs + kk) : make_double2(0.0, 0.0);  // L2: x may be this GMRES step's v_j
    acc[k] = make_double2(0.0, 0.0);
  }
  for (int ent = 0; ent < 2; ++ent) {
    const int code = ent == 0 ? info.z : info.w;
    if (code < 0) continue;
    const int slot = code >> 1, trans = code & 1;
    const double2* W = (trans ? a.U : a.V) + static_cast<long long>(slot) * a.rank * M;
    const double2* W2 = (trans ? a.V : a.U) + static_cast<long long>(slot) * a.rank * M;
#pragma unroll
    for (int k = 0; k < KPL; ++k)
      if (lane + 32 * k < M) cfma(acc[k], __ldg(a.D + slot * M + lane + 32 * k), xv[k]);
    for (int q0 = 0; q0 < a.rank; q0 += QB) {
      double2 sq[QB];
#pragma unroll
      for (int q = 0; q < QB; ++q) {
        sq[q] = make_double2(0.0, 0.0);
        if (q0 + q < a.rank) {
#pragma unroll
          for (int k = 0; k < KPL; ++k)
            if (lane + 32 * k < M) cfma(sq[q], __ldg(W + (q0 + q) * M + lane + 32 * k), xv[k]);
        }
      }
#pragma unroll
      for (int q = 0; q < QB; ++q) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) sq[q] = cadd(sq[q], shflXorP(sq[q], off));
      }
#pragma unroll
      for (int q = 0; q < QB; ++q)
        if (q0 + q < a.rank) {
#pragma unroll
          for (int k = 0; k < KPL; ++k)
            if (lane + 32 * k < M) cfma(acc[k], __ldg(W2 + (q0 + q) * M + lane + 32 * k), sq[q]);
        }
    }
  }
#pragma unroll
  for (int k = 0; k < KPL; ++k)
    if (lane + 32 * k < M) a.tvec[static_cast<long long>(p) * M + lane + 32 * k] = acc[k];
}

template <int M>
__device__ void sumTermsItem(const PArgs& a, int ti) {
  constexpr int KPL = (M + 31) / 32;
  constexpr int TMAX = 6;
  const int lane = threadIdx.x & 31;
  const int e = a.targetList[ti];
  const int t0 = a.pTargetPtr[ti], t1 = a.pTargetPtr[ti + 1];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int kk = lane + 32 * k;
    if (kk >= M) continue;
    double2 v[TMAX];
#pragma unroll
    for (int j = 0; j < TMAX; ++j)
      v[j] = (t0 + j < t1) ? __ldcg(a.tvec + static_cast<long long>(t0 + j) * M + kk) : make_double2(0.0, 0.0);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < TMAX; ++j) acc = cadd(acc, v[j]);
    for (int t = t0 + TMAX; t < t1; ++t) acc = cadd(acc, __ldcg(a.tvec + static_cast<long long>(t) * M + kk));
    a.ycorr[static_cast<long long>(e) * M + kk] = acc;
  }
}

template <int M, int TC, int RCH, int STAGES, int N0, int N1, bool LAGGED = false>
struct PCfg {
  static constexpr int TRN = kConsumers / TC;
  static constexpr int CPT = M / TC;
  static constexpr int RPT = RCH / TRN;
  static constexpr int NCH = M / RCH;
  static constexpr uint32_t CHUNK = RCH * M * 16;
  static constexpr uint32_t XF = M * 16;
  static constexpr uint32_t XG = RCH * 16;
  static constexpr uint32_t STAGE = CHUNK + XF + XG;
  static constexpr uint32_t RED = 2 * (kConsumers / 32) * M * 16;
  static constexpr int SLAB0 = WarpFft<N0>::SLAB, SLAB1 = WarpFft<N1>::SLAB;
  static constexpr int SLAB = (SLAB0 > SLAB1 ? SLAB0 : SLAB1) > 1 ? (SLAB0 > SLAB1 ? SLAB0 : SLAB1) : 1;
  static constexpr uint32_t FFTB = (kConsumers / 32) * SLAB * 16;
  // The transpose-product reduction buffer (phase B only) aliases the FFT
  // slabs (phases A / C only): a grid barrier separates every phase.
  static constexpr uint32_t WORK = RED > FFTB ? RED : FFTB;
  // LAGGED launches: the lagged Givens step's staging + the previous
  // column's norm, kept apart from the ring (primed while it runs).
  static constexpr uint32_t GVOFF = STAGES * STAGE + WORK + 2 * STAGES * 8;
  static constexpr uint32_t GVB = LAGGED ? (3 * gmresdev::RMAX + 4 + 1) * 16 : 0;
  static constexpr uint32_t SMEM = GVOFF + GVB;
};

// L2 bulk prefetch of the spectrum chunks after the ring's first `pre`.
template <int M, int RCH>
__device__ __forceinline__ void prefetchL2(const PArgs& a, long long pre, long long total) {
  constexpr int NCH = M / RCH;
  const long long pfEnd = pre + a.l2Chunks < total ? pre + a.l2Chunks : total;
  for (long long it = pre; it < pfEnd; ++it) {
    const long long p = blockIdx.x + (it / NCH) * gridDim.x;
    const int ch = static_cast<int>(it % NCH);
    bulkPrefetchL2(a.S + p * M * M + static_cast<long long>(ch) * RCH * M, RCH * M * 16);
  }
}

// LAGGED: the GMRES-step variant with lagged normalisation, a separate
// instantiation so that its extra state costs the plain apply no registers
// (a first version that looped over a whole restart cycle inside one launch
// spilled in phase B: C2 apply 35.7 -> 40.4 us, GMRES 66 -> 72 us/iteration).
template <int M, int TC, int RCH, int STAGES, int N0, int N1, bool LAGGED>
__global__ void __launch_bounds__(kThreadsP, 1) matvecPersistent(PArgs a) {
  using C = PCfg<M, TC, RCH, STAGES, N0, N1, LAGGED>;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* red = reinterpret_cast<double2*>(smem + STAGES * C::STAGE);
  double2* fftb = red;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE + C::WORK);
  uint64_t* empty = full + STAGES;
  double2* gvSh = reinterpret_cast<double2*>(smem + C::GVOFF);
  double* hnS = reinterpret_cast<double*>(gvSh + 3 * gmresdev::RMAX + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kConsumers / 32;
  const bool aux = warp > kConsumers / 32;
  const int auxId = blockIdx.x * kAux + (warp - kConsumers / 32 - 1);  // valid when aux
  double2* slab = fftb + ((producer || aux) ? 0 : warp) * C::SLAB;
  const int nwarps = gridDim.x * (kConsumers / 32);
  // Global consumer warp id of a transform phase's first item: warp-major
  // (consecutive items on different SMs) when the phase has at most one item
  // per warp, so a short phase spreads over every SM (C2); CTA-major (a
  // CTA's warps on neighbouring lines) when warps loop over several items,
  // and for zero-copy launches, whose PCIe reads prefer that locality.
  auto firstItem = [&](int items) {
    return items <= nwarps && !a.ctaMajor ? warp * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x)
                           : static_cast<int>(blockIdx.x) * (kConsumers / 32) + warp;
  };

  trace(a, 0);
  trace(a, 11);
  if (!LAGGED && a.skip && *reinterpret_cast<const volatile int*>(a.skip)) return;  // uniform: set before launch
  stamp(a, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbarInit(full + s, 1);
      mbarInit(empty + s, kConsumers / 32);
    }
    fenceBarrierInit();
  }
  __syncthreads();

  const long long mine = blockIdx.x < a.npairs ? (a.npairs - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long total = mine * C::NCH;
  const long long pre = total < STAGES ? total : STAGES;
  uint64_t polS = 0, polX = 0;
  // The pi-th bin pair of this CTA (round robin over the grid); reversed,
  // a CTA starts on the pairs it streamed last in the previous apply.
  auto pairAt = [&](long long pi) -> long long {
    return blockIdx.x + (a.rev ? mine - 1 - pi : pi) * gridDim.x;
  };
  auto prefetch = [&]() {
    // Spectrum chunks of the first STAGES items: independent of x.
    for (long long it = 0; it < pre; ++it) {
      const long long p = pairAt(it / C::NCH);
      const int ch = static_cast<int>(it % C::NCH);
      mbarArriveExpectTx(full + it, C::STAGE);
      bulkG2S(smem + it * C::STAGE, a.S + p * M * M + static_cast<long long>(ch) * RCH * M, C::CHUNK, full + it,
              polS);
    }
  };
  if (producer && lane == 0) {
    polS = policyEvictFirst();
    polX = policyEvictLast();
    if (a.prefetchAt == 0) prefetch();
    // Zero-copy applies read x from host memory over PCIe in phase A1 while
    // HBM idles: stream the chunks after the ring's into L2 meanwhile, so
    // phase B starts on L2 hits (l2Chunks is 0 for device-resident x).
    if (a.l2At == 0) prefetchL2<M, RCH>(a, pre, total);
  }
  // Programmatic dependent launch: the CTA started while the previous apply
  // was finishing (its set-up and the spectrum prime above touch nothing the
  // previous grid writes); wait for it before x / T / xhat / y are used.
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  trace(a, 1);

  using W0 = WarpFft<N0>;
  using W1 = WarpFft<N1>;
  const double2 zero = make_double2(0.0, 0.0);
  // Completes the primed ring stages with (unused) x-hat parts and waits
  // for them, so that a CTA leaving before phase B has no copies in flight.
  auto drainPrimed = [&]() {
    if (producer && lane == 0)
      for (long long it = 0; it < pre; ++it) {
        bulkG2S(smem + it * C::STAGE + C::CHUNK, a.xhat, C::XF, full + it, polX);
        bulkG2S(smem + it * C::STAGE + C::CHUNK + C::XF, a.xhat, C::XG, full + it, polX);
      }
    if (threadIdx.x == 0)
      for (long long it = 0; it < pre; ++it) mbarWait(full + it, 0);
    __syncthreads();
  };
  // LAGGED (GMRES column j of a captured restart cycle, the launches
  // serialised programmatically): a node after the cycle's last column
  // returns (its stop flag is final once the previous node has completed).
  // For j >= 1, x = v_j is the previous step's w' (unnormalised): in phase
  // B one auxiliary warp per CTA reduces its norm from the previous step's
  // partials (every CTA gets the same bits) and CTA 0's runs the Givens step
  // of column j-1; if that ended the cycle, the LS step of this node is
  // skipped (its apply ran for nothing, once per cycle). y is scaled by
  // 1/||w'|| in phase C2 and v_j's rows are normalised by the LS step.
  const int jcol = a.gm.j;
  const bool lagStep = LAGGED && jcol > 0;
  if constexpr (LAGGED) {
    const volatile GmresState* st = a.gm.st;
    if (!st->cycleActive || st->stopInner) {  // uniform: the previous node completed
      drainPrimed();
      return;
    }
  }

  // ---- phase A1: row FFTs (level 0)
  if (!producer && !aux) {
    const int chunks0 = M / W0::WB;
    const int rowItems = a.ny * chunks0;
    const int items = rowItems;
    for (int it = firstItem(items); it < items; it += nwarps) {
      if (it < rowItems) {
        const int r = it / chunks0, b0 = (it % chunks0) * W0::WB;
        warpLineFft<N0, false>(
            slab, a.tw0,
            [&](int c, int b) {
              if (c >= a.nx) return zero;
              const long long q = (static_cast<long long>(r) * a.nx + c) * M + b0 + b;
              const double2 v = a.x[q];
              if (a.xStage) a.xStage[q] = v;  // zero-copy: later readers use the HBM copy
              return v;
            },
            [&](int s0, int b, double2 v, int) { a.T[(static_cast<long long>(r) * a.L0 + s0) * M + b0 + b] = v; });
      }
    }
  }
  gridSync(a.barFlags, a, 0);
  stamp(a, 1);

  if (producer && lane == 0 && a.prefetchAt == 1) prefetch();
  if (producer && lane == 0 && a.l2At == 1) prefetchL2<M, RCH>(a, pre, total);
  // ---- phase A2: column FFTs (level 1) -> xhat
  if (!producer && !aux) {
    const int chunks1 = M / W1::WB;
    const int colItems = a.L0 * chunks1;
    const int items = colItems;
    for (int it = firstItem(items); it < items; it += nwarps) {
      const int s0 = it / chunks1, b0 = (it % chunks1) * W1::WB;
      warpLineFft<N1, false>(
          slab, a.tw1,
          [&](int r, int b) { return r < a.ny ? a.T[(static_cast<long long>(r) * a.L0 + s0) * M + b0 + b] : zero; },
          [&](int s1, int b, double2 v, int) { a.xhat[(static_cast<long long>(s1) * a.L0 + s0) * M + b0 + b] = v; });
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  gridSync(a.barFlags, a, 1);
  stamp(a, 2);
  if (producer && lane == 0 && a.prefetchAt == 2) prefetch();

  // ---- phase B: bin-pair products (+ correction term vectors on the aux warp)
  if (aux) {
    // Lagged: the previous column's norm (every CTA) and Givens step (CTA 0)
    // under the spectrum stream, ahead of this warp's correction terms.
    if (lagStep && warp == kConsumers / 32 + 1) {
      const double hn = sqrt(gmresdev::warpTotal(gmresdev::partSlot(a.gm, 0, 0)).x);
      if (lane == 0) *hnS = hn;
      if (blockIdx.x == 0) gmresdev::givensWarp(a.gm, 0, jcol - 1, hn, gvSh);
    }
    if (a.corr)
      for (int p = auxId; p < a.nPairs; p += gridDim.x * kAux) termItem<M>(a, a.xc, p);
  } else if (producer) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for (long long it = 0; it < total; ++it) {
        const int s = static_cast<int>(it % STAGES);
        const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
        const long long p = pairAt(it / C::NCH);
        const int ch = static_cast<int>(it % C::NCH);
        const long long f = a.pairF[p], g = a.pairG[p];
        unsigned char* st = smem + s * C::STAGE;
        if (it >= pre) {
          mbarWait(empty + s, ph ^ 1u);
          mbarArriveExpectTx(full + s, C::STAGE);
          bulkG2S(st, a.S + p * M * M + static_cast<long long>(ch) * RCH * M, C::CHUNK, full + s, polS);
        }
        bulkG2S(st + C::CHUNK, a.xhat + f * M, C::XF, full + s, polX);
        bulkG2S(st + C::CHUNK + C::XF, a.xhat + g * M + ch * RCH, C::XG, full + s, polX);
      }
    }
  } else {
    const int tc = threadIdx.x % TC, tr = threadIdx.x / TC;
    double2 yga[C::CPT];
    for (long long it = 0; it < total; ++it) {
      const int s = static_cast<int>(it % STAGES);
      const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
      const long long pi = it / C::NCH;
      const int ch = static_cast<int>(it % C::NCH);
      const long long p = pairAt(pi);
      if (ch == 0) {
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) yga[j] = zero;
      }
      mbarWait(full + s, ph);
      const double2* A = reinterpret_cast<const double2*>(smem + s * C::STAGE);
      const double2* xf = A + RCH * M;
      const double2* xg = xf + M;
      double2 av[C::RPT][C::CPT], xfr[C::CPT], xgv[C::RPT];
#pragma unroll
      for (int j = 0; j < C::CPT; ++j) xfr[j] = xf[tc + TC * j];
#pragma unroll
      for (int i = 0; i < C::RPT; ++i) {
        xgv[i] = xg[tr + C::TRN * i];
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) av[i][j] = A[(tr + C::TRN * i) * M + tc + TC * j];
      }
      __syncwarp();
      if (lane == 0) mbarArrive(empty + s);
      const long long f = a.pairF[p], g = a.pairG[p];
#pragma unroll
      for (int i = 0; i < C::RPT; ++i) {
        double2 acc = zero;
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) cfma(acc, av[i][j], xfr[j]);
#pragma unroll
        for (int off = TC / 2; off >= 1; off >>= 1) acc = cadd(acc, shflXorP(acc, off));
        if (tc == 0) a.yhat[f * M + ch * RCH + tr + C::TRN * i] = acc;
      }
#pragma unroll
      for (int i = 0; i < C::RPT; ++i)
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) cfma(yga[j], av[i][j], xgv[i]);
      if (ch == C::NCH - 1) {
        if (TC == 16) {
#pragma unroll
          for (int j = 0; j < C::CPT; ++j) yga[j] = cadd(yga[j], shflXorP(yga[j], 16));
        }
        double2* rb = red + (pi & 1) * (kConsumers / 32) * M;
        if (lane < TC) {
#pragma unroll
          for (int j = 0; j < C::CPT; ++j) rb[warp * M + tc + TC * j] = yga[j];
        }
        namedBarrier(1, kConsumers);
        if (f != g) {
          for (int q = threadIdx.x; q < M; q += kConsumers) {
            double2 acc = rb[q];
#pragma unroll
            for (int w = 1; w < kConsumers / 32; ++w) acc = cadd(acc, rb[w * M + q]);
            a.yhat[g * M + q] = acc;
          }
        }
      }
    }
  }
  gridSync(a.barFlags, a, 2);
  stamp(a, 3);


  // ---- phase C1: inverse column FFTs, keep ny rows -> T (+ correction sums on the aux warp)
  if (aux) {
    if (a.corr)
      for (int ti = auxId; ti < a.nTargets; ti += gridDim.x * kAux) sumTermsItem<M>(a, ti);
  } else if (!producer) {
    const int chunks1 = M / W1::WB;
    const int items = a.L0 * chunks1;
    for (int it = firstItem(items); it < items; it += nwarps) {
      const int s0 = it / chunks1, b0 = (it % chunks1) * W1::WB;
      warpLineFft<N1, true>(
          slab, a.tw1, [&](int s1, int b) { return a.yhat[(static_cast<long long>(s1) * a.L0 + s0) * M + b0 + b]; },
          [&](int r, int b, double2 v, int) {
            if (r < a.ny) a.T[(static_cast<long long>(r) * a.L0 + s0) * M + b0 + b] = v;
          });
    }
  }
  gridSync(a.barFlags, a, 3);
  stamp(a, 4);
  // Past the last grid barrier: the next apply may launch its CTAs now.
  if (a.pdl && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- phase C2: inverse row FFTs, keep nx points, scale, correction -> y
  const double hnPrev = lagStep ? *hnS : 1.0;
  const double hnInv = 1.0 / hnPrev;
  if (!producer && !aux) {
    constexpr int RO = Split<N0>::R2 == 1 ? Split<N0>::R1 : Split<N0>::R2;  // outputs per lane
    const int chunks0 = M / W0::WB;
    const int items = a.ny * chunks0;
    const int bl = (threadIdx.x & 31) % W0::WB;
    for (int it = firstItem(items); it < items; it += nwarps) {
      const int r = it / chunks0, b0 = (it % chunks0) * W0::WB;
      double2 pre[RO];
#pragma unroll
      for (int q = 0; q < RO; ++q) {
        const int c = outPoint<N0>(q);
        pre[q] = zero;
        if (a.corr && outActive<N0>() && c < a.nx)  // ycorr is zero off the targets
          pre[q] = __ldcg(a.ycorr + (static_cast<long long>(r) * a.nx + c) * M + b0 + bl);
      }
      warpLineFft<N0, true>(
          slab, a.tw0, [&](int s0, int b) { return a.T[(static_cast<long long>(r) * a.L0 + s0) * M + b0 + b]; },
          [&](int c, int b, double2 v, int q) {
            if (c < a.nx) {
              const long long e = static_cast<long long>(r) * a.nx + c;
              double2 out = cadd(cscale(v, a.scale), pre[q]);
              if (lagStep) out = cscale(out, hnInv);
              a.y[e * M + b0 + b] = out;
            }
          });
    }
  }
  stamp(a, 5);
  if (a.cta) {
    __syncthreads();
    trace(a, 10);
  }
  if (a.arnoldi) {
    gridSync(a.barFlags, a, 4);  // y (= w) complete grid-wide
    trace(a, 12);
    // Shared memory is free again: LS scratch, then hcol / Givens staging.
    const long long chunk = (static_cast<long long>(a.gm.ne) * a.gm.m + gridDim.x - 1) / gridDim.x;
    double2* shw = reinterpret_cast<double2*>(smem);
    double2* tail = shw + gmresdev::arnoldiLSSmem(chunk, a.gm.restart);
    double2* hcol = tail;
    double2* sh = hcol + gmresdev::RMAX + 2;
    double2* scratch = sh + 3 * gmresdev::RMAX + 4;
    __syncthreads();
    gmresdev::arnoldiLS(a.gm, jcol, a.lsS, a.lsDots, a.lsPart, shw, scratch, hcol, sh, a.barFlags, LAGGED,
                        hnPrev, a.cta ? a.cta + 13 * kCtaTraceMaxGrid : nullptr);
    trace(a, 14);
  }
}

template <int M, int TC, int RCH, int STAGES, int N0, int N1, bool LAGGED = false>
bool launchP(Ctx& c, const double2* x, double2* y, bool withCorr, const GmresArgs* gm = nullptr,
             double2* lsS = nullptr, double2* lsDots = nullptr, double2* lsPart = nullptr) {
  using C = PCfg<M, TC, RCH, STAGES, N0, N1, LAGGED>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  auto kern = matvecPersistent<M, TC, RCH, STAGES, N0, N1, LAGGED>;
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [&] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  PArgs a{};
  a.S = c.dSpectra;
  a.pairF = c.dPairF;
  a.pairG = c.dPairG;
  a.npairs = c.npairs;
  a.x = x;
  a.y = y;
  a.xStage = c.zeroCopyStage ? c.dXin : nullptr;
  a.xc = a.xStage ? a.xStage : x;
  a.xhat = c.dXhat;
  a.yhat = c.dYhat;
  a.T = c.dT;
  a.tw0 = c.dTw0;
  a.tw1 = c.dTw1;
  a.nx = c.nx;
  a.ny = c.ny;
  a.L0 = c.L0;
  a.L1 = c.L1;
  a.scale = 1.0 / static_cast<double>(c.L);
  a.bar = c.dGridBar;
  a.barFlags = c.dBarFlags;
  a.corr = (withCorr && c.haveCorr && c.nTerms > 0) ? 1 : 0;
  a.tInfo = c.dTermInfo;
  a.targetList = c.dTargetList;
  a.targetPtr = c.dTargetPtr;
  a.nTargets = c.nTargets;
  a.elemPtr = c.dElemPtr;
  a.D = c.dCorrD;
  a.U = c.dCorrU;
  a.V = c.dCorrV;
  a.rank = c.rank;
  a.nTerms = c.nTerms;
  a.tvec = c.dTermVec;
  a.nPairs = c.nCorrPairs;
  a.pInfo = c.dPairInfo;
  a.pTargetPtr = c.dPairTargetPtr;
  a.ycorr = c.dYcorrP;
  a.phaseNs = c.phaseTiming ? c.dPhaseNs : nullptr;
  a.cta = nullptr;
  if (c.dCtaTrace) {
    a.cta = c.dCtaTrace + (c.ctaTraceLaunches % kCtaTraceSlots) * kCtaTraceEvents * kCtaTraceMaxGrid;
    ++c.ctaTraceLaunches;
  }
  a.prefetchAt = c.prefetchAt;
  a.l2Chunks = c.zeroCopyL2Bytes / (static_cast<long long>(smCount(c.device)) * C::CHUNK);
  a.l2At = 0;
  a.skip = c.skipFlag;
  a.pdl = (c.usePdl && !gm && !c.skipFlag) ? 1 : 0;
  a.ctaMajor = a.xStage ? 1 : 0;  // zero-copy: CTA-major keeps a CTA's host reads together (e2e +2-3 %)
  // Inside a GMRES solve consecutive applies alternate the pair order, so
  // each starts on the spectrum chunks the previous one streamed last (the
  // part still in L2; C2 GMRES 62.0 -> 60.8 us per iteration, DESIGN 4.1).
  // Plain applies keep one order: a benchmark loop of back-to-back applies
  // gains no cache carry-over (it would: C2 36.8 -> 33.6 us). TBT_ZIGZAG=0
  // turns it off in solves too. Only spectra within a few L2 sizes carry
  // anything over (C4's 2.2 GB: 514 vs 521 us, noise), so larger ones keep
  // the address order.
  static const bool zzOff = getenv("TBT_ZIGZAG") && getenv("TBT_ZIGZAG")[0] == '0';
  const bool zzSize = c.npairs * static_cast<long long>(M) * M * 16 <= (512LL << 20);
  a.rev = (c.inSolve && zzSize && !zzOff && !a.xStage) ? static_cast<int>(c.zigzagSeq++ & 1) : 0;
  a.arnoldi = 0;
  if (gm) {
    const long long chunk = (static_cast<long long>(gm->ne) * gm->m + smCount(c.device) - 1) / smCount(c.device);
    const long long need =
        (gmresdev::arnoldiLSSmem(chunk, gm->restart) + gmresdev::RMAX + 2 + 3 * gmresdev::RMAX + 4 + 32) *
        static_cast<long long>(sizeof(double2));
    // The LS scratch reuses the ring and reduction space, never the mbarriers.
    if (need > static_cast<long long>(STAGES * C::STAGE + C::WORK)) return false;
    a.arnoldi = 1;
    if (LAGGED) {
      // Captured restart-cycle nodes, serialised programmatically (the
      // stop flag is read after the programmatic wait).
      a.pdl = c.usePdl ? 1 : 0;
      a.skip = nullptr;
      a.prefetchAt = 0;  // a skipped node drains the primed stages
    }
    a.gm = *gm;
    a.lsS = lsS;
    a.lsDots = lsDots;
    a.lsPart = lsPart;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(smCount(c.device));
  cfg.blockDim = dim3(kThreadsP);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = c.stream;
  // Launch mode. The grid barriers need all CTAs co-resident (one per SM).
  // A cooperative launch guarantees it (or fails), but a cooperative grid is
  // only dispatched once the previous grid has fully drained: measured C2
  // back to back 37.1 us vs 35.7 us for a plain launch with programmatic
  // dependent launch, whose CTAs are placed the moment the previous apply's
  // CTAs exit (its griddepcontrol.wait then covers the rest). So the first
  // apply of a context is launched cooperatively — it fails rather than
  // hangs if this process cannot have one CTA on every SM (e.g. an MPS SM
  // limit) — and later PDL applies launch plainly with the same grid, as
  // long as this is the only live context on the device (plainLaunchOk).
  // TBT_COOP=1 keeps every launch cooperative.
  static const bool forceCoop = getenv("TBT_COOP") && getenv("TBT_COOP")[0] == '1';
  const bool coop = forceCoop || !a.pdl || !c.coopChecked || !plainLaunchOk(c);
  cudaLaunchAttribute at[2];
  int na = 0;
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na++].val.cooperative = 1;
  }
  if (a.pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  TBT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
  if (coop) c.coopChecked = true;
  return true;
}

}  // namespace

bool persistentSupported(const Ctx& c) {
  if (c.hasAntisym || c.fullMode) return false;
  const int key = c.m * 1000000 + c.L0 * 1000 + c.L1;
  switch (key) {
    case 64064064: case 128128128: case 192256256: case 64032032: case 128032016: case 64016032:
    // beyond the BASELINE shapes: other array sizes and basis counts
    case 96128128: case 64128064: case 64064128: case 64128128: case 128064064: case 128256256: case 192128128:
      return true;
    default:
      return false;
  }
}

template <int M, int TC, int RCH, int STAGES, int N0, int N1>
bool laggedFits(const Ctx& c, const GmresArgs& gm) {
  using C = PCfg<M, TC, RCH, STAGES, N0, N1, true>;
  const long long chunk = (static_cast<long long>(gm.ne) * gm.m + smCount(c.device) - 1) / smCount(c.device);
  const long long need =
      (gmresdev::arnoldiLSSmem(chunk, gm.restart) + gmresdev::RMAX + 2 + 3 * gmresdev::RMAX + 4 + 32) *
      static_cast<long long>(sizeof(double2));
  return need <= static_cast<long long>(STAGES * C::STAGE + C::WORK);
}

bool persistentLaggedFits(const Ctx& c, const GmresArgs& gm) {
  if (!persistentSupported(c) || c.dist || gm.ncols != 1) return false;
  switch (c.m * 1000000 + c.L0 * 1000 + c.L1) {
    case 64064064: return laggedFits<64, 16, 32, 4, 64, 64>(c, gm);
    case 64032032: return laggedFits<64, 16, 64, 2, 32, 32>(c, gm);
    case 64016032: return laggedFits<64, 16, 64, 2, 16, 32>(c, gm);
    case 128032016: return laggedFits<128, 32, 16, 4, 32, 16>(c, gm);
    case 64128064: return laggedFits<64, 16, 64, 2, 128, 64>(c, gm);
    case 64064128: return laggedFits<64, 16, 64, 2, 64, 128>(c, gm);
    case 64128128: return laggedFits<64, 16, 64, 2, 128, 128>(c, gm);
    case 128064064: return laggedFits<128, 32, 16, 4, 64, 64>(c, gm);
    default: return false;
  }
}

bool launchPersistentApply(Ctx& c, const double2* x, double2* y, bool withCorr, const GmresArgs* gm,
                           double2* lsS, double2* lsDots, double2* lsPart, bool lagged) {
  if (!persistentSupported(c) || c.dist) return false;
  const int key = c.m * 1000000 + c.L0 * 1000 + c.L1;
  switch (key) {
    // Ring shape: half blocks (32 rows) x 4 stages. Measured (C2 back to
    // back): 37.6 us; whole blocks x 2 38.2, half x 5 40.6, quarter x 8
    // 41.0, quarter x 11 47.1 — more bytes in flight per SM than 128 KB only
    // slows the stream. LAGGED GMRES-step variants exist for the shapes whose
    // LS row chunk can fit next to the ring (<= 2048 rows per CTA).
    case 64064064: return lagged ? launchP<64, 16, 32, 4, 64, 64, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 32, 4, 64, 64>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 64032032: return lagged ? launchP<64, 16, 64, 2, 32, 32, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 64, 2, 32, 32>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 64016032: return lagged ? launchP<64, 16, 64, 2, 16, 32, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 64, 2, 16, 32>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 128128128: return !lagged && launchP<128, 32, 16, 4, 128, 128>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 128032016: return lagged ? launchP<128, 32, 16, 4, 32, 16, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<128, 32, 16, 4, 32, 16>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 192256256: return !lagged && launchP<192, 32, 16, 2, 256, 256>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 96128128: return !lagged && launchP<96, 32, 16, 4, 128, 128>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 64128064: return lagged ? launchP<64, 16, 64, 2, 128, 64, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 64, 2, 128, 64>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 64064128: return lagged ? launchP<64, 16, 64, 2, 64, 128, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 64, 2, 64, 128>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 64128128: return lagged ? launchP<64, 16, 64, 2, 128, 128, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<64, 16, 64, 2, 128, 128>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 128064064: return lagged ? launchP<128, 32, 16, 4, 64, 64, true>(c, x, y, withCorr, gm, lsS, lsDots, lsPart)
                         : launchP<128, 32, 16, 4, 64, 64>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 128256256: return !lagged && launchP<128, 32, 16, 4, 256, 256>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    case 192128128: return !lagged && launchP<192, 32, 16, 2, 128, 128>(c, x, y, withCorr, gm, lsS, lsDots, lsPart);
    default: return false;
  }
}

}  // namespace tbt
