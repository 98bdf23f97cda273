// C ABI (include/tbt.h): context lifecycle, input staging, apply / solve
// entry points. Host-side C++; all arithmetic runs in the kernels of
// fft.cu / spectra.cu / binprod.cu / correction.cu / gmres.cu.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "gmres_dev.cuh"
#include "tbt_internal.cuh"

namespace tbt {


namespace {
thread_local std::string gLastError;
const int kSlotOfComp[10] = {-1, 0, 1, 2, 3, -1, 4, 5, 6, 7};

int componentOf(int nx, int ny, int r, int c) {  // include/tbt_gen.h
  const bool left = c == 0, right = c == nx - 1;
  const bool bottom = r == 0, top = r == ny - 1;
  if (left && bottom) return 1;
  if (left && top) return 3;
  if (right && bottom) return 7;
  if (right && top) return 9;
  if (left) return 2;
  if (right) return 8;
  if (bottom) return 4;
  if (top) return 6;
  return 5;
}

int pow2AtLeast(int n) {  // nextPow2, proj/src/fft.cpp:22-26
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Smallest transform length with a compiled mixed-radix (2^a 3^b) plan.
int smoothAtLeast(int n) {
  static const int kSizes[] = {1, 2, 3, 4, 6, 8, 9, 12, 16, 18, 24, 32, 36, 48, 64, 72, 96, 128, 144, 192, 256};
  for (int s : kSizes)
    if (s >= n) return s;
  return pow2AtLeast(n);
}

template <typename Fn>
tbt_status guarded(Fn&& fn) {
  try {
    fn();
    return TBT_OK;
  } catch (const Error& e) {
    gLastError = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    gLastError = e.what();
    return TBT_CUDA_ERROR;
  }
}

void freePtr(void* p) {
  if (p) cudaFree(p);
}

std::vector<double2> twiddles(int n) {
  std::vector<double2> t(n);
  for (int k = 0; k < n; ++k) {
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * k / n;
    t[k] = make_double2(static_cast<double>(cosl(ang)), static_cast<double>(sinl(ang)));
  }
  return t;
}

// Inverse diagonal on the host (iterativeSolve, linsolve.cpp:556-563).
void refreshDiagonal(Ctx& c, std::vector<double2>* dOut) {
  const int m = c.m;
  std::vector<double2> d(static_cast<size_t>(c.n));
  const double2* z0 = c.genHost.data();  // block (0,0), column-major
  for (int e = 0; e < c.ne; ++e)
    for (int a = 0; a < m; ++a) d[static_cast<size_t>(e) * m + a] = z0[static_cast<size_t>(a) * m + a];
  if (c.haveCorr) {
    // Self relation contributes P + P^T, diagonal 2 (d_a + sum_q U_aq V_aq).
    std::vector<double2> hu(static_cast<size_t>(40) * c.rank * m), hv(hu.size());
    if (c.rank > 0) {
      TBT_CUDA_CHECK(cudaMemcpy(hu.data(), c.dCorrU, hu.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      TBT_CUDA_CHECK(cudaMemcpy(hv.data(), c.dCorrV, hv.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    }
    for (int r = 0; r < c.ny; ++r)
      for (int col = 0; col < c.nx; ++col) {
        const int comp = componentOf(c.nx, c.ny, r, col);
        if (comp == 5) continue;
        const int slot = kSlotOfComp[comp] * 5;
        const int e = r * c.nx + col;
        for (int a = 0; a < m; ++a) {
          double2 p = c.corrDHost[static_cast<size_t>(slot) * m + a];
          for (int q = 0; q < c.rank; ++q) {
            const double2 u = hu[(static_cast<size_t>(slot) * c.rank + q) * m + a];
            const double2 v = hv[(static_cast<size_t>(slot) * c.rank + q) * m + a];
            p = cadd(p, cmul(u, v));
          }
          double2& dd = d[static_cast<size_t>(e) * m + a];
          dd = cadd(dd, make_double2(2.0 * p.x, 2.0 * p.y));
        }
      }
  }
  marginDiagonal(c, d);  // C's diagonal after the element part (linsolve.cpp:400-406)
  if (dOut) {  // tbt_diagonal: read only, the device Jacobi buffers stay as they are
    *dOut = d;
    return;
  }
  auto invert = [](const std::vector<double2>& dv) {
    std::vector<double2> inv(dv.size());
    for (size_t k = 0; k < dv.size(); ++k) {
      const double2 v = dv[k];
      if (std::hypot(v.x, v.y) > 0.0) {
        // 1 / (a + bi) with Smith scaling.
        if (std::fabs(v.x) >= std::fabs(v.y)) {
          const double t = v.y / v.x, den = v.x + v.y * t;
          inv[k] = make_double2(1.0 / den, -t / den);
        } else {
          const double t = v.x / v.y, den = v.x * t + v.y;
          inv[k] = make_double2(t / den, -1.0 / den);
        }
      } else {
        inv[k] = make_double2(1.0, 0.0);
      }
    }
    return inv;
  };
  // Full operator (iterativeSolve) and pure A (schurSolve's inner solves,
  // linsolve.cpp:604-610): A's diagonal is aEntry(0,0,m,m) alone.
  std::vector<double2> dA(static_cast<size_t>(c.n));
  for (int e = 0; e < c.ne; ++e)
    for (int a = 0; a < m; ++a) dA[static_cast<size_t>(e) * m + a] = z0[static_cast<size_t>(a) * m + a];
  auto inv = invert(d);
  const auto invA = invert(dA);
  // Internal length: the margin pseudo-elements' padding gets 1.
  const size_t nInt = static_cast<size_t>(c.ne + c.neM) * m;
  inv.resize(nInt, make_double2(1.0, 0.0));
  if (c.dDiagInv) cudaFree(c.dDiagInv);
  c.dDiagInv = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&c.dDiagInv, nInt * sizeof(double2)));
  if (!c.dDiagInvA) TBT_CUDA_CHECK(cudaMalloc(&c.dDiagInvA, c.n * sizeof(double2)));
  uploadSync(c.dDiagInv, inv.data(), nInt * sizeof(double2), c.stream);
  uploadSync(c.dDiagInvA, invA.data(), c.n * sizeof(double2), c.stream);
}

// Page-locked host memory is device-addressable through UVA.
bool isPinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void requireReady(const Ctx& c) {
  TBT_USER_CHECK(c.havePrecompute, "tbt: call tbt_precompute before apply/solve");
}

// One single-column apply, replayed from the cached CUDA graph unless K3
// timing is on.
void runApply1(Ctx& c, const double2* x, double2* y, bool withCorr) {
  // The loopback transport meets the other ranks on the host: no capture.
  if (c.timeBinprod || (c.dist && c.comm->kind() != 1)) {
    applyInternal(c, x, y, 1, withCorr);
    return;
  }
  if (c.usePdl && !c.zeroCopyStage && !c.dist) {  // direct launch: consecutive applies overlap launch and tail (PDL)
    applyInternal(c, x, y, 1, withCorr);
    return;
  }
  // Sharded over NCCL: the ~12 kernels and three grouped send / receive
  // exchanges of an apply replay as one CUDA graph (NCCL operations are
  // capturable), so small operators are not bound by launch overhead.
  if (c.dist && withCorr && c.haveCorr && c.nTerms > 0) distCorrPrepare(c);
  if (!c.graphExec || c.graphX != x || c.graphY != y || c.graphCorr != withCorr) {
    c.dropGraph();
    cudaGraph_t graph;
    TBT_CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      applyInternal(c, x, y, 1, withCorr);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &graph);
      throw;
    }
    TBT_CUDA_CHECK(cudaStreamEndCapture(c.stream, &graph));
    const cudaError_t e = cudaGraphInstantiate(&c.graphExec, graph, 0);
    cudaGraphDestroy(graph);
    TBT_CUDA_CHECK(e);
    c.graphX = x;
    c.graphY = y;
    c.graphCorr = withCorr;
  }
  TBT_CUDA_CHECK(cudaGraphLaunch(c.graphExec, c.stream));
}

}  // namespace

std::vector<double2> twiddleTable(int n) { return twiddles(n); }

// Host -> device uploads and fills ordered on the context's (non-blocking)
// stream and completed before returning: a plain cudaMemcpy from pageable
// memory may return before its DMA lands, and the legacy stream does not
// order against non-blocking streams.
void uploadSync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  TBT_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
}

void memsetSync(void* dst, int value, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  TBT_CUDA_CHECK(cudaMemsetAsync(dst, value, bytes, s));
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
}

bool stagedE2E() {  // TBT_E2E=staged: pinned host buffers through explicit copies, not zero-copy
  static const bool on = [] {
    const char* e = getenv("TBT_E2E");
    return e && std::string(e) == "staged";
  }();
  return on;
}

bool poisonBuffers() {
  static const bool on = [] {
    const char* e = getenv("TBT_POISON");
    return e && e[0] == '1';
  }();
  return on;
}

int smCount(int device) {
  static std::atomic<int> cached[64] = {};
  if (device >= 0 && device < 64) {
    const int c = cached[device].load(std::memory_order_relaxed);
    if (c) return c;
  }
  int v = 0;
  TBT_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (device >= 0 && device < 64) cached[device].store(v, std::memory_order_relaxed);
  return v;
}

void setError(const std::string& msg) { gLastError = msg; }

// The nine-component correction as terms grouped by target (tbt_gen.h):
// for every element e of a non-interior component and relation rel with an
// in-array neighbour e', y_e += P x_e' and y_e' += P^T x_e.
std::vector<std::vector<std::array<int, 4>>> corrTermsByTarget(int nx, int ny) {
  static const int dr[5] = {0, 0, 0, 1, -1};
  static const int dc[5] = {0, 1, -1, 0, 0};
  std::vector<std::vector<std::array<int, 4>>> byTarget(static_cast<size_t>(nx) * ny);
  for (int r = 0; r < ny; ++r)
    for (int col = 0; col < nx; ++col) {
      const int comp = componentOf(nx, ny, r, col);
      if (comp == 5) continue;
      const int e = r * nx + col;
      for (int rel = 0; rel < 5; ++rel) {
        const int r2 = r + dr[rel], c2 = col + dc[rel];
        if (r2 < 0 || r2 >= ny || c2 < 0 || c2 >= nx) continue;
        const int e2 = r2 * nx + c2;
        const int slot = kSlotOfComp[comp] * 5 + rel;
        byTarget[e].push_back({e, e2, slot, 0});   // y_e  += P   x_e'
        byTarget[e2].push_back({e2, e, slot, 1});  // y_e' += P^T x_e
      }
    }
  return byTarget;
}

namespace {
std::atomic<int> gLiveContexts[64];
}
void liveContextAdd(Ctx& c) {
  if (c.device >= 0 && c.device < 64 && !c.countedLive) {
    gLiveContexts[c.device].fetch_add(1);
    c.countedLive = true;
  }
}
void liveContextRemove(Ctx& c) {
  if (c.countedLive) {
    gLiveContexts[c.device].fetch_sub(1);
    c.countedLive = false;
  }
}
bool plainLaunchOk(const Ctx& c) {
  return c.device >= 0 && c.device < 64 && gLiveContexts[c.device].load() == 1;
}

}  // namespace tbt

using namespace tbt;

struct tbt_ctx {
  Ctx c;
  // One call at a time per context: the reference's apply is re-entrant
  // (per-call scratch, linsolve.cpp:263-265) and is called from parallelFor
  // workers; here the device buffers, stream and graphs are per context, so
  // concurrent callers on one context are serialised (use one context per
  // thread for concurrency).
  std::recursive_mutex mu;
};

namespace {
template <typename Fn>
tbt_status guardedCtx(tbt_ctx* h, Fn&& fn) {
  if (!h) return guarded(fn);  // fn reports the null argument
  std::lock_guard<std::recursive_mutex> lock(h->mu);
  const tbt_status st = guarded(fn);
  // A failed call on one rank of a loopback group must not leave the other
  // ranks waiting at its next exchange.
  if (st != TBT_OK && h->c.comm) h->c.comm->abort();
  return st;
}
}  // namespace

extern "C" {

const char* tbt_last_error(void) { return gLastError.c_str(); }

tbt_status tbt_create(const tbt_desc* desc, tbt_ctx** out) {
  return guarded([&] {
    TBT_USER_CHECK(desc && out, "tbt_create: null argument");
    TBT_USER_CHECK(desc->nx >= 1 && desc->ny >= 1 && desc->m >= 1, "tbt_create: nx, ny, m must be >= 1");
    TBT_USER_CHECK(desc->max_nrhs >= 1, "tbt_create: max_nrhs must be >= 1");
    *out = nullptr;
    int ndev = 0;
    TBT_CUDA_CHECK(cudaGetDeviceCount(&ndev));
    TBT_USER_CHECK(desc->device >= 0 && desc->device < ndev, "tbt_create: no such CUDA device");
    cudaDeviceProp prop;
    TBT_CUDA_CHECK(cudaGetDeviceProperties(&prop, desc->device));
    if (prop.major != 10) throw Error{TBT_CUDA_ERROR, "tbt_create: built for sm_100a (B200), device is sm_" +
                                                          std::to_string(prop.major * 10 + prop.minor)};
    TBT_CUDA_CHECK(cudaSetDevice(desc->device));
    auto* h = new tbt_ctx;
    Ctx& c = h->c;
    c.nx = desc->nx;
    c.ny = desc->ny;
    c.m = desc->m;
    c.ne = c.nx * c.ny;
    c.n = static_cast<long long>(c.ne) * c.m;
    c.maxNrhs = desc->max_nrhs;
    c.device = desc->device;
    // Circulant embedding length per level >= 2n-1: the reference's next
    // power of two (linsolve.cpp:240-242), or with TBT_EMBED_SMOOTH the
    // smallest 3-smooth length (e.g. 36 x 18 instead of 64 x 32 for C3);
    // both embed the same Toeplitz operator exactly.
    const bool smooth = (desc->flags & TBT_EMBED_SMOOTH) != 0;
    c.L1 = smooth ? smoothAtLeast(2 * c.ny - 1) : pow2AtLeast(2 * c.ny - 1);
    c.L0 = smooth ? smoothAtLeast(2 * c.nx - 1) : pow2AtLeast(2 * c.nx - 1);
    c.L = static_cast<long long>(c.L0) * c.L1;
    try {
      TBT_USER_CHECK(c.L0 <= 256 && c.L1 <= 256, "tbt_create: embedding length above 256 (nx, ny <= 128)");
      TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.ownStream = true;
      const long long B = static_cast<long long>(c.maxNrhs) * c.m;
      TBT_CUDA_CHECK(cudaMalloc(&c.dT, static_cast<long long>(c.ny) * c.L0 * B * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dXhat, c.L * B * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dYhat, c.L * B * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dXin, c.ne * B * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dYout, c.ne * B * sizeof(double2)));
      if (poisonBuffers()) {  // TBT_POISON=1: NaN-fill scratch so a read-before-write shows up
        memsetSync(c.dT, 0xFF, static_cast<long long>(c.ny) * c.L0 * B * sizeof(double2), c.stream);
        memsetSync(c.dXhat, 0xFF, c.L * B * sizeof(double2), c.stream);
        memsetSync(c.dYhat, 0xFF, c.L * B * sizeof(double2), c.stream);
        memsetSync(c.dXin, 0xFF, c.ne * B * sizeof(double2), c.stream);
        memsetSync(c.dYout, 0xFF, c.ne * B * sizeof(double2), c.stream);
      }
      const auto t0 = twiddles(c.L0), t1 = twiddles(c.L1);
      TBT_CUDA_CHECK(cudaMalloc(&c.dTw0, c.L0 * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dTw1, c.L1 * sizeof(double2)));
      uploadSync(c.dTw0, t0.data(), c.L0 * sizeof(double2), c.stream);
      uploadSync(c.dTw1, t1.data(), c.L1 * sizeof(double2), c.stream);
      TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
      TBT_CUDA_CHECK(cudaEventCreateWithFlags(&c.evFork, cudaEventDisableTiming));
      TBT_CUDA_CHECK(cudaEventCreateWithFlags(&c.evJoin, cudaEventDisableTiming));
      c.fused2d = fft2dSupported(c.L0, c.L1);
      TBT_CUDA_CHECK(cudaMalloc(&c.dGridBar, 2 * sizeof(unsigned)));
      memsetSync(c.dGridBar, 0, 2 * sizeof(unsigned), c.stream);
      {
        const size_t nfl = (2 * static_cast<size_t>(smCount(c.device)) + 1) * 16;
        TBT_CUDA_CHECK(cudaMalloc(&c.dBarFlags, nfl * sizeof(unsigned long long)));
        memsetSync(c.dBarFlags, 0, nfl * sizeof(unsigned long long), c.stream);
      }
      TBT_CUDA_CHECK(cudaMalloc(&c.dPhaseNs, 32 * sizeof(unsigned long long)));
      memsetSync(c.dPhaseNs, 0, 32 * sizeof(unsigned long long), c.stream);
      if (const char* tenv = getenv("TBT_CTATRACE"); tenv && tenv[0] == '1') {
        const size_t nb = static_cast<size_t>(kCtaTraceSlots) * kCtaTraceEvents * kCtaTraceMaxGrid * 8;
        TBT_CUDA_CHECK(cudaMalloc(&c.dCtaTrace, nb));
        memsetSync(c.dCtaTrace, 0, nb, c.stream);
      }
      const char* aenv = getenv("TBT_APPLY");
      c.persistent = !(aenv && std::string(aenv) == "multi");
      const char* penv = getenv("TBT_PREFETCH");
      if (penv) c.prefetchAt = std::max(0, std::min(2, atoi(penv)));
      const char* fenv = getenv("TBT_FFT");
      c.forceMultiPass = fenv && std::string(fenv) == "passes";
      c.forceFused2d = fenv && std::string(fenv) == "fused";
      const char* genv = getenv("TBT_GMRES");
      c.forceUnfused = genv && std::string(genv) == "unfused";
      c.forceCols = genv && std::string(genv) == "cols";
      const char* pdlEnv = getenv("TBT_PDL");
      c.usePdl = !(pdlEnv && pdlEnv[0] == '0');  // default on; TBT_PDL=0 restores the cached graph
      TBT_CUDA_CHECK(cudaEventCreate(&c.evBinA));
      TBT_CUDA_CHECK(cudaEventCreate(&c.evBinB));
      c.binprodKernel = binprodVariant(c.m);
      // K3 v2 (TMA ring) for single-RHS applies unless TBT_BINPROD=1 asks for v1.
      const char* env = getenv("TBT_BINPROD");
      if (c.binprodKernel > 0 && !(env && env[0] == '1')) c.binprodKernel += 10;
    } catch (...) {
      tbt_destroy(h);
      throw;
    }
    liveContextAdd(h->c);
    *out = h;
  });
}

void tbt_destroy(tbt_ctx* h) {
  if (!h) return;
  Ctx& c = h->c;
  liveContextRemove(c);
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  for (void* p : {static_cast<void*>(c.dSpectra), static_cast<void*>(c.dSpectraAnti), static_cast<void*>(c.dGenAnti),
                  static_cast<void*>(c.dPairF), static_cast<void*>(c.dPairG),
                  static_cast<void*>(c.dAntisym), static_cast<void*>(c.dTw0), static_cast<void*>(c.dTw1),
                  static_cast<void*>(c.dCorrD), static_cast<void*>(c.dCorrU), static_cast<void*>(c.dCorrV),
                  static_cast<void*>(c.dTermInfo), static_cast<void*>(c.dTargetList),
                  static_cast<void*>(c.dTargetPtr), static_cast<void*>(c.dElemPtr), static_cast<void*>(c.dProj), static_cast<void*>(c.dYcorr), static_cast<void*>(c.dYcorrP), static_cast<void*>(c.dTermVec),
                  static_cast<void*>(c.dPairInfo), static_cast<void*>(c.dPairTargetPtr),
                  static_cast<void*>(c.dT),
                  static_cast<void*>(c.dXhat), static_cast<void*>(c.dYhat), static_cast<void*>(c.dXin),
                  static_cast<void*>(c.dYout), static_cast<void*>(c.dDiagInv), static_cast<void*>(c.dDiagInvA),
                  static_cast<void*>(c.dGridBar), static_cast<void*>(c.dPhaseNs), static_cast<void*>(c.dBarFlags),
                  static_cast<void*>(c.dCtaTrace),
                  static_cast<void*>(c.dGen)})
    freePtr(p);
  c.dropGraph();
  distFree(c);
  marginFree(c);
  clusterSmallFree(c);
  freeGmresWorkspace(c);
  for (int k = 0; k < 2; ++k) {
    freePtr(c.dManyX[k]);
    freePtr(c.dManyY[k]);
  }
  for (cudaEvent_t e : c.manyEv)
    if (e) cudaEventDestroy(e);
  if (c.manyIn) cudaStreamDestroy(c.manyIn);
  if (c.manyOut) cudaStreamDestroy(c.manyOut);
  for (auto e : c.tEvA) cudaEventDestroy(e);
  for (auto e : c.tEvB) cudaEventDestroy(e);
  if (c.evBinA) cudaEventDestroy(c.evBinA);
  if (c.evBinB) cudaEventDestroy(c.evBinB);
  if (c.evFork) cudaEventDestroy(c.evFork);
  if (c.evJoin) cudaEventDestroy(c.evJoin);
  if (c.side) cudaStreamDestroy(c.side);
  if (c.ownStream && c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

tbt_status tbt_set_stream(tbt_ctx* h, void* stream) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h, "tbt_set_stream: null context");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (c.ownStream) {
      TBT_CUDA_CHECK(cudaStreamDestroy(c.stream));
      c.ownStream = false;
      c.stream = nullptr;
    }
    if (stream) {
      c.stream = static_cast<cudaStream_t>(stream);
    } else {
      TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.ownStream = true;
    }
  });
}

void* tbt_get_stream(tbt_ctx* h) { return h ? static_cast<void*>(h->c.stream) : nullptr; }

long long tbt_size_a(const tbt_ctx* h) { return h ? h->c.n : 0; }
long long tbt_size_m(const tbt_ctx* h) { return h ? h->c.nM : 0; }

namespace {
// After a margin operator was (re)built: staging vectors that hold the
// padded pseudo-elements, and the Jacobi diagonal.
void marginResized(Ctx& c) {
  const size_t len = static_cast<size_t>(c.ne + c.neM) * c.maxNrhs * c.m;
  freePtr(c.dXin);
  freePtr(c.dYout);
  c.dXin = c.dYout = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&c.dXin, len * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dYout, len * sizeof(double2)));
  if (poisonBuffers()) {
    memsetSync(c.dXin, 0xFF, len * sizeof(double2), c.stream);
    memsetSync(c.dYout, 0xFF, len * sizeof(double2), c.stream);
  }
  if (c.havePrecompute) refreshDiagonal(c, nullptr);
}

long long marginCount(const Ctx& c, const int* e) {
  return static_cast<long long>(c.ny) * (e[1] + e[7]) + static_cast<long long>(c.nx) * (e[5] + e[3]) + e[2] + e[8] +
         e[0] + e[6];
}
}  // namespace

tbt_status tbt_set_margin(tbt_ctx* h, const int* e, const double* bside, const double* brow, const double* bcorner,
                          const double* cmat) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && e, "tbt_set_margin: null argument");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.dropGraph();
    freeGmresWorkspace(c);
    const long long nM = marginCount(c, e);
    TBT_USER_CHECK(nM == 0 || cmat, "tbt_set_margin: C is required when there are margin unknowns");
    TBT_USER_CHECK((e[1] + e[7] == 0 || bside) && (e[5] + e[3] == 0 || brow) &&
                       (e[2] + e[8] + e[0] + e[6] == 0 || bcorner),
                   "tbt_set_margin: missing generator array");
    marginSet(c, e, reinterpret_cast<const double2*>(bside), reinterpret_cast<const double2*>(brow),
              reinterpret_cast<const double2*>(bcorner), reinterpret_cast<const double2*>(cmat));
    marginResized(c);
  });
}

tbt_status tbt_set_margin_dense(tbt_ctx* h, const int* e, const double* bfull, const double* cmat) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && e, "tbt_set_margin_dense: null argument");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.dropGraph();
    freeGmresWorkspace(c);
    const long long nM = marginCount(c, e);
    TBT_USER_CHECK(nM == 0 || (bfull && cmat), "tbt_set_margin_dense: B and C are required when there are margin unknowns");
    marginSetDense(c, e, reinterpret_cast<const double2*>(bfull), reinterpret_cast<const double2*>(cmat));
    marginResized(c);
  });
}
tbt_status tbt_set_generators(tbt_ctx* h, const double* blocks, long long nblocks) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && blocks, "tbt_set_generators: null argument");
    Ctx& c = h->c;
    const long long want = static_cast<long long>(c.nx) * c.ny + static_cast<long long>(c.nx - 1) * (c.ny - 1);
    TBT_USER_CHECK(nblocks == want, "tbt_set_generators: expected " + std::to_string(want) +
                                        " canonical blocks (nx*ny + (nx-1)*(ny-1)), got " +
                                        std::to_string(nblocks));
    // Blocks go straight to the device (freed after tbt_precompute); the host
    // keeps only Z(0,0) for the diagonal and the antisymmetric split, so a
    // 19 GB generator set (C5) is not duplicated in host memory.
    const size_t mm = static_cast<size_t>(c.m) * c.m;
    const size_t cnt = static_cast<size_t>(want) * mm;
    c.genHost.assign(reinterpret_cast<const double2*>(blocks), reinterpret_cast<const double2*>(blocks) + mm);
    if (c.dGen) cudaFree(c.dGen);
    c.dGen = nullptr;
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    TBT_CUDA_CHECK(cudaMalloc(&c.dGen, cnt * sizeof(double2)));
    uploadSync(c.dGen, blocks, cnt * sizeof(double2), c.stream);
    if (c.dGenAnti) cudaFree(c.dGenAnti);
    c.dGenAnti = nullptr;
    c.fullMode = false;
    c.haveGenerators = true;
    c.havePrecompute = false;
  });
}

// FULL generator layout: every shift's block, also for
// non-reciprocal operators the reference's Sparse ToeplitzRep cannot hold
// (toeplitz.hpp:72-74). Split into a reciprocal part, stored and applied
// exactly like tbt_set_generators' (Z_s(s) = (Z(s) + Z(-s)^T)/2, and the
// whole self block Z(0,0), whose antisymmetric part goes to K as usual), and
// an anti-reciprocal part Z_a(s) = (Z(s) - Z(-s)^T)/2 for s != 0, whose
// spectrum obeys Ahat_a(-f) = -Ahat_a(f)^T (second half spectrum, second K3
// pass). Blocks: i = 1-ny .. ny-1 (outer), j = 1-nx .. nx-1, m x m
// column-major.
tbt_status tbt_set_generators_full(tbt_ctx* h, const double* blocks, long long nblocks) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && blocks, "tbt_set_generators_full: null argument");
    Ctx& c = h->c;
    TBT_USER_CHECK(!c.dist, "tbt_set_generators_full: not supported on a distributed context");
    const int nx = c.nx, ny = c.ny, m = c.m;
    const long long want = static_cast<long long>(2 * nx - 1) * (2 * ny - 1);
    TBT_USER_CHECK(nblocks == want, "tbt_set_generators_full: expected " + std::to_string(want) +
                                        " blocks ((2ny-1)*(2nx-1)), got " + std::to_string(nblocks));
    const size_t mm = static_cast<size_t>(m) * m;
    const double2* z = reinterpret_cast<const double2*>(blocks);
    auto full = [&](int i, int j) {  // block of shift (i, j)
      return z + (static_cast<size_t>(i + ny - 1) * (2 * nx - 1) + static_cast<size_t>(j + nx - 1)) * mm;
    };
    const long long ncan = static_cast<long long>(nx) * ny + static_cast<long long>(nx - 1) * (ny - 1);
    std::vector<double2> gs(static_cast<size_t>(ncan) * mm), ga(static_cast<size_t>(ncan) * mm);
    bool anti = false;
    long long t = 0;
    for (int i = 0; i < ny; ++i)
      for (int j = (i == 0 ? 0 : 1 - nx); j <= nx - 1; ++j, ++t) {
        const double2* zp = full(i, j);
        const double2* zn = full(-i, -j);
        for (int b = 0; b < m; ++b)
          for (int a = 0; a < m; ++a) {
            const double2 v = zp[static_cast<size_t>(b) * m + a];   // Z(s)(a, b)
            const double2 w = zn[static_cast<size_t>(a) * m + b];   // Z(-s)(b, a) = Z(-s)^T(a, b)
            const size_t o = static_cast<size_t>(t) * mm + static_cast<size_t>(b) * m + a;
            if (i == 0 && j == 0) {
              gs[o] = v;
              ga[o] = make_double2(0.0, 0.0);
            } else {
              gs[o] = make_double2(0.5 * (v.x + w.x), 0.5 * (v.y + w.y));
              ga[o] = make_double2(0.5 * (v.x - w.x), 0.5 * (v.y - w.y));
              if (ga[o].x != 0.0 || ga[o].y != 0.0) anti = true;
            }
          }
      }
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    c.genHost.assign(gs.begin(), gs.begin() + static_cast<long long>(mm));
    if (c.dGen) cudaFree(c.dGen);
    if (c.dGenAnti) cudaFree(c.dGenAnti);
    c.dGen = c.dGenAnti = nullptr;
    TBT_CUDA_CHECK(cudaMalloc(&c.dGen, gs.size() * sizeof(double2)));
    uploadSync(c.dGen, gs.data(), gs.size() * sizeof(double2), c.stream);
    c.fullMode = anti;
    if (anti) {
      TBT_CUDA_CHECK(cudaMalloc(&c.dGenAnti, ga.size() * sizeof(double2)));
      uploadSync(c.dGenAnti, ga.data(), ga.size() * sizeof(double2), c.stream);
    }
    c.haveGenerators = true;
    c.havePrecompute = false;
  });
}

tbt_status tbt_set_correction(tbt_ctx* h, int rank, const double* d, const double* u, const double* v) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h, "tbt_set_correction: null context");
    Ctx& c = h->c;
    TBT_USER_CHECK(rank >= 0, "tbt_set_correction: rank must be >= 0");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    c.distCorrReady = false;  // a distributed context rebuilds its local term tables
    freePtr(c.dCorrD);
    freePtr(c.dCorrU);
    freePtr(c.dCorrV);
    freePtr(c.dTermInfo);
    freePtr(c.dTargetList);
    freePtr(c.dTargetPtr);
    freePtr(c.dProj);
    freePtr(c.dElemPtr);
    freePtr(c.dYcorr);
    freePtr(c.dYcorrP);
    freePtr(c.dTermVec);
    freePtr(c.dPairInfo);
    freePtr(c.dPairTargetPtr);
    c.dYcorr = nullptr;
    c.dYcorrP = nullptr;
    c.dTermVec = nullptr;
    c.dPairInfo = c.dPairTargetPtr = nullptr;
    c.nCorrPairs = 0;
    c.dCorrD = c.dCorrU = c.dCorrV = c.dProj = nullptr;
    c.dTermInfo = c.dTargetList = c.dTargetPtr = c.dElemPtr = nullptr;
    c.haveCorr = false;
    c.nTerms = c.nTargets = 0;
    c.dropGraph();
    freeGmresWorkspace(c);
    if (d == nullptr) {
      if (c.havePrecompute) refreshDiagonal(c, nullptr);
      return;
    }
    TBT_USER_CHECK(rank == 0 || (u && v), "tbt_set_correction: rank > 0 needs U and V");
    const int m = c.m;
    c.rank = rank;
    c.corrDHost.assign(reinterpret_cast<const double2*>(d), reinterpret_cast<const double2*>(d) + 40 * m);
    TBT_CUDA_CHECK(cudaMalloc(&c.dCorrD, 40 * m * sizeof(double2)));
    uploadSync(c.dCorrD, d, 40 * m * sizeof(double2), c.stream);
    const size_t uvBytes = static_cast<size_t>(40) * std::max(rank, 1) * m * sizeof(double2);
    TBT_CUDA_CHECK(cudaMalloc(&c.dCorrU, uvBytes));
    TBT_CUDA_CHECK(cudaMalloc(&c.dCorrV, uvBytes));
    if (rank > 0) {
      uploadSync(c.dCorrU, u, static_cast<size_t>(40) * rank * m * sizeof(double2), c.stream);
      uploadSync(c.dCorrV, v, static_cast<size_t>(40) * rank * m * sizeof(double2), c.stream);
    }
    // Term list grouped by target element (CSR).
    const auto byTarget = corrTermsByTarget(c.nx, c.ny);
    std::vector<int> info, targets, ptr{0}, eptr{0};
    for (int e = 0; e < c.ne; ++e) {
      eptr.push_back(eptr.back() + static_cast<int>(byTarget[e].size()));
      if (byTarget[e].empty()) continue;
      targets.push_back(e);
      for (auto& t : byTarget[e]) info.insert(info.end(), t.begin(), t.end());
      ptr.push_back(static_cast<int>(info.size() / 4));
    }
    c.nTerms = static_cast<int>(info.size() / 4);
    c.nTargets = static_cast<int>(targets.size());
    c.maxTermsPerTarget = 0;
    for (size_t k = 0; k + 1 < ptr.size(); ++k) c.maxTermsPerTarget = std::max(c.maxTermsPerTarget, ptr[k + 1] - ptr[k]);
    if (c.nTerms > 0) {
      TBT_CUDA_CHECK(cudaMalloc(&c.dTermInfo, info.size() * sizeof(int)));
      // [nTargets] target elements, then [nTargets] target indices by descending
      // term count (the many-column kernels launch their longest CTAs first)
      std::vector<int> order(targets.size());
      for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<int>(k);
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
      targets.insert(targets.end(), order.begin(), order.end());
      TBT_CUDA_CHECK(cudaMalloc(&c.dTargetList, targets.size() * sizeof(int)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dTargetPtr, ptr.size() * sizeof(int)));
      uploadSync(c.dTermInfo, info.data(), info.size() * sizeof(int), c.stream);
      uploadSync(c.dTargetList, targets.data(), targets.size() * sizeof(int), c.stream);
      uploadSync(c.dTargetPtr, ptr.data(), ptr.size() * sizeof(int), c.stream);
      TBT_CUDA_CHECK(cudaMalloc(&c.dElemPtr, eptr.size() * sizeof(int)));
      uploadSync(c.dElemPtr, eptr.data(), eptr.size() * sizeof(int), c.stream);
      TBT_CUDA_CHECK(cudaMalloc(&c.dProj, static_cast<size_t>(c.nTerms) * c.maxNrhs * std::max(rank, 1) *
                                              sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dYcorr, static_cast<size_t>(c.ne) * c.maxNrhs * c.m * sizeof(double2)));
      memsetSync(c.dYcorr, 0, static_cast<size_t>(c.ne) * c.maxNrhs * c.m * sizeof(double2), c.stream);
      TBT_CUDA_CHECK(cudaMalloc(&c.dYcorrP, static_cast<size_t>(c.ne) * c.m * sizeof(double2)));
      memsetSync(c.dYcorrP, 0, static_cast<size_t>(c.ne) * c.m * sizeof(double2), c.stream);
      // (target, source) pairs: terms of one target grouped by source.
      std::vector<int> pinfo, pptr{0};
      for (int e : targets) {
        std::vector<std::array<int, 4>> mine;
        for (auto& t : byTarget[e]) {
          const int code = t[2] * 2 + t[3];
          bool merged = false;
          for (auto& q : mine)
            if (q[1] == t[1] && q[3] < 0) {
              q[3] = code;
              merged = true;
              break;
            }
          if (!merged) mine.push_back({e, t[1], code, -1});
        }
        for (auto& q : mine) pinfo.insert(pinfo.end(), q.begin(), q.end());
        pptr.push_back(static_cast<int>(pinfo.size() / 4));
      }
      c.nCorrPairs = static_cast<int>(pinfo.size() / 4);
      TBT_CUDA_CHECK(cudaMalloc(&c.dPairInfo, pinfo.size() * sizeof(int)));
      TBT_CUDA_CHECK(cudaMalloc(&c.dPairTargetPtr, pptr.size() * sizeof(int)));
      uploadSync(c.dPairInfo, pinfo.data(), pinfo.size() * sizeof(int), c.stream);
      uploadSync(c.dPairTargetPtr, pptr.data(), pptr.size() * sizeof(int), c.stream);
      TBT_CUDA_CHECK(cudaMalloc(&c.dTermVec, static_cast<size_t>(c.nCorrPairs) * c.m * sizeof(double2)));
    }
    c.haveCorr = true;
    if (c.havePrecompute) refreshDiagonal(c, nullptr);
  });
}

tbt_status tbt_precompute(tbt_ctx* h) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h, "tbt_precompute: null context");
    Ctx& c = h->c;
    TBT_USER_CHECK(c.haveGenerators && c.dGen, "tbt_precompute: call tbt_set_generators first");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    c.dropGraph();
    freeGmresWorkspace(c);
    buildSpectra(c);
    refreshDiagonal(c, nullptr);
    cudaFree(c.dGen);
    c.dGen = nullptr;
    if (c.dGenAnti) cudaFree(c.dGenAnti);
    c.dGenAnti = nullptr;
    c.haveGenerators = false;  // a new precompute needs the blocks again
    c.havePrecompute = true;
  });
}

static tbt_status applyCommon(tbt_ctx* h, const double* x, double* y, int nrhs, int where, bool withCorr) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && x && y, "tbt_apply: null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(nrhs >= 1 && nrhs <= c.maxNrhs, "tbt_apply: nrhs outside [1, max_nrhs]");
    TBT_USER_CHECK(where == TBT_HOST || where == TBT_DEVICE, "tbt_apply: bad memory kind");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    const long long nloc = c.dist ? static_cast<long long>(c.myRows) * c.nx * c.m : c.n;
    const long long total = nloc * nrhs;
    const size_t bytes = total * sizeof(double2);
    const double2* xin = reinterpret_cast<const double2*>(x);
    double2* yout = reinterpret_cast<double2*>(y);
    if (withCorr && c.margin) {
      // Full operator with margin parts: vectors of nA + nM rows, internally
      // padded pseudo-elements after the elements (margin.cu).
      const long long nU = c.n + c.nM, nInt = static_cast<long long>(c.ne + c.neM) * c.m;
      const size_t ubytes = static_cast<size_t>(nU) * nrhs * sizeof(double2);
      if (where == TBT_HOST) {
        TBT_CUDA_CHECK(cudaMemcpyAsync(c.dYout, xin, ubytes, cudaMemcpyHostToDevice, c.stream));
        launchLayoutU(c.dYout, c.dXin, nU, nInt, nrhs, true, c.stream, c.m);
      } else {
        launchLayoutU(xin, c.dXin, nU, nInt, nrhs, true, c.stream, c.m);
      }
      applyOperator(c, c.dXin, c.dYout, nrhs, true);
      if (where == TBT_HOST) {
        launchLayoutU(c.dYout, c.dXin, nU, nInt, nrhs, false, c.stream, c.m);
        TBT_CUDA_CHECK(cudaMemcpyAsync(yout, c.dXin, ubytes, cudaMemcpyDeviceToHost, c.stream));
        TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      } else {
        launchLayoutU(c.dYout, yout, nU, nInt, nrhs, false, c.stream, c.m);
      }
      return;
    }
    if (where == TBT_HOST && nrhs == 1 && !c.dist && c.persistent && persistentSupported(c) && !c.timeBinprod &&
        isPinned(xin) && isPinned(yout) && !stagedE2E()) {
      // Zero-copy: the persistent kernel reads x and writes y in pinned host
      // memory over PCIe/C2C itself, overlapping both transfers with the
      // HBM spectrum stream instead of serialising two memcpys around it.
      // Phase A1 is PCIe-bound here: L2-prefetch up to ~3/4 of L2 worth of
      // the spectrum meanwhile (TBT_ZC_L2_MB overrides, 0 disables).
      static const long long zcBytes = [] {
        const char* e = getenv("TBT_ZC_L2_MB");
        return static_cast<long long>(e ? std::max(0, atoi(e)) : 96) << 20;
      }();
      c.zeroCopyL2Bytes = zcBytes;
      c.zeroCopyStage = true;
      try {
        runApply1(c, xin, yout, withCorr);
      } catch (...) {
        c.zeroCopyL2Bytes = 0;
        c.zeroCopyStage = false;
        throw;
      }
      c.zeroCopyL2Bytes = 0;
      c.zeroCopyStage = false;
      TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    } else if (where == TBT_HOST && nrhs > 1 && !c.timeBinprod && [&] {
                 TBT_CUDA_CHECK(cudaMemcpyAsync(c.dYout, xin, bytes, cudaMemcpyHostToDevice, c.stream));
                 return applyUserLayout(c, c.dYout, c.dXin, nrhs, withCorr);
               }()) {
      // Many columns without the layout kernels (transform passes read and
      // write the column-major layout themselves).
      TBT_CUDA_CHECK(cudaMemcpyAsync(yout, c.dXin, bytes, cudaMemcpyDeviceToHost, c.stream));
      TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    } else if (where == TBT_HOST) {
      if (nrhs == 1) {
        TBT_CUDA_CHECK(cudaMemcpyAsync(c.dXin, xin, bytes, cudaMemcpyHostToDevice, c.stream));
      } else {
        TBT_CUDA_CHECK(cudaMemcpyAsync(c.dYout, xin, bytes, cudaMemcpyHostToDevice, c.stream));
        launchLayout(c.dYout, c.dXin, nloc, nrhs, true, c.stream, c.m);
      }
      if (nrhs == 1)
        runApply1(c, c.dXin, c.dYout, withCorr);
      else
        applyInternal(c, c.dXin, c.dYout, nrhs, withCorr);
      if (nrhs == 1) {
        TBT_CUDA_CHECK(cudaMemcpyAsync(yout, c.dYout, bytes, cudaMemcpyDeviceToHost, c.stream));
      } else {
        launchLayout(c.dYout, c.dXin, nloc, nrhs, false, c.stream, c.m);
        TBT_CUDA_CHECK(cudaMemcpyAsync(yout, c.dXin, bytes, cudaMemcpyDeviceToHost, c.stream));
      }
      TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    } else {
      if (nrhs == 1) {
        runApply1(c, xin, yout, withCorr);
      } else if (c.timeBinprod || !applyUserLayout(c, xin, yout, nrhs, withCorr)) {
        launchLayout(xin, c.dXin, nloc, nrhs, true, c.stream, c.m);
        applyInternal(c, c.dXin, c.dYout, nrhs, withCorr);
        launchLayout(c.dYout, yout, nloc, nrhs, false, c.stream, c.m);
      }
    }
  });
}

tbt_status tbt_apply(tbt_ctx* h, const double* x, double* y, int nrhs, int where) {
  return applyCommon(h, x, y, nrhs, where, true);
}

tbt_status tbt_apply_many(tbt_ctx* h, const double* x, double* y, long long count) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && (count == 0 || (x && y)) && count >= 0, "tbt_apply_many: bad argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(!c.dist && !c.margin, "tbt_apply_many: single-GPU operator without margin parts only");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    if (count == 0) return;
    const size_t bytes = static_cast<size_t>(c.n) * sizeof(double2);
    if (!c.manyIn) {
      for (int k = 0; k < 2; ++k) {
        TBT_CUDA_CHECK(cudaMalloc(&c.dManyX[k], bytes));
        TBT_CUDA_CHECK(cudaMalloc(&c.dManyY[k], bytes));
      }
      for (cudaEvent_t& e : c.manyEv) TBT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.manyIn, cudaStreamNonBlocking));
      TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.manyOut, cudaStreamNonBlocking));
    }
    // Everything earlier on the context stream (previous applies that may
    // still read a slot) precedes the first copy.
    TBT_CUDA_CHECK(cudaEventRecord(c.manyEv[2], c.stream));
    TBT_CUDA_CHECK(cudaEventRecord(c.manyEv[3], c.stream));
    TBT_CUDA_CHECK(cudaStreamWaitEvent(c.manyIn, c.manyEv[2], 0));
    const char* xh = reinterpret_cast<const char*>(x);
    char* yh = reinterpret_cast<char*>(y);
    for (long long i = 0; i < count; ++i) {
      const int k = static_cast<int>(i & 1);
      // x_i -> slot k once the apply of i-2 has finished reading it
      if (i >= 2) TBT_CUDA_CHECK(cudaStreamWaitEvent(c.manyIn, c.manyEv[2 + k], 0));
      TBT_CUDA_CHECK(cudaMemcpyAsync(c.dManyX[k], xh + i * bytes, bytes, cudaMemcpyHostToDevice, c.manyIn));
      TBT_CUDA_CHECK(cudaEventRecord(c.manyEv[k], c.manyIn));
      // apply i once x_i landed and y slot k was read back (i-2)
      TBT_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.manyEv[k], 0));
      if (i >= 2) TBT_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.manyEv[4 + k], 0));
      runApply1(c, c.dManyX[k], c.dManyY[k], true);
      TBT_CUDA_CHECK(cudaEventRecord(c.manyEv[2 + k], c.stream));
      // y_i back to the host on the outbound copy engine
      TBT_CUDA_CHECK(cudaStreamWaitEvent(c.manyOut, c.manyEv[2 + k], 0));
      TBT_CUDA_CHECK(cudaMemcpyAsync(yh + i * bytes, c.dManyY[k], bytes, cudaMemcpyDeviceToHost, c.manyOut));
      TBT_CUDA_CHECK(cudaEventRecord(c.manyEv[4 + k], c.manyOut));
    }
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.manyOut));
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

tbt_status tbt_apply_a(tbt_ctx* h, const double* x, double* y, int nrhs, int where) {
  return applyCommon(h, x, y, nrhs, where, false);
}

// One margin block: the input is embedded in a full [xA; xM] vector with the
// other part zero and only the margin products run (marginApply on a zero
// y): y = [B^T xM ; B xA + C xM], from which the requested part is read.
//   part 0: B (xA -> yM), 1: B^T (xM -> yA), 2: C (xM -> yM)
static tbt_status applyMarginPart(tbt_ctx* h, const double* x, double* y, int nrhs, int where, int part) {
  static const char* names[3] = {"tbt_apply_b", "tbt_apply_bt", "tbt_apply_c"};
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && x && y, std::string(names[part]) + ": null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(c.margin && c.nM > 0, std::string(names[part]) + ": no margin parts (tbt_set_margin)");
    TBT_USER_CHECK(nrhs >= 1 && nrhs <= c.maxNrhs, std::string(names[part]) + ": nrhs outside [1, max_nrhs]");
    TBT_USER_CHECK(where == TBT_HOST || where == TBT_DEVICE, std::string(names[part]) + ": bad memory kind");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    const long long nA = c.n, nM = c.nM, nU = nA + nM, nInt = static_cast<long long>(c.ne + c.neM) * c.m;
    const long long inOff = part == 0 ? 0 : nA, inRows = part == 0 ? nA : nM;
    const long long outOff = part == 1 ? 0 : nA, outRows = part == 1 ? nA : nM;
    const cudaMemcpyKind in = where == TBT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind out = where == TBT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    cudaStream_t s = c.stream;
    // [xA; xM] user layout (nU rows per column) in dYout, then internal in dXin.
    TBT_CUDA_CHECK(cudaMemsetAsync(c.dYout, 0, static_cast<size_t>(nU) * nrhs * sizeof(double2), s));
    TBT_CUDA_CHECK(cudaMemcpy2DAsync(c.dYout + inOff, nU * sizeof(double2), x, inRows * sizeof(double2),
                                     inRows * sizeof(double2), nrhs, in, s));
    launchLayoutU(c.dYout, c.dXin, nU, nInt, nrhs, true, s, c.m);
    TBT_CUDA_CHECK(cudaMemsetAsync(c.dYout, 0, static_cast<size_t>(nInt) * nrhs * sizeof(double2), s));
    marginApply(c, c.dXin, c.dYout, nrhs);
    launchLayoutU(c.dYout, c.dXin, nU, nInt, nrhs, false, s, c.m);
    TBT_CUDA_CHECK(cudaMemcpy2DAsync(y, outRows * sizeof(double2), c.dXin + outOff, nU * sizeof(double2),
                                     outRows * sizeof(double2), nrhs, out, s));
    if (where == TBT_HOST) TBT_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

tbt_status tbt_apply_b(tbt_ctx* h, const double* x, double* y, int nrhs, int where) {
  return applyMarginPart(h, x, y, nrhs, where, 0);
}
tbt_status tbt_apply_bt(tbt_ctx* h, const double* x, double* y, int nrhs, int where) {
  return applyMarginPart(h, x, y, nrhs, where, 1);
}
tbt_status tbt_apply_c(tbt_ctx* h, const double* x, double* y, int nrhs, int where) {
  return applyMarginPart(h, x, y, nrhs, where, 2);
}

tbt_status tbt_diagonal(tbt_ctx* h, double* d) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && d, "tbt_diagonal: null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    std::vector<double2> dd;
    refreshDiagonal(c, &dd);
    const size_t first = c.dist ? static_cast<size_t>(c.myRow0) * c.nx * c.m : 0;
    const size_t count = c.dist ? static_cast<size_t>(c.myRows) * c.nx * c.m : dd.size();
    std::memcpy(d, dd.data() + first, count * sizeof(double2));
  });
}

tbt_status tbt_gmres(tbt_ctx* h, const double* b, double* x, int nrhs, const tbt_gmres_opts* opts,
                     tbt_gmres_stats* stats, int where) {
  std::string failure;
  tbt_status st = guardedCtx(h, [&] {
    TBT_USER_CHECK(h && b && x && opts, "tbt_gmres: null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(nrhs >= 1 && nrhs <= c.maxNrhs, "tbt_gmres: nrhs outside [1, max_nrhs]");
    TBT_USER_CHECK(opts->restart >= 1 && opts->max_iter >= 0 && opts->tol > 0.0, "tbt_gmres: bad options");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    // Multi-GPU: b and x are this rank's element-row slab (tbt_dist_rows).
    // Margin parts (full operator): nA + nM user rows, padded internally.
    const bool withMargin = c.margin && !opts->use_a_only;
    const long long nUser = c.dist ? static_cast<long long>(c.myRows) * c.nx * c.m : c.n + (withMargin ? c.nM : 0);
    const long long nloc = withMargin ? static_cast<long long>(c.ne + c.neM) * c.m : nUser;
    const long long total = nloc * nrhs;
    const size_t bytes = static_cast<size_t>(nUser) * nrhs * sizeof(double2);
    GmresWs* W = gmresWorkspace(c);
    if (W->bufLen < total) {
      if (W->bufB) cudaFree(W->bufB);
      if (W->bufX) cudaFree(W->bufX);
      W->bufB = W->bufX = nullptr;
      W->bufLen = 0;
      TBT_CUDA_CHECK(cudaMalloc(&W->bufB, total * sizeof(double2)));
      TBT_CUDA_CHECK(cudaMalloc(&W->bufX, total * sizeof(double2)));
      W->bufLen = total;
    }
    double2* db = W->bufB;
    double2* dx = W->bufX;
    std::vector<GmresState> out;
    std::vector<double> hist;
    int matvecs = 0;
    const double2* bsrc = reinterpret_cast<const double2*>(b);
    if (where == TBT_HOST) {
      TBT_CUDA_CHECK(cudaMemcpyAsync(dx, bsrc, bytes, cudaMemcpyHostToDevice, c.stream));
      launchLayoutU(dx, db, nUser, nloc, nrhs, true, c.stream, c.m);
    } else {
      launchLayoutU(bsrc, db, nUser, nloc, nrhs, true, c.stream, c.m);
    }
    gmresSolve(c, db, dx, nrhs, *opts, opts->use_a_only != 0, out, hist, matvecs);
    double2* xdst = reinterpret_cast<double2*>(x);
    if (where == TBT_HOST) {
      launchLayoutU(dx, db, nUser, nloc, nrhs, false, c.stream, c.m);
      TBT_CUDA_CHECK(cudaMemcpyAsync(xdst, db, bytes, cudaMemcpyDeviceToHost, c.stream));
    } else {
      launchLayoutU(dx, xdst, nUser, nloc, nrhs, false, c.stream, c.m);
    }
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (stats) {
      const int cap = std::max(0, opts->hist_cap);
      for (int k = 0; k < nrhs; ++k) {
        if (stats->iterations) stats->iterations[k] = out[k].iterations;
        if (stats->residual) stats->residual[k] = out[k].residual;
        if (stats->converged) stats->converged[k] = out[k].converged;
        if (stats->history_len) stats->history_len[k] = out[k].histLen;
        if (stats->history && cap > 0)
          std::memcpy(stats->history + static_cast<size_t>(2) * cap * k, hist.data() + static_cast<size_t>(2) * cap * k,
                      sizeof(double) * 2 * cap);
      }
      stats->matvecs = matvecs;
    }
    for (int k = 0; k < nrhs; ++k)
      if (!out[k].converged && failure.empty())
        failure = "gmres did not converge for column " + std::to_string(k) + ": best residual " +
                  std::to_string(out[k].residual) + " after " + std::to_string(out[k].iterations) + " iterations";
  });
  if (st == TBT_OK && !failure.empty()) {
    gLastError = failure;
    return TBT_NUMERIC_ERROR;
  }
  return st;
}

tbt_status tbt_schur_solve(tbt_ctx* h, const double* b, double* x, int nrhs, const tbt_gmres_opts* opts,
                           tbt_gmres_stats* stats, int where) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && b && x && opts, "tbt_schur_solve: null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(!c.dist, "tbt_schur_solve: not available on a distributed context");
    TBT_USER_CHECK(nrhs >= 1, "tbt_schur_solve: nrhs must be >= 1");
    TBT_USER_CHECK(opts->restart >= 1 && opts->max_iter >= 0 && opts->tol > 0.0, "tbt_schur_solve: bad options");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    const long long ntot = c.n + c.nM;
    const size_t bytes = static_cast<size_t>(ntot) * nrhs * sizeof(double2);
    double2* db = nullptr;
    double2* dx = nullptr;
    struct Free {
      double2** a;
      double2** b;
      ~Free() {
        if (*a) cudaFree(*a);
        if (*b) cudaFree(*b);
      }
    } fr{&db, &dx};
    TBT_CUDA_CHECK(cudaMalloc(&db, bytes));
    TBT_CUDA_CHECK(cudaMalloc(&dx, bytes));
    TBT_CUDA_CHECK(cudaMemcpyAsync(db, b, bytes, where == TBT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                   c.stream));
    std::vector<int> its;
    std::vector<double> res;
    schurSolve(c, db, dx, nrhs, *opts, its, res);
    TBT_CUDA_CHECK(cudaMemcpyAsync(x, dx, bytes, where == TBT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                   c.stream));
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (stats) {
      for (int k = 0; k < nrhs; ++k) {
        if (stats->iterations) stats->iterations[k] = its[k];
        if (stats->residual) stats->residual[k] = res[k];
        if (stats->converged) stats->converged[k] = 1;
        if (stats->history_len) stats->history_len[k] = 0;
      }
      stats->matvecs = 0;
    }
  });
}

tbt_status tbt_load_ztoe1(const char* path, int max_nrhs, int device, int flags, tbt_ctx** out) {
  return guarded([&] {
    TBT_USER_CHECK(path && out, "tbt_load_ztoe1: null argument");
    *out = nullptr;
    Ztoe1Data z;
    readZtoe1(path, z);
    tbt_desc d{z.nx, z.ny, z.e[4], max_nrhs, device, flags};
    tbt_ctx* h = nullptr;
    const tbt_status st = tbt_create(&d, &h);
    if (st != TBT_OK) throw Error{st, gLastError};
    try {
      auto chk = [](tbt_status s2) {
        if (s2 != TBT_OK) throw Error{s2, gLastError};
      };
      chk(tbt_set_generators(h, reinterpret_cast<const double*>(z.gen.data()),
                             static_cast<long long>(z.gen.size() / (static_cast<size_t>(z.e[4]) * z.e[4]))));
      if (z.nM > 0 && z.mode == 1)
        chk(tbt_set_margin_dense(h, z.e, reinterpret_cast<const double*>(z.bfull.data()),
                                 reinterpret_cast<const double*>(z.c.data())));
      else if (z.nM > 0)
        chk(tbt_set_margin(h, z.e, reinterpret_cast<const double*>(z.bside.data()),
                           reinterpret_cast<const double*>(z.brow.data()),
                           reinterpret_cast<const double*>(z.bcorner.data()),
                           reinterpret_cast<const double*>(z.c.data())));
      chk(tbt_precompute(h));
    } catch (...) {
      tbt_destroy(h);
      throw;
    }
    *out = h;
  });
}

tbt_status tbt_ztoe1_dims(const char* path, int* nx, int* ny, int* e) {
  return guarded([&] {
    TBT_USER_CHECK(path && nx && ny && e, "tbt_ztoe1_dims: null argument");
    std::ifstream in(path, std::ios::binary);
    TBT_USER_CHECK(static_cast<bool>(in), std::string("cannot open block cache: ") + path);
    char head[5 + 1 + 4 * 11];
    in.read(head, sizeof head);
    TBT_USER_CHECK(in && std::string(head, 5) == "ZTOE1", std::string("not a ZTOE1 block cache: ") + path);
    std::memcpy(nx, head + 6, 4);
    std::memcpy(ny, head + 10, 4);
    std::memcpy(e, head + 14, 36);
  });
}

tbt_status tbt_ztoe1_read(const char* path, double* gen, double* bside, double* brow, double* bcorner, double* cm) {
  return guarded([&] {
    TBT_USER_CHECK(path, "tbt_ztoe1_read: null path");
    Ztoe1Data z;
    readZtoe1(path, z);
    auto put = [](double* dst, const std::vector<double2>& src) {
      if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double2));
    };
    put(gen, z.gen);
    put(bside, z.bside);
    put(brow, z.brow);
    put(bcorner, z.bcorner);
    put(cm, z.c);
  });
}

tbt_status tbt_ztoe1_mode(const char* path, int* mode) {
  return guarded([&] {
    TBT_USER_CHECK(path && mode, "tbt_ztoe1_mode: null argument");
    std::ifstream in(path, std::ios::binary);
    TBT_USER_CHECK(static_cast<bool>(in), std::string("cannot open block cache: ") + path);
    char head[6];
    in.read(head, 6);
    TBT_USER_CHECK(in && std::string(head, 5) == "ZTOE1", std::string("not a ZTOE1 block cache: ") + path);
    *mode = static_cast<unsigned char>(head[5]);
  });
}

tbt_status tbt_ztoe1_read_dense(const char* path, double* gen, double* bfull, double* cm) {
  return guarded([&] {
    TBT_USER_CHECK(path, "tbt_ztoe1_read_dense: null path");
    Ztoe1Data z;
    readZtoe1(path, z);
    TBT_USER_CHECK(z.mode == 1, "tbt_ztoe1_read_dense: not a SemiSparse cache");
    auto put = [](double* dst, const std::vector<double2>& src) {
      if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double2));
    };
    put(gen, z.gen);
    put(bfull, z.bfull);
    put(cm, z.c);
  });
}

tbt_status tbt_set_cache_key(tbt_ctx* h, const unsigned char* key, int len) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && (key || len == 0) && len >= 0 && len <= 32, "tbt_set_cache_key: bad arguments");
    Ctx& c = h->c;
    std::memset(c.cacheKey, 0, sizeof c.cacheKey);
    if (len > 0) std::memcpy(c.cacheKey, key, static_cast<size_t>(len));
    c.haveCacheKey = len > 0;
  });
}

tbt_status tbt_save_spectra(tbt_ctx* h, const char* path) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && path, "tbt_save_spectra: null argument");
    TBT_CUDA_CHECK(cudaSetDevice(h->c.device));
    saveSpectra(h->c, path);
  });
}

tbt_status tbt_load_spectra(tbt_ctx* h, const char* path) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && path, "tbt_load_spectra: null argument");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    c.dropGraph();
    freeGmresWorkspace(c);
    loadSpectra(c, path);
    if (c.dGen) {
      cudaFree(c.dGen);
      c.dGen = nullptr;
    }
    c.haveGenerators = false;
    c.havePrecompute = true;
    refreshDiagonal(c, nullptr);
  });
}

namespace {
// Device copy of a host (or device) input; owns the allocation when copied.
struct In {
  const void* dev = nullptr;
  void* own = nullptr;
  In(const void* src, size_t bytes, int where, cudaStream_t s) {
    if (!src || bytes == 0) return;
    if (where == TBT_DEVICE) {
      dev = src;
      return;
    }
    TBT_CUDA_CHECK(cudaMalloc(&own, bytes));
    uploadSync(own, src, bytes, s);
    dev = own;
  }
  ~In() {
    if (own) cudaFree(own);
  }
};
struct Out {
  void* dev = nullptr;
  void* own = nullptr;
  void* host = nullptr;
  size_t bytes = 0;
  Out(void* dst, size_t b, int where) : bytes(b) {
    if (!dst) return;
    if (where == TBT_DEVICE) {
      dev = dst;
      return;
    }
    TBT_CUDA_CHECK(cudaMalloc(&own, std::max<size_t>(b, 16)));
    dev = own;
    host = dst;
  }
  void fetch(cudaStream_t s) {
    if (host) TBT_CUDA_CHECK(cudaMemcpyAsync(host, own, bytes, cudaMemcpyDeviceToHost, s));
  }
  ~Out() {
    if (own) cudaFree(own);
  }
};
}  // namespace

tbt_status tbt_port_network(tbt_ctx* h, const double* current, long long ld, int p, const long long* feed_rows,
                            double edge_len, const double* z0, double* y, double* z, double* s, int where) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && current && feed_rows && z0 && y && z && s, "tbt_port_network: null argument");
    Ctx& c = h->c;
    TBT_USER_CHECK(p >= 1 && ld >= 1, "tbt_port_network: bad sizes");
    TBT_USER_CHECK(edge_len > 0.0, "portNetwork: feed edge length must be positive");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    std::vector<double> z0h(p);
    std::vector<long long> fh(p);
    if (where == TBT_HOST) {
      std::memcpy(z0h.data(), z0, p * sizeof(double));
      std::memcpy(fh.data(), feed_rows, p * sizeof(long long));
    } else {
      TBT_CUDA_CHECK(cudaMemcpy(z0h.data(), z0, p * sizeof(double), cudaMemcpyDeviceToHost));
      TBT_CUDA_CHECK(cudaMemcpy(fh.data(), feed_rows, p * sizeof(long long), cudaMemcpyDeviceToHost));
    }
    for (int i = 0; i < p; ++i) {  // postproc.cpp:191-193
      TBT_USER_CHECK(z0h[i] > 0.0, "portNetwork: reference impedances must be positive");
      TBT_USER_CHECK(fh[i] >= 0 && fh[i] < ld, "portNetwork: feed row outside the current vector");
    }
    cudaStream_t st = c.stream;
    // Host input: only the p port rows travel (ExcitationSet::feedRows).
    std::vector<double2> rows;
    long long ldUse = ld;
    if (where == TBT_HOST) {
      rows.resize(static_cast<size_t>(p) * p);
      const double2* cur = reinterpret_cast<const double2*>(current);
      for (int col = 0; col < p; ++col)
        for (int i = 0; i < p; ++i) rows[static_cast<size_t>(col) * p + i] = cur[fh[i] + col * ld];
      for (int i = 0; i < p; ++i) fh[i] = i;
      ldUse = p;
    }
    In dCur(where == TBT_HOST ? static_cast<const void*>(rows.data()) : current,
            static_cast<size_t>(ldUse) * p * sizeof(double2), TBT_HOST == where ? TBT_HOST : where, st);
    In dFeed(fh.data(), p * sizeof(long long), TBT_HOST, st);
    In dZ0(z0h.data(), p * sizeof(double), TBT_HOST, st);
    const size_t pp = static_cast<size_t>(p) * p * sizeof(double2);
    Out oy(y, pp, where), oz(z, pp, where), os(s, pp, where);
    portNetwork(c, static_cast<const double2*>(dCur.dev), ldUse, p, static_cast<const long long*>(dFeed.dev), edge_len,
                static_cast<const double*>(dZ0.dev), static_cast<double2*>(oy.dev), static_cast<double2*>(oz.dev),
                static_cast<double2*>(os.dev));
    oy.fetch(st);
    oz.fetch(st);
    os.fetch(st);
    TBT_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

tbt_status tbt_array_farfield(tbt_ctx* h, const double* const* tensors_co, const double* const* tensors_cx,
                              const int* e, int ndir, const double* dirs, double dx, double dy, double k, double eta,
                              const double* current, int p, const double* weights, int q, double* co, double* cx,
                              int where) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && tensors_co && tensors_cx && e && dirs && current && weights && co && cx,
                   "tbt_array_farfield: null argument");
    Ctx& c = h->c;
    TBT_USER_CHECK(ndir >= 1 && p >= 1 && q >= 1, "tbt_array_farfield: bad sizes");
    TBT_USER_CHECK(e[4] == c.m, "arrayFarfield: e[4] must equal the element basis size");
    TBT_CUDA_CHECK(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    const long long ntot = static_cast<long long>(c.nx) * c.ny * e[4] +
                           static_cast<long long>(c.ny) * (e[1] + e[7]) + static_cast<long long>(c.nx) * (e[5] + e[3]) +
                           e[2] + e[8] + e[0] + e[6];
    std::vector<std::unique_ptr<In>> keep;
    const double2* tco[9];
    const double2* tcx[9];
    for (int i = 0; i < 9; ++i) {
      TBT_USER_CHECK(e[i] == 0 || (tensors_co[i] && tensors_cx[i]), "arrayFarfield: missing component tensor");
      const size_t b = static_cast<size_t>(ndir) * e[i] * sizeof(double2);
      keep.emplace_back(new In(tensors_co[i], b, where, st));
      tco[i] = static_cast<const double2*>(keep.back()->dev);
      keep.emplace_back(new In(tensors_cx[i], b, where, st));
      tcx[i] = static_cast<const double2*>(keep.back()->dev);
    }
    In dDirs(dirs, static_cast<size_t>(ndir) * 3 * sizeof(double), where, st);
    In dCur(current, static_cast<size_t>(ntot) * p * sizeof(double2), where, st);
    In dW(weights, static_cast<size_t>(p) * q * sizeof(double2), where, st);
    const size_t ob = static_cast<size_t>(ndir) * q * sizeof(double2);
    Out oco(co, ob, where), ocx(cx, ob, where);
    arrayFarfield(c, tco, tcx, e, ndir, static_cast<const double*>(dDirs.dev), dx, dy, k, eta,
                  static_cast<const double2*>(dCur.dev), ntot, p, static_cast<const double2*>(dW.dev), q,
                  static_cast<double2*>(oco.dev), static_cast<double2*>(ocx.dev));
    oco.fetch(st);
    ocx.fetch(st);
    TBT_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

tbt_status tbt_get_info(const tbt_ctx* h, tbt_info* info) {
  return guarded([&] {
    TBT_USER_CHECK(h && info, "tbt_get_info: null argument");
    const Ctx& c = h->c;
    info->n = c.n;
    info->bins = c.L;
    info->pairs = c.npairs;
    info->L0 = c.L0;
    info->L1 = c.L1;
    info->spectra_bytes = c.npairs * static_cast<long long>(c.m) * c.m * 16;
    info->binprod_kernel = c.binprodKernel;
    const bool pers = !c.dist && c.persistent && persistentSupported(c);
    const bool fused = !pers && c.fused2d && !c.forceMultiPass;
    info->kernels_per_apply = pers ? 1
                              : fused ? 3 + (c.hasAntisym ? 1 : 0) + (c.haveCorr ? 1 : 0)
                                      : 5 + (c.hasAntisym ? 1 : 0) + (c.haveCorr ? (c.rank > 0 ? 2 : 1) : 0);
    info->apply_path = c.dist ? 3 : (pers ? 2 : (fused ? 1 : 0));
    info->has_antisym = c.hasAntisym ? 1 : 0;
  });
}

tbt_status tbt_get_spectrum_bin(tbt_ctx* h, long long f, double* out) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && out, "tbt_get_spectrum_bin: null argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(f >= 0 && f < c.L, "tbt_get_spectrum_bin: bin out of range");
    const long long code = c.pairOfBin[f];
    const long long p = code >= 0 ? code : -code - 1;
    const size_t mm = static_cast<size_t>(c.m) * c.m;
    std::vector<double2> blk(mm);
    TBT_CUDA_CHECK(cudaMemcpy(blk.data(), c.dSpectra + p * mm, mm * sizeof(double2), cudaMemcpyDeviceToHost));
    double2* o = reinterpret_cast<double2*>(out);
    for (int a = 0; a < c.m; ++a)
      for (int b = 0; b < c.m; ++b)
        o[static_cast<size_t>(a) * c.m + b] = code >= 0 ? blk[static_cast<size_t>(a) * c.m + b]
                                                        : blk[static_cast<size_t>(b) * c.m + a];
  });
}

tbt_status tbt_set_timing(tbt_ctx* h, int on) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h, "tbt_set_timing: null context");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.timeBinprod = on != 0;
    c.tCount = 0;
  });
}

tbt_status tbt_timing_read(tbt_ctx* h, double* total, int* count) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && total && count, "tbt_timing_read: null argument");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    double sum = 0.0;
    for (int k = 0; k < c.tCount; ++k) {
      float ms = 0.f;
      TBT_CUDA_CHECK(cudaEventElapsedTime(&ms, c.tEvA[k], c.tEvB[k]));
      sum += ms;
    }
    *total = sum;
    *count = c.tCount;
  });
}

tbt_status tbt_dist_unique_id(char* id) {
  return guarded([&] {
    TBT_USER_CHECK(id, "tbt_dist_unique_id: null argument");
    ncclUniqueId u;
    const ncclResult_t r = nccl().getUniqueId(&u);
    if (r != ncclSuccess) throw Error{TBT_CUDA_ERROR, std::string("ncclGetUniqueId: ") + nccl().errorString(r)};
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

tbt_status tbt_dist_plan(int ny, int L0, int nranks, int rank, int* row_begin, int* row_end, int* ncols,
                         int* cols) {
  return guarded([&] {
    TBT_USER_CHECK(nranks >= 1 && rank >= 0 && rank < nranks && ny >= 1 && L0 >= 1, "tbt_dist_plan: bad arguments");
    TBT_USER_CHECK(nranks <= ny && nranks <= L0, "tbt_dist_plan: more ranks than element rows or level-0 bins");
    std::vector<int> rs;
    std::vector<std::vector<int>> cl;
    distPlan(ny, L0, nranks, rs, cl);
    if (row_begin) *row_begin = rs[rank];
    if (row_end) *row_end = rs[rank + 1];
    if (ncols) *ncols = static_cast<int>(cl[rank].size());
    if (cols) std::copy(cl[rank].begin(), cl[rank].end(), cols);
  });
}

namespace {
// Shared by both transports: the partition (dist.cu distPlan), the
// exchange buffers and the communicator of this rank.
void distInit(tbt_ctx* h, int nranks, int rank, const char* id, bool loopback) {
  TBT_USER_CHECK(h && id, "tbt_dist_init: null argument");
  Ctx& c = h->c;
  TBT_USER_CHECK(!c.havePrecompute, "tbt_dist_init: call before tbt_precompute");
  TBT_USER_CHECK(!c.margin, "tbt_dist_init: margin parts are not supported on a distributed context");
  TBT_USER_CHECK(!c.fullMode, "tbt_dist_init: FULL (non-reciprocal) generators are not supported on a distributed context");
  TBT_USER_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "tbt_dist_init: bad rank");
  TBT_USER_CHECK(nranks <= c.L0, "tbt_dist_init: more ranks than level-0 bins");
  // Every rank owns at least one element row (its slab of the vectors, the
  // halo rows of the correction, non-empty reduction grids).
  TBT_USER_CHECK(nranks <= c.ny, "tbt_dist_init: more ranks than element rows (ny)");
  TBT_CUDA_CHECK(cudaSetDevice(c.device));
  distFree(c);
  c.dropGraph();
  c.nranks = nranks;
  c.myRank = rank;
  distPlan(c.ny, c.L0, nranks, c.rowStart, c.colsOfRank);
  c.myRow0 = c.rowStart[rank];
  c.myRows = c.rowStart[rank + 1] - c.rowStart[rank];
  c.myColList = c.colsOfRank[rank];
  c.colsOffset.assign(nranks + 1, 0);
  std::vector<int> flat;
  for (int q = 0; q < nranks; ++q) {
    flat.insert(flat.end(), c.colsOfRank[q].begin(), c.colsOfRank[q].end());
    c.colsOffset[q + 1] = static_cast<int>(flat.size());
  }
  const long long B = static_cast<long long>(c.maxNrhs) * c.m;
  const long long myCols = static_cast<long long>(c.myColList.size());
  TBT_CUDA_CHECK(cudaMalloc(&c.dColsOfRank, flat.size() * sizeof(int)));
  uploadSync(c.dColsOfRank, flat.data(), flat.size() * sizeof(int), c.stream);
  std::vector<int4> tab;
  for (int q = 0; q < nranks; ++q)
    for (int j = 0; j < static_cast<int>(c.colsOfRank[q].size()); ++j)
      tab.push_back(make_int4(c.colsOfRank[q][j], j, static_cast<int>(c.colsOfRank[q].size()), c.colsOffset[q]));
  TBT_CUDA_CHECK(cudaMalloc(&c.dColTab, tab.size() * sizeof(int4)));
  uploadSync(c.dColTab, tab.data(), tab.size() * sizeof(int4), c.stream);
  TBT_CUDA_CHECK(cudaMalloc(&c.dTrow, std::max<long long>(1, c.myRows * c.L0 * B) * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dSend, std::max<long long>(1, c.myRows * c.L0 * B) * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dTcol, std::max<long long>(1, c.ny * myCols * B) * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dRecv, std::max<long long>(1, c.ny * myCols * B) * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dXhalo, (c.myRows + 2) * static_cast<long long>(c.nx) * B * sizeof(double2)));
  memsetSync(c.dXhalo, 0, (c.myRows + 2) * static_cast<long long>(c.nx) * B * sizeof(double2), c.stream);
  TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&c.commStream, cudaStreamNonBlocking));
  for (cudaEvent_t& e : c.distEv) TBT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c.comm = loopback ? makeLoopbackComm(nranks, rank, id) : makeNcclComm(nranks, rank, id);
  c.dist = true;
}
}  // namespace

tbt_status tbt_dist_init(tbt_ctx* h, int nranks, int rank, const char* id) {
  return guardedCtx(h, [&] { distInit(h, nranks, rank, id, false); });
}

tbt_status tbt_dist_init_loopback(tbt_ctx* h, int nranks, int rank, const char* id) {
  return guardedCtx(h, [&] { distInit(h, nranks, rank, id, true); });
}

tbt_status tbt_dist_transport(const tbt_ctx* h, int* kind) {
  return guarded([&] {
    TBT_USER_CHECK(h && kind, "tbt_dist_transport: null argument");
    *kind = h->c.dist && h->c.comm ? h->c.comm->kind() : 0;
  });
}

tbt_status tbt_dist_rows(const tbt_ctx* h, int* row_begin, int* row_end) {
  return guarded([&] {
    TBT_USER_CHECK(h && row_begin && row_end, "tbt_dist_rows: null argument");
    const Ctx& c = h->c;
    *row_begin = c.dist ? c.myRow0 : 0;
    *row_end = c.dist ? c.myRow0 + c.myRows : c.ny;
  });
}

tbt_status tbt_phase_times(tbt_ctx* h, int on, double* out_us) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h, "tbt_phase_times: null context");
    Ctx& c = h->c;
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.dropGraph();
    if (out_us) {
      unsigned long long ns[32];
      TBT_CUDA_CHECK(cudaMemcpy(ns, c.dPhaseNs, sizeof(ns), cudaMemcpyDeviceToHost));
      for (int k = 0; k < 5; ++k) out_us[k] = ns[k + 1] >= ns[k] ? 1e-3 * static_cast<double>(ns[k + 1] - ns[k]) : 0.0;
      // [5..8]: latest CTA arrival at barrier k relative to CTA 0's phase start;
      // [9..12]: earliest arrival.
      for (int k = 0; k < 4; ++k) {
        out_us[5 + k] = ns[8 + k] >= ns[k] ? 1e-3 * static_cast<double>(ns[8 + k] - ns[k]) : -1.0;
        out_us[9 + k] = ns[16 + k] >= ns[k] ? 1e-3 * static_cast<double>(ns[16 + k] - ns[k]) : -1.0;
      }
    }
    // Reset the arrival extrema for the next armed apply.
    std::vector<unsigned long long> init(32, 0ULL);
    for (int k = 16; k < 24; ++k) init[k] = ~0ULL;
    uploadSync(c.dPhaseNs, init.data(), 32 * sizeof(unsigned long long), c.stream);
    c.phaseTiming = on != 0;
  });
}

tbt_status tbt_cta_trace(tbt_ctx* h, unsigned long long* out, long long cap, long long* launches) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && out && launches, "tbt_cta_trace: bad argument");
    Ctx& c = h->c;
    TBT_USER_CHECK(c.dCtaTrace, "tbt_cta_trace: tracing is off (set TBT_CTATRACE=1 before tbt_create)");
    const long long n = static_cast<long long>(kCtaTraceSlots) * kCtaTraceEvents * kCtaTraceMaxGrid;
    TBT_USER_CHECK(cap >= n, "tbt_cta_trace: buffer too small");
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    TBT_CUDA_CHECK(cudaMemcpy(out, c.dCtaTrace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    *launches = c.ctaTraceLaunches;
  });
}

tbt_status tbt_bench_apply(tbt_ctx* h, const double* x_dev, double* y_dev, int nrhs, int iters, int use_graph,
                           double* out_ms, double* out_binprod_ms) {
  return guardedCtx(h, [&] {
    TBT_USER_CHECK(h && x_dev && y_dev && iters >= 1, "tbt_bench_apply: bad argument");
    Ctx& c = h->c;
    requireReady(c);
    TBT_USER_CHECK(nrhs == 1, "tbt_bench_apply: nrhs must be 1");
    const double2* x = reinterpret_cast<const double2*>(x_dev);
    double2* y = reinterpret_cast<double2*>(y_dev);
    cudaEvent_t e0, e1;
    TBT_CUDA_CHECK(cudaEventCreate(&e0));
    TBT_CUDA_CHECK(cudaEventCreate(&e1));
    cudaGraphExec_t exec = nullptr;
    if (use_graph) {
      cudaGraph_t graph;
      TBT_CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      applyInternal(c, x, y, 1, true);
      TBT_CUDA_CHECK(cudaStreamEndCapture(c.stream, &graph));
      TBT_CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
    }
    // Whole applies.
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    TBT_CUDA_CHECK(cudaEventRecord(e0, c.stream));
    for (int k = 0; k < iters; ++k) {
      if (exec)
        TBT_CUDA_CHECK(cudaGraphLaunch(exec, c.stream));
      else
        applyInternal(c, x, y, 1, true);
    }
    TBT_CUDA_CHECK(cudaEventRecord(e1, c.stream));
    TBT_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    TBT_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (out_ms) *out_ms = ms / iters;
    // The bin-product kernel alone, back to back on the same data.
    if (out_binprod_ms) {
      TBT_CUDA_CHECK(cudaEventRecord(e0, c.stream));
      for (int k = 0; k < iters; ++k) launchBinProduct(c, 1);
      TBT_CUDA_CHECK(cudaEventRecord(e1, c.stream));
      TBT_CUDA_CHECK(cudaEventSynchronize(e1));
      TBT_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      *out_binprod_ms = ms / iters;
    }
    if (exec) cudaGraphExecDestroy(exec);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
