// Internal declarations of the B200 block-Toeplitz library (libtbt.so).
#pragma once

#include <array>
#include <atomic>

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tbt.h"

namespace tbt {

// ---------------------------------------------------------------- errors
void setError(const std::string& msg);
struct Error {
  tbt_status code;
  std::string msg;
};
#define TBT_CUDA_CHECK(expr)                                                     \
  do {                                                                           \
    cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                       \
      throw ::tbt::Error{TBT_CUDA_ERROR, std::string(#expr) + ": " +             \
                                            cudaGetErrorString(e_)};             \
  } while (0)
#define TBT_USER_CHECK(cond, msg)                                                \
  do {                                                                           \
    if (!(cond)) throw ::tbt::Error{TBT_USER_ERROR, (msg)};                     \
  } while (0)

// ---------------------------------------------------------------- complex
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc += a * b
__host__ __device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__host__ __device__ __forceinline__ void cfma_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// ---------------------------------------------------------------- FFT plan
// One batched 1-D pass over "lines" of a [point][batch] layout (batch
// contiguous). Line l, point p, batch b lives at
//   base + l*line_stride + p*point_stride + b      (complex units).
struct FftPass {
  const double2* in = nullptr;
  double2* out = nullptr;
  long long in_line_stride = 0, in_point_stride = 0;
  long long out_line_stride = 0, out_point_stride = 0;
  int lines = 0;
  int n = 1;       // transform length
  int n_in = 1;    // leading input points that may be non-zero
  int n_out = 1;   // leading output points written
  int batch = 0;   // batch entries per point
  int inverse = 0;
  double scale = 1.0;
  const double2* tw = nullptr;  // exp(-2 pi i t / n), t < n
  // Optional store epilogue (the last inverse pass of a multi-RHS apply):
  // out += ycorr at the same index for elements e = line * corrNx + point
  // with correction terms (tPtr[e] != tPtr[e + 1]).
  const int* tPtr = nullptr;
  const double2* ycorr = nullptr;
  int corrNx = 0;
  // Register passes only: read `in` / write `out` in the user's column-major
  // n x nrhs layout (element e = line * userNx + point, batch entry
  // bg = rhs * userM + a -> rhs * userN + e * userM + a) instead of the
  // strided internal one.
  int inUser = 0, outUser = 0, userNx = 0, userM = 0;
  long long userN = 0;
};
void launchFftPass(const FftPass& p, cudaStream_t s);
// Register line pass (fft.cu): one thread per (line, batch entry), the whole
// line in registers; for n <= 64 and wide batches. Returns false otherwise.
bool launchFftPassReg(const FftPass& p, cudaStream_t s);

// Cluster-fused 2-D transform (fft2d.cu).
struct Fft2dArgs {
  const double2* in = nullptr;
  double2* out = nullptr;
  int nx = 0, ny = 0, L0 = 1, L1 = 1, B = 0;
  const double2* tw0 = nullptr;
  const double2* tw1 = nullptr;
  double scale = 1.0;
  // Inverse-transform epilogue: edge/corner correction (correction.cu).
  int corr = 0;
  const int* tPtr = nullptr;       // [ne+1] terms of element e (non-empty -> add ycorr)
  const double2* ycorr = nullptr;  // [e][B] correction vector (launchCorrVector)
};
bool fft2dSupported(int L0, int L1);
void fft2dPlan(int L0, int L1, int nx, int ny, int B, int sms, int* CL, int* BC);
bool launchFft2d(const Fft2dArgs& a, int CL, int BC, bool inverse, cudaStream_t s);

// ---------------------------------------------------------------- context
struct CorrTerm {  // y[target] += P x[source] (trans 0) or P^T x[source]
  int target, source, slot, trans;
};

// Transport of the sharded operator (dist.cu): grouped point-to-point
// exchanges and a sum all-reduce, on the calling context's stream.
//  * NCCL: one process per GPU (ncclSend / ncclRecv / ncclAllReduce over
//    NVLink / NVSwitch), the production path;
//  * loopback: P rank contexts of ONE process on one device, each driven by
//    its own host thread; groupEnd / allReduceSum synchronise the caller's
//    stream, meet the other ranks at a host barrier and move the data with
//    device-to-device copies (sums in fixed rank order). No kernel ever
//    waits on another rank, so it is safe on a single GPU, and it runs the
//    exact pack / exchange / unpack code of the NCCL path at any P.
struct Comm {
  virtual ~Comm() = default;
  virtual void groupStart() = 0;
  virtual void send(const void* buf, size_t ndoubles, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t ndoubles, int peer, cudaStream_t s) = 0;
  virtual void groupEnd(cudaStream_t s) = 0;
  virtual void allReduceSum(double* buf, size_t ndoubles, cudaStream_t s) = 0;  // in place
  virtual void abort() {}  // a rank failed: release the others (loopback)
  virtual int kind() const = 0;  // 1 NCCL, 2 loopback
};
Comm* makeNcclComm(int nranks, int rank, const char* id);
Comm* makeLoopbackComm(int nranks, int rank, const char* id);

struct Ctx {
  int nx = 0, ny = 0, m = 0, ne = 0, maxNrhs = 1, device = 0;
  long long n = 0;  // nx*ny*m
  int L0 = 1, L1 = 1;
  long long L = 1;
  cudaStream_t stream = nullptr;
  bool ownStream = false;
  cudaStream_t side = nullptr;             // parallel branch (correction projection)
  cudaEvent_t evFork = nullptr, evJoin = nullptr;
  bool fused2d = false;                    // cluster-fused 2-D transforms available
  bool persistent = false;                 // single-kernel apply (matvec_persistent.cu)
  unsigned* dGridBar = nullptr;            // grid barrier counter / generation
  unsigned long long* dBarFlags = nullptr; // flag-line grid barrier (matvec_persistent.cu)
  bool phaseTiming = false;
  int prefetchAt = 0;                      // TBT_PREFETCH: 0 kernel start, 1 after rows, 2 after columns
  long long zeroCopyL2Bytes = 0;  // set around zero-copy launches: spectrum bytes to prefetch into L2
  bool zeroCopyStage = false;     // set around zero-copy launches: stage x in dXin for the correction reads
  bool coopChecked = false;      // a cooperative persistent launch succeeded on this context (co-residency)
  bool countedLive = false;      // included in the live-context count of its device (plainLaunchOk)
  bool inSolve = false;               // a GMRES solve is issuing this context's applies
  unsigned long long zigzagSeq = 0;  // persistent applies in solves so far (pair-order parity)
  bool usePdl = true;             // device-resident single-column applies launched directly with PDL (TBT_PDL=0: graph)
  const int* skipFlag = nullptr;  // device flag: persistent applies become no-ops when set
  unsigned long long* dPhaseNs = nullptr;  // [6] globaltimer stamps of the last persistent apply
  unsigned long long* dCtaTrace = nullptr; // TBT_CTATRACE=1: per-CTA event times of the persistent apply
  long long ctaTraceLaunches = 0;          // launches traced so far (slot = count % kCtaTraceSlots)
  bool forceMultiPass = false;             // TBT_FFT=passes
  bool forceFused2d = false;               // TBT_FFT=fused: cluster 2-D kernels also for wide batches
  bool forceUnfused = false;               // TBT_GMRES=unfused: separate apply / Arnoldi launches
  bool forceCols = false;                  // TBT_GMRES=cols: column-blocked Arnoldi for one column too

  // Multi-GPU (dist.cu): this rank owns element rows [myRow0, myRow0 +
  // myRows) of the vectors and the bin columns myColList (closed under
  // s0 -> L0 - s0, so both bins of every stored pair are local).
  bool dist = false;
  int nranks = 1, myRank = 0;
  // tbt_apply_many: two device slots per direction, copy streams and the
  // events that order H2D -> apply -> D2H per slot (allocated on first use).
  double2* dManyX[2] = {nullptr, nullptr};
  double2* dManyY[2] = {nullptr, nullptr};
  cudaStream_t manyIn = nullptr, manyOut = nullptr;
  cudaEvent_t manyEv[6] = {};  // [0..1] x landed, [2..3] apply done, [4..5] y read back
  Comm* comm = nullptr;
  cudaStream_t commStream = nullptr;  // exchanges of the chunked (overlapped) sharded apply
  cudaEvent_t distEv[8] = {};         // fork / join events between the compute and comm streams
  std::vector<int> rowStart;                  // [nranks+1]
  std::vector<std::vector<int>> colsOfRank;   // [nranks]
  std::vector<int> myColList;
  int myRow0 = 0, myRows = 0;
  int* dColsOfRank = nullptr;                 // concatenated column lists
  int4* dColTab = nullptr;                    // [L0] {column, j, peer's column count, peer's colsOffset}
  std::vector<int> colsOffset;                // [nranks+1] offsets into dColsOfRank
  double2* dTrow = nullptr;   // [myRows][L0][B]
  double2* dTcol = nullptr;   // [ny][myCols][B]
  double2* dSend = nullptr;
  double2* dRecv = nullptr;
  double2* dXhalo = nullptr;  // [myRows + 2 halo rows][nx][B]: x for the local correction
  // Correction terms whose target is a local element, sources indexed into
  // dXhalo (row - (myRow0 - 1)), targets into this rank's slab.
  int* dTermInfoLoc = nullptr;
  int* dTargetListLoc = nullptr;
  int* dTargetPtrLoc = nullptr;
  int nTargetsLoc = 0, maxTermsLoc = 0;
  double2* dYcorrLoc = nullptr;  // [myRows*nx][B], zero outside the targets
  bool distCorrReady = false;

  // Generators (host copy kept for diagonal / K) and spectra.
  std::vector<double2> genHost;   // only the self block Z(0,0) (m*m, column-major)
  double2* dGen = nullptr;        // all canonical blocks on the device until tbt_precompute
  bool haveGenerators = false, havePrecompute = false;
  // Identity of the generator set for TBTS1 spectrum caches (tbt_set_cache_key):
  // written with the cache, and a load into a context that has a key
  // requires the same key.
  unsigned char cacheKey[32] = {};
  bool haveCacheKey = false;
  long long npairs = 0;
  double2* dSpectra = nullptr;    // [npairs][m][m] row-major
  // FULL (non-reciprocal) generators, tbt_set_generators_full: A = A_s + A_a
  // with A_s reciprocal (the usual half spectrum, dGen / dSpectra) and A_a
  // anti-reciprocal, A_a(-s) = -A_a(s)^T (canonical half in dGenAnti until
  // tbt_precompute, its half spectrum in dSpectraAnti, applied by a second
  // K3 pass that negates the partner product). Multi-launch apply path only.
  bool fullMode = false;
  double2* dGenAnti = nullptr;
  double2* dSpectraAnti = nullptr;
  int* dPairF = nullptr;          // representative bin of pair p
  int* dPairG = nullptr;          // partner bin (== F for self-paired)
  std::vector<int> pairF, pairG;  // host copies
  std::vector<long long> pairOfBin;  // bin -> pair (negative: -(p+1) transposed)
  bool hasAntisym = false;
  double2* dAntisym = nullptr;    // K = (Z0 - Z0^T)/2, [a][b] row-major

  // Twiddles for L0, L1.
  double2* dTw0 = nullptr;
  double2* dTw1 = nullptr;

  // Correction.
  int rank = 0;
  bool haveCorr = false;
  double2* dCorrD = nullptr;  // [40][m]
  double2* dCorrU = nullptr;  // [40][rank][m]
  double2* dCorrV = nullptr;
  std::vector<double2> corrDHost;
  int nTerms = 0, nTargets = 0, maxTermsPerTarget = 0;
  double2* dYcorr = nullptr;    // [ne][maxNrhs*m] correction vector (multi-launch paths)
  // The persistent kernel's own [ne][m] correction vector: it writes only
  // the target elements and reads every element, so the entries off the
  // targets must stay zero whatever column count the other paths used.
  double2* dYcorrP = nullptr;
  double2* dTermVec = nullptr;  // [nCorrPairs][m] per-(target,source) vectors (persistent apply)
  int nCorrPairs = 0;
  int* dPairInfo = nullptr;       // [pair][4] {target, source, code0, code1}
  int* dPairTargetPtr = nullptr;  // [nTargets+1]
  int* dTermInfo = nullptr;     // [nTerms][4] {target, source, slot, trans}
  int* dTargetList = nullptr;   // [nTargets] target elements
  int* dTargetPtr = nullptr;    // [nTargets+1] CSR over terms
  int* dElemPtr = nullptr;      // [ne+1] CSR over terms by element
  double2* dProj = nullptr;     // [nTerms][nrhs][rank]

  // Work buffers sized for maxNrhs.
  double2* dT = nullptr;      // [ny][L0][B]
  double2* dXhat = nullptr;   // [L][B]
  double2* dYhat = nullptr;   // [L][B]
  double2* dXin = nullptr;    // [ne][B] staging (host/colmajor input)
  double2* dYout = nullptr;   // [ne][B]
  double2* dDiagInv = nullptr;   // 1/diag(Z), Jacobi of iterativeSolve
  double2* dDiagInvA = nullptr;  // 1/diag(A), Jacobi of the A-only solves

  struct GmresWs* gmresWs = nullptr;
  struct ClusterSmall* clusterSmall = nullptr;  // one-cluster apply / GMRES for tiny operators (cluster_small.cu)

  // Margin coupling B / B^T / C (margin.cu): nM margin unknowns stored as
  // neM = ceil(nM/m) zero-padded pseudo-elements after the ne elements.
  struct MarginOp* margin = nullptr;
  long long nM = 0;
  int neM = 0;  // cached GMRES workspace + inner-loop graph (gmres.cu)

  // Timing hooks: event pairs around K3, one per timed apply.
  cudaEvent_t evBinA = nullptr, evBinB = nullptr;
  bool timeBinprod = false;
  std::vector<cudaEvent_t> tEvA, tEvB;
  int tCount = 0;
  int binprodKernel = 0;

  // CUDA graph of one device-resident single-column apply.
  cudaGraphExec_t graphExec = nullptr;
  const void* graphX = nullptr;
  void* graphY = nullptr;
  bool graphCorr = false;
  void dropGraph() {
    if (graphExec) cudaGraphExecDestroy(graphExec);
    graphExec = nullptr;
    graphX = graphY = nullptr;
  }
};

// Kernels / launchers implemented in the .cu files.
void buildSpectra(Ctx& c);                                    // spectra.cu
std::vector<double2> splitSelfBlock(Ctx& c);                   // spectra.cu: K on device, returns S0
void planPairs(Ctx& c, std::vector<int>& pairFGlobal);         // spectra.cu: pair tables + spectrum allocation
void applyInternal(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr);  // apply.cu
// Many columns straight from / to the user's column-major layout (no layout
// kernels) when the register-pass path serves the context; false otherwise.
bool applyUserLayout(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr);  // apply.cu
void launchBinProduct(Ctx& c, int nrhs);                      // binprod.cu
void launchBinProductAnti(Ctx& c, int nrhs);                  // binprod.cu: FULL generators, yhat += A_a xhat
int binprodVariant(int m);                                    // binprod.cu
constexpr int kCtaTraceSlots = 8, kCtaTraceEvents = 16, kCtaTraceMaxGrid = 256;  // TBT_CTATRACE buffer shape
constexpr int kGemmMinRhs = 8;  // from this many columns on, K3 is the DMMA GEMM
bool launchBinProductGemm(Ctx& c, int nrhs);                 // binprod_gemm.cu
void launchCorrection(Ctx& c, const double2* x, double2* y, int nrhs);  // correction.cu
// xUserN > 0: x in the user's column-major n x nrhs layout instead of [e][rhs][a].
void launchCorrVector(Ctx& c, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                      long long xUserN = 0);  // correction.cu
// A term table (CSR by target): termInfo[4t..] = (target, source, slot, trans).
struct CorrTables {
  const int* termInfo;
  const int* targetList;
  const int* targetPtr;
  int nTargets, maxTerms;
  const int* order = nullptr;  // [nTargets] launch order of the targets (longest term lists first), or identity
};
void launchCorrVectorOn(Ctx& c, const CorrTables& t, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                        long long xUserN = 0);
// Per target element, its correction terms {target, source, slot, trans} in
// the order every apply path accumulates them (api.cu).
std::vector<std::vector<std::array<int, 4>>> corrTermsByTarget(int nx, int ny);
void launchAntisym(Ctx& c, const double2* x, double2* y, int nrhs, int nElems = -1);  // correction.cu
void launchLayout(const double2* in, double2* out, long long n, int nrhs, bool toInternal, cudaStream_t s, int m);  // apply.cu
// External n_user x nrhs column-major <-> internal [e][rhs][m] of n_int rows per column (zero padding).
void launchLayoutU(const double2* in, double2* out, long long nUser, long long nInt, int nrhs, bool toInternal,
                   cudaStream_t s, int m);
// The full operator on internal vectors: applyInternal (+ margin B/B^T/C when present and withCorr).
void applyOperator(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr);

// GMRES (gmres.cu): per-column state mirrored to the host.
struct GmresState {
  double bnorm, beta, residual, beta0;
  int iterations, ncount, stopInner, done, converged, cycleActive, histLen;
  int checks;  // true-residual applies (restart checks + the final one), cluster solve
};
void gmresSolve(Ctx& c, const double2* b, double2* x, int ncols, const tbt_gmres_opts& o, bool useAOnly,
                std::vector<GmresState>& out, std::vector<double>& hist, int& matvecs);

// Multi-GPU (dist.cu). NCCL entry points resolved at run time.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl();

#define TBT_NCCL_CHECK(expr)                                                                  \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      throw ::tbt::Error{TBT_CUDA_ERROR, std::string(#expr) + ": " + nccl().errorString(r_)}; \
  } while (0)
// io.cu (row f3): reference ZTOE1 block caches, persisted spectra.
struct Ztoe1Data {
  int mode = 2;  // StorageMode: 1 SemiSparse, 2 Sparse
  int nx = 0, ny = 0;
  int e[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long nM = 0;
  std::vector<double2> gen, bside, brow, bcorner, c;  // tbt_gen.h layouts; c: nM x nM column-major
  std::vector<double2> bfull;                         // SemiSparse: nM x nA column-major
};
void readZtoe1(const std::string& path, Ztoe1Data& out);
void saveSpectra(Ctx& c, const std::string& path);
void loadSpectra(Ctx& c, const std::string& path);

// cluster_small.cu: tiny operators (C1) on one 8-CTA cluster.
bool clusterSmallSupported(const Ctx& c, int restart);
void launchClusterApply(Ctx& c, const double2* x, double2* y, bool withCorr);
void clusterSmallFree(Ctx& c);

// postproc.cu (row f4), device pointers.
void portNetwork(Ctx& c, const double2* current, long long ldc, int p, const long long* feedDev, double len,
                 const double* z0Dev, double2* y, double2* z, double2* s);
void arrayFarfield(Ctx& c, const double2* const* tco, const double2* const* tcx, const int* e, int ndir,
                   const double* dirsDev, double dx, double dy, double k, double eta, const double2* current,
                   long long ntot, int p, const double2* W, int q, double2* co, double2* cx);

// margin.cu
void marginSet(Ctx& c, const int* e, const double2* bside, const double2* brow, const double2* bcorner,
               const double2* C);
void marginSetDense(Ctx& c, const int* e, const double2* B, const double2* C);  // SemiSparse: dense B, C
void marginFree(Ctx& c);
void marginApply(Ctx& c, const double2* x, double2* y, int nrhs);  // y's element part already holds A x
void marginDiagonal(const Ctx& c, std::vector<double2>& d);          // appends C's diagonal
// schur.cu: b, x device (nA + nM) x p column-major (user layout).
void schurSolve(Ctx& c, const double2* b, double2* x, int p, const tbt_gmres_opts& o, std::vector<int>& iterations,
                std::vector<double>& residual);
std::vector<double2> twiddleTable(int n);                           // api.cu
bool poisonBuffers();
bool stagedE2E();                                               // api.cu: TBT_POISON=1
void uploadSync(void* dst, const void* src, size_t bytes, cudaStream_t s);  // api.cu
void memsetSync(void* dst, int value, size_t bytes, cudaStream_t s);        // api.cu

void distPlan(int ny, int L0, int P, std::vector<int>& rowStart, std::vector<std::vector<int>>& cols);
void applyDist(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr);
void distCorrPrepare(Ctx& c);  // local correction tables (allocates: call outside stream capture)
void distFree(Ctx& c);

// Persistent single-kernel apply (matvec_persistent.cu).
bool persistentSupported(const Ctx& c);
struct GmresArgs;
struct GmresWs;
void freeGmresWorkspace(Ctx& c);  // gmres.cu
bool launchPersistentApply(Ctx& c, const double2* x, double2* y, bool withCorr, const GmresArgs* gm = nullptr,
                           double2* lsS = nullptr, double2* lsDots = nullptr, double2* lsPart = nullptr,
                           bool lagged = false);
// A LAGGED (lagged-normalisation) GMRES-step instantiation exists for this
// shape and its LS scratch fits next to the ring.
bool persistentLaggedFits(const Ctx& c, const GmresArgs& gm);

// Launch configuration helper: SM count of the context's device.
int smCount(int device);
// Context lifetime bookkeeping per device. Persistent kernels launch plainly
// (not cooperatively) only while ONE context lives on the device: two
// plain grid-barrier grids issued from different contexts' streams could
// each end up partly resident and wait on each other forever, which a
// cooperative launch rules out.
void liveContextAdd(Ctx& c);
void liveContextRemove(Ctx& c);
bool plainLaunchOk(const Ctx& c);

// Runs f (a cudaFuncSetAttribute call) once per device for the kernel that
// owns `mask`: function attributes are per device, so a process driving
// contexts on several GPUs must set them on each. The bit is published only
// after f returned, so no caller launches before its attribute is set.
template <class F>
inline void oncePerDevice(std::atomic<unsigned long long>& mask, F&& f) {
  int dev = 0;
  TBT_CUDA_CHECK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return;
  f();
  mask.fetch_or(bit, std::memory_order_release);
}

}  // namespace tbt
