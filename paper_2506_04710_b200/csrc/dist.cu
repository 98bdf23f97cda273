// Multi-GPU operator: one process per GPU, the operator
// sharded over P ranks with NCCL over NVLink/NVSwitch.
//
//  * Bins are split by level-0 column s0 into P slabs. Columns are assigned
//    in groups {0}, {L0/2}, {s, L0-s} (closed under s0 -> -s0), so both bins
//    of every stored pair {f, -f} live on one rank and the half-spectrum
//    storage of spectra.cu carries over unchanged: each rank keeps ~1/P of
//    the Fourier blocks (C5: 38.65 GB full / 19.3 GB half -> ~2.4 GB per
//    rank at P = 8).
//  * Vectors are split by element row (contiguous slabs of ny/P rows).
//  * apply: row FFTs of the local rows -> all-to-all (grouped ncclSend /
//    ncclRecv; NCCL has no all-to-all primitive) -> column FFTs of the local
//    columns -> bin products of the local pairs (the K3 kernels) -> inverse
//    column FFTs keeping ny rows -> all-to-all back -> inverse row FFTs.
//    The edge/corner correction of an element reads x of its 4-neighbours
//    only: one halo element row is exchanged with each slab neighbour and
//    each rank evaluates the terms of its own target elements.
//  * The exchanges go through a Comm (tbt_internal.cuh): NCCL across
//    processes / GPUs, or the in-process loopback transport that runs P
//    rank contexts on one device (tbt_dist_init_loopback).
// Replaces applyA / apply (proj/src/linsolve.cpp:260-290,373-388), which has
// no distributed counterpart ("Non-goals: distributed").
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>

#include "tbt_internal.cuh"

namespace tbt {

// NCCL is loaded on first use (dlopen), not linked: a process that already
// loaded torch's NCCL reuses it (same SONAME), and importing this library
// before torch cannot bind torch to an older system NCCL.
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
#define TBT_SYM(name, field) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #name))
    TBT_SYM(ncclGetUniqueId, getUniqueId);
    TBT_SYM(ncclCommInitRank, commInitRank);
    TBT_SYM(ncclCommDestroy, commDestroy);
    TBT_SYM(ncclGroupStart, groupStart);
    TBT_SYM(ncclGroupEnd, groupEnd);
    TBT_SYM(ncclSend, send);
    TBT_SYM(ncclRecv, recv);
    TBT_SYM(ncclGetErrorString, errorString);
    TBT_SYM(ncclAllReduce, allReduce);
#undef TBT_SYM
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd &&
             api.send && api.recv && api.errorString && api.allReduce;
  });
  if (!api.ok) throw Error{TBT_CUDA_ERROR, "NCCL (libnccl.so.2) could not be loaded"};
  return api;
}

// ---------------------------------------------------------------- NCCL
namespace {

class NcclComm final : public Comm {
 public:
  NcclComm(int nranks, int rank, const char* id) {
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    const ncclResult_t r = nccl().commInitRank(&comm_, nranks, u, rank);
    if (r != ncclSuccess) throw Error{TBT_CUDA_ERROR, std::string("ncclCommInitRank: ") + nccl().errorString(r)};
  }
  ~NcclComm() override {
    if (comm_) nccl().commDestroy(comm_);
  }
  void groupStart() override { TBT_NCCL_CHECK(nccl().groupStart()); }
  void send(const void* buf, size_t n, int peer, cudaStream_t s) override {
    TBT_NCCL_CHECK(nccl().send(buf, n, ncclDouble, peer, comm_, s));
  }
  void recv(void* buf, size_t n, int peer, cudaStream_t s) override {
    TBT_NCCL_CHECK(nccl().recv(buf, n, ncclDouble, peer, comm_, s));
  }
  void groupEnd(cudaStream_t) override { TBT_NCCL_CHECK(nccl().groupEnd()); }
  void allReduceSum(double* buf, size_t n, cudaStream_t s) override {
    TBT_NCCL_CHECK(nccl().allReduce(buf, buf, n, ncclDouble, ncclSum, comm_, s));
  }
  int kind() const override { return 1; }

 private:
  ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------- loopback
constexpr int kLoopMaxRanks = 64;
constexpr auto kLoopTimeout = std::chrono::seconds(120);

struct LoopSend {
  int peer;
  const void* buf;
  size_t n;
};

// Shared state of the P contexts of one loopback group (same process).
struct LoopGroup {
  int P = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  bool aborted = false;
  std::vector<std::vector<LoopSend>> sends;  // [rank] this group's posted sends
  std::vector<const double*> reduceIn;       // [rank] all-reduce inputs

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Error{TBT_CUDA_ERROR, "loopback transport: another rank failed"};
    const unsigned long long g = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, kLoopTimeout, [&] { return generation != g || aborted; })) {
      aborted = true;
      cv.notify_all();
      throw Error{TBT_CUDA_ERROR, "loopback transport: timed out waiting for the other ranks"};
    }
    if (aborted) throw Error{TBT_CUDA_ERROR, "loopback transport: another rank failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

std::mutex gLoopMu;
std::map<std::string, std::weak_ptr<LoopGroup>> gLoopGroups;

struct SumArgs {
  const double* in[kLoopMaxRanks];
};

// out[k] = in[0][k] + in[1][k] + ... + in[P-1][k], in that order on every
// rank, so all ranks hold bitwise identical totals.
__global__ void loopSum(SumArgs a, int P, double* __restrict__ out, long long n) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    double v = a.in[0][k];
    for (int r = 1; r < P; ++r) v += a.in[r][k];
    out[k] = v;
  }
}

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(int nranks, int rank, const char* id) : rank_(rank) {
    if (nranks > kLoopMaxRanks) throw Error{TBT_USER_ERROR, "tbt_dist_init_loopback: at most 64 ranks"};
    const std::string key(id, NCCL_UNIQUE_ID_BYTES);
    std::lock_guard<std::mutex> lk(gLoopMu);
    for (auto it = gLoopGroups.begin(); it != gLoopGroups.end();)
      it = it->second.expired() ? gLoopGroups.erase(it) : std::next(it);
    auto& slot = gLoopGroups[key];
    g_ = slot.lock();
    if (!g_) {
      g_ = std::make_shared<LoopGroup>();
      g_->P = nranks;
      g_->sends.assign(nranks, {});
      g_->reduceIn.assign(nranks, nullptr);
      slot = g_;
    }
    if (g_->P != nranks) throw Error{TBT_USER_ERROR, "tbt_dist_init_loopback: ranks disagree on the group size"};
  }
  ~LoopbackComm() override {
    if (tmp_) cudaFree(tmp_);
  }
  void groupStart() override {
    sends_.clear();
    recvs_.clear();
  }
  void send(const void* buf, size_t n, int peer, cudaStream_t) override { sends_.push_back({peer, buf, n}); }
  void recv(void* buf, size_t n, int peer, cudaStream_t) override { recvs_.push_back({peer, buf, n}); }
  void groupEnd(cudaStream_t s) override {
    guard([&] {
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));  // send buffers complete
      g_->sends[rank_] = sends_;
      g_->barrier();
      // The k-th receive from q matches q's k-th send to this rank (NCCL's
      // ordering rule for grouped point-to-point operations).
      std::vector<int> used(g_->P, 0);
      for (const LoopSend& r : recvs_) {
        const std::vector<LoopSend>& theirs = g_->sends[r.peer];
        int seen = 0;
        const LoopSend* match = nullptr;
        for (const LoopSend& t : theirs)
          if (t.peer == rank_ && seen++ == used[r.peer]) {
            match = &t;
            break;
          }
        if (!match || match->n != r.n)
          throw Error{TBT_CUDA_ERROR, "loopback transport: unmatched or mis-sized receive"};
        ++used[r.peer];
        if (r.n)
          TBT_CUDA_CHECK(cudaMemcpyAsync(const_cast<void*>(r.buf), match->buf, r.n * sizeof(double),
                                         cudaMemcpyDeviceToDevice, s));
      }
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));  // received data landed
      g_->barrier();                             // every peer finished reading my sends
    });
  }
  void allReduceSum(double* buf, size_t n, cudaStream_t s) override {
    guard([&] {
      if (n > tmpN_) {
        if (tmp_) cudaFree(tmp_);
        tmp_ = nullptr;
        TBT_CUDA_CHECK(cudaMalloc(&tmp_, n * sizeof(double)));
        tmpN_ = n;
      }
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
      g_->reduceIn[rank_] = buf;
      g_->barrier();
      SumArgs a{};
      for (int r = 0; r < g_->P; ++r) a.in[r] = g_->reduceIn[r];
      const int blocks = static_cast<int>(std::min<long long>((static_cast<long long>(n) + 255) / 256, 1024));
      if (n) loopSum<<<std::max(blocks, 1), 256, 0, s>>>(a, g_->P, tmp_, static_cast<long long>(n));
      TBT_CUDA_CHECK(cudaGetLastError());
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
      g_->barrier();  // every rank read every input
      if (n) TBT_CUDA_CHECK(cudaMemcpyAsync(buf, tmp_, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    });
  }
  void abort() override { g_->abort(); }
  int kind() const override { return 2; }

 private:
  template <class F>
  void guard(F&& f) {
    try {
      f();
    } catch (...) {
      g_->abort();
      throw;
    }
  }
  int rank_;
  std::shared_ptr<LoopGroup> g_;
  std::vector<LoopSend> sends_, recvs_;
  double* tmp_ = nullptr;
  size_t tmpN_ = 0;
};

}  // namespace

Comm* makeNcclComm(int nranks, int rank, const char* id) { return new NcclComm(nranks, rank, id); }
Comm* makeLoopbackComm(int nranks, int rank, const char* id) { return new LoopbackComm(nranks, rank, id); }

// Row slabs and column groups (pure host logic; tested on the CPU).
void distPlan(int ny, int L0, int P, std::vector<int>& rowStart, std::vector<std::vector<int>>& cols) {
  rowStart.assign(P + 1, 0);
  for (int r = 0; r < P; ++r) rowStart[r + 1] = rowStart[r] + ny / P + (r < ny % P ? 1 : 0);
  cols.assign(P, {});
  std::vector<int> load(P, 0);
  for (int s = 0; s <= L0 / 2; ++s) {
    const int partner = (L0 - s) % L0;
    if (partner < s) continue;
    const int size = partner == s ? 1 : 2;
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    cols[r].push_back(s);
    if (partner != s) cols[r].push_back(partner);
    load[r] += size;
  }
  for (auto& v : cols) std::sort(v.begin(), v.end());
}

namespace {

// All peers at once: t runs over the concatenated column lists (peer q's
// columns at t in [colsOffset[q], colsOffset[q+1])); tab[t] = {column s0,
// position j in q's list, q's column count, colsOffset[q]}. Peer q's block
// starts at rows * colsOffset[q] * B (the send offsets of the all-to-all).
//   gather:  dst[rows*base*B + (row*nq + j)*B + b] = src[row*rowLen + col*colStride + b]
//   scatter: the inverse map. (B = the chunk's batch entries, colStride =
//   the full batch of the grid layout.)
template <bool GATHER>
__global__ void permuteColumns(const double2* __restrict__ src, double2* __restrict__ dst, int rows, int L0,
                               const int4* __restrict__ tab, int B, long long rowLen, long long colStride) {
  const long long total = static_cast<long long>(rows) * L0 * B;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(q % B);
    const long long rt = q / B;
    const int t = static_cast<int>(rt % L0), row = static_cast<int>(rt / L0);
    const int4 e = tab[t];
    const long long packed = static_cast<long long>(rows) * e.w * B + (static_cast<long long>(row) * e.z + e.y) * B + b;
    const long long grid = row * rowLen + static_cast<long long>(e.x) * colStride + b;
    if (GATHER)
      dst[packed] = src[grid];
    else
      dst[grid] = src[packed];
  }
}

__global__ void addRows(double2* __restrict__ y, const double2* __restrict__ full, long long count) {
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < count;
       q += static_cast<long long>(gridDim.x) * blockDim.x)
    y[q] = cadd(y[q], full[q]);
}

int gridFor(long long n, int sms) { return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 16LL * sms))); }

}  // namespace

void distFree(Ctx& c) {
  for (void* p : {static_cast<void*>(c.dColsOfRank), static_cast<void*>(c.dColTab), static_cast<void*>(c.dTrow),
                  static_cast<void*>(c.dTcol),
                  static_cast<void*>(c.dSend), static_cast<void*>(c.dRecv), static_cast<void*>(c.dXhalo),
                  static_cast<void*>(c.dTermInfoLoc), static_cast<void*>(c.dTargetListLoc),
                  static_cast<void*>(c.dTargetPtrLoc), static_cast<void*>(c.dYcorrLoc)})
    if (p) cudaFree(p);
  c.dColsOfRank = nullptr;
  c.dColTab = nullptr;
  c.dTrow = c.dTcol = c.dSend = c.dRecv = c.dXhalo = c.dYcorrLoc = nullptr;
  c.dTermInfoLoc = c.dTargetListLoc = c.dTargetPtrLoc = nullptr;
  c.nTargetsLoc = c.maxTermsLoc = 0;
  c.distCorrReady = false;
  delete c.comm;
  c.comm = nullptr;
  for (cudaEvent_t& e : c.distEv)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  if (c.commStream) cudaStreamDestroy(c.commStream);
  c.commStream = nullptr;
}

// The correction terms whose target is one of this rank's elements
// (corrTermsByTarget, api.cu: the single-GPU term order per target), with
// sources re-indexed into the halo buffer dXhalo = x rows
// [myRow0 - 1, myRow0 + myRows] (rows outside the array unused) and
// targets into the local slab. Built on the first distributed apply.
void distCorrPrepare(Ctx& c) {
  if (c.distCorrReady) return;
  for (void* p : {static_cast<void*>(c.dTermInfoLoc), static_cast<void*>(c.dTargetListLoc),
                  static_cast<void*>(c.dTargetPtrLoc), static_cast<void*>(c.dYcorrLoc)})
    if (p) cudaFree(p);
  c.dTermInfoLoc = c.dTargetListLoc = c.dTargetPtrLoc = nullptr;
  c.dYcorrLoc = nullptr;
  const auto byTarget = corrTermsByTarget(c.nx, c.ny);
  const int r0 = c.myRow0, r1 = c.myRow0 + c.myRows;
  std::vector<int> info, targets, ptr{0};
  int maxTerms = 0;
  for (int e = r0 * c.nx; e < r1 * c.nx; ++e) {
    const auto& terms = byTarget[e];
    if (terms.empty()) continue;
    targets.push_back(e - r0 * c.nx);
    for (const auto& t : terms) {
      const int srow = t[1] / c.nx, scol = t[1] % c.nx;
      if (srow < r0 - 1 || srow > r1) throw Error{TBT_CUDA_ERROR, "distributed correction: source outside the halo"};
      info.insert(info.end(), {targets.back(), (srow - (r0 - 1)) * c.nx + scol, t[2], t[3]});
    }
    ptr.push_back(static_cast<int>(info.size() / 4));
    maxTerms = std::max(maxTerms, static_cast<int>(terms.size()));
  }
  c.nTargetsLoc = static_cast<int>(targets.size());
  c.maxTermsLoc = maxTerms;
  const size_t slab = static_cast<size_t>(c.myRows) * c.nx * c.maxNrhs * c.m;
  TBT_CUDA_CHECK(cudaMalloc(&c.dYcorrLoc, std::max<size_t>(1, slab) * sizeof(double2)));
  memsetSync(c.dYcorrLoc, 0, std::max<size_t>(1, slab) * sizeof(double2), c.stream);
  if (c.nTargetsLoc > 0) {
    TBT_CUDA_CHECK(cudaMalloc(&c.dTermInfoLoc, info.size() * sizeof(int)));
    TBT_CUDA_CHECK(cudaMalloc(&c.dTargetListLoc, targets.size() * sizeof(int)));
    TBT_CUDA_CHECK(cudaMalloc(&c.dTargetPtrLoc, ptr.size() * sizeof(int)));
    uploadSync(c.dTermInfoLoc, info.data(), info.size() * sizeof(int), c.stream);
    uploadSync(c.dTargetListLoc, targets.data(), targets.size() * sizeof(int), c.stream);
    uploadSync(c.dTargetPtrLoc, ptr.data(), ptr.size() * sizeof(int), c.stream);
  }
  c.distCorrReady = true;
}

namespace {
// With tbt_set_timing on, a distributed context times its NCCL exchanges
// (events on the context stream around each group; nothing overlaps them,
// so this is the exposed communication time) instead of the bin product.
template <class F>
void commSection(Ctx& c, F&& f) {
  if (!c.timeBinprod) {
    f();
    return;
  }
  if (c.tCount == static_cast<int>(c.tEvA.size())) {
    cudaEvent_t a, b;
    TBT_CUDA_CHECK(cudaEventCreate(&a));
    TBT_CUDA_CHECK(cudaEventCreate(&b));
    c.tEvA.push_back(a);
    c.tEvB.push_back(b);
  }
  TBT_CUDA_CHECK(cudaEventRecord(c.tEvA[c.tCount], c.stream));
  f();
  TBT_CUDA_CHECK(cudaEventRecord(c.tEvB[c.tCount], c.stream));
  ++c.tCount;
}
}  // namespace

void applyDist(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  const int P = c.nranks, me = c.myRank;
  const int B = nrhs * c.m;
  const int myCols = static_cast<int>(c.myColList.size());
  const int sms = smCount(c.device);
  cudaStream_t s = c.stream;
  // Exchanges overlap the transforms: the batch (basis x RHS) is cut into
  // nch chunks; chunk k's all-to-all runs on the comm stream while chunk
  // k+1 is row-transformed and packed (forward), and chunk k's inverse rows
  // run while chunk k+1 comes back. K3 needs every basis index of a bin, so
  // the chunks meet before it. Timed runs (tbt_set_timing) keep one chunk
  // on the compute stream so the exchange time is the exposed one.
  // TBT_DIST_CHUNKS=k forces k chunks (also with one rank; tests).
  static const int forced = [] {
    const char* e = getenv("TBT_DIST_CHUNKS");
    return e ? std::max(1, std::min(4, atoi(e))) : 0;
  }();
  // Default: two chunks only when this rank's exchange is large enough for
  // its transfer to outweigh the extra NCCL launch latency (>= 8 MB; one
  // rank measured +30% on C2, +4.5% on C4, +1.2% on C5 from the chunking
  // alone).
  const double xbytes = static_cast<double>(c.myRows) * c.L0 * B * sizeof(double2);
  int nch = (P > 1 && B >= 32 && xbytes >= 8.0 * (1 << 20)) ? 2 : 1;
  if (forced) nch = forced;
  if (c.timeBinprod || B % nch != 0) nch = 1;
  const int Bc = B / nch;
  cudaStream_t sc = nch > 1 ? c.commStream : s;

  auto rowFft = [&](int k) {  // 1. row FFTs (level 0) of the local rows -> dTrow[r][s0][b]
    FftPass fa;
    fa.in = x + static_cast<long long>(k) * Bc;
    fa.out = c.dTrow + static_cast<long long>(k) * Bc;
    fa.lines = c.myRows;
    fa.in_line_stride = static_cast<long long>(c.nx) * B;
    fa.in_point_stride = B;
    fa.out_line_stride = static_cast<long long>(c.L0) * B;
    fa.out_point_stride = B;
    fa.n = c.L0;
    fa.n_in = c.nx;
    fa.n_out = c.L0;
    fa.batch = Bc;
    fa.tw = c.dTw0;
    launchFftPass(fa, s);
  };
  // Chunk k's packed regions: send [q][row][j][b] at k * myRows*L0*Bc,
  // receive / dTcol [r][j][b] at k * ny*myCols*Bc.
  const long long sendChunk = static_cast<long long>(c.myRows) * c.L0 * Bc;
  const long long recvChunk = static_cast<long long>(c.ny) * myCols * Bc;
  auto sendOff = [&](int k, int q) { return k * sendChunk + static_cast<long long>(c.myRows) * c.colsOffset[q] * Bc; };
  auto recvOff = [&](int k, int q) {
    return k * recvChunk + static_cast<long long>(c.rowStart[q]) * myCols * Bc;
  };
  auto permute = [&](int k, bool gather) {
    const long long cnt = static_cast<long long>(c.myRows) * c.L0 * Bc;
    if (cnt == 0) return;
    double2* grid = c.dTrow + static_cast<long long>(k) * Bc;
    double2* packed = c.dSend + k * sendChunk;
    if (gather)
      permuteColumns<true><<<gridFor(cnt, sms), 256, 0, s>>>(grid, packed, c.myRows, c.L0, c.dColTab, Bc,
                                                             static_cast<long long>(c.L0) * B, B);
    else
      permuteColumns<false><<<gridFor(cnt, sms), 256, 0, s>>>(packed, grid, c.myRows, c.L0, c.dColTab, Bc,
                                                              static_cast<long long>(c.L0) * B, B);
    TBT_CUDA_CHECK(cudaGetLastError());
  };
  // 2. all-to-all of chunk k: my rows x columns of q -> rank q.
  auto exchangeFwd = [&](int k) {
    commSection(c, [&] {
      c.comm->groupStart();
      for (int q = 0; q < P; ++q) {
        const size_t scount = static_cast<size_t>(c.myRows) * c.colsOfRank[q].size() * Bc * 2;
        const size_t rcount = static_cast<size_t>(c.rowStart[q + 1] - c.rowStart[q]) * myCols * Bc * 2;
        if (scount) c.comm->send(c.dSend + sendOff(k, q), scount, q, sc);
        if (rcount) c.comm->recv(c.dRecv + recvOff(k, q), rcount, q, sc);
      }
      c.comm->groupEnd(sc);
    });
  };
  // 6. all-to-all back of chunk k: rows of rank q x my columns -> q.
  auto exchangeBack = [&](int k) {
    commSection(c, [&] {
      c.comm->groupStart();
      for (int q = 0; q < P; ++q) {
        const size_t scount = static_cast<size_t>(c.rowStart[q + 1] - c.rowStart[q]) * myCols * Bc * 2;
        const size_t rcount = static_cast<size_t>(c.myRows) * c.colsOfRank[q].size() * Bc * 2;
        if (scount) c.comm->send(c.dTcol + recvOff(k, q), scount, q, sc);
        if (rcount) c.comm->recv(c.dSend + sendOff(k, q), rcount, q, sc);
      }
      c.comm->groupEnd(sc);
    });
  };
  auto colFft = [&](int k, bool inverse) {  // 3. / 5. column FFTs of my columns
    FftPass f;
    const long long packed = k * recvChunk;
    if (!inverse) {  // received [r][j][bc] -> xhat[s1][j][b]
      f.in = c.dRecv + packed;
      f.out = c.dXhat + static_cast<long long>(k) * Bc;
      f.in_line_stride = Bc;
      f.in_point_stride = static_cast<long long>(myCols) * Bc;
      f.out_line_stride = B;
      f.out_point_stride = static_cast<long long>(myCols) * B;
      f.n_in = c.ny;
      f.n_out = c.L1;
      f.tw = c.dTw1;
    } else {  // yhat[s1][j][b] -> dTcol [r][j][bc], keep the ny element rows
      f.in = c.dYhat + static_cast<long long>(k) * Bc;
      f.out = c.dTcol + packed;
      f.in_line_stride = B;
      f.in_point_stride = static_cast<long long>(myCols) * B;
      f.out_line_stride = Bc;
      f.out_point_stride = static_cast<long long>(myCols) * Bc;
      f.n_in = c.L1;
      f.n_out = c.ny;
      f.inverse = 1;
      f.tw = c.dTw1;
    }
    f.lines = myCols;
    f.n = c.L1;
    f.batch = Bc;
    launchFftPass(f, s);
  };
  auto rowFftInv = [&](int k) {  // 7. inverse row FFTs, keep nx points, 1/L -> y slab
    FftPass ia;
    ia.in = c.dTrow + static_cast<long long>(k) * Bc;
    ia.out = y + static_cast<long long>(k) * Bc;
    ia.lines = c.myRows;
    ia.in_line_stride = static_cast<long long>(c.L0) * B;
    ia.in_point_stride = B;
    ia.out_line_stride = static_cast<long long>(c.nx) * B;
    ia.out_point_stride = B;
    ia.n = c.L0;
    ia.n_in = c.L0;
    ia.n_out = c.nx;
    ia.batch = Bc;
    ia.inverse = 1;
    ia.scale = 1.0 / static_cast<double>(c.L);
    ia.tw = c.dTw0;
    launchFftPass(ia, s);
  };
  auto handOff = [&](cudaStream_t from, cudaStream_t to, int ev) {
    if (from == to) return;
    TBT_CUDA_CHECK(cudaEventRecord(c.distEv[ev], from));
    TBT_CUDA_CHECK(cudaStreamWaitEvent(to, c.distEv[ev], 0));
  };

  // Events: 0-3 pack done (k), 4-7 received (k); reused for the inverse
  // (same stream order, so a reused event is never waited on stale).
  // Forward: rows + pack of chunk k+1 overlap the exchange of chunk k.
  for (int k = 0; k < nch; ++k) {
    rowFft(k);
    permute(k, true);
    handOff(s, sc, k);
    exchangeFwd(k);
  }
  for (int k = 0; k < nch; ++k) {
    handOff(sc, s, 4 + k);
    colFft(k, false);
  }
  // 4. Bin-pair products on the local pairs (every basis index of a bin).
  if (c.npairs > 0) launchBinProduct(c, nrhs);
  // Inverse: the exchange back of chunk k overlaps the inverse columns of
  // chunk k+1, then the inverse rows of chunk k the exchange of chunk k+1.
  for (int k = 0; k < nch; ++k) {
    colFft(k, true);
    handOff(s, sc, k);
    exchangeBack(k);
  }
  for (int k = 0; k < nch; ++k) {
    handOff(sc, s, 4 + k);
    permute(k, false);
    rowFftInv(k);
  }

  // 8. Spatial terms: K (element-local) and the correction. A correction
  //    term couples an element with its 4-neighbours only, so one halo row
  //    from each slab neighbour suffices: dXhalo = [row r0-1][my rows][row
  //    r1] (every rank owns >= 1 row, tbt_dist_init checks nranks <= ny).
  launchAntisym(c, x, y, nrhs, c.myRows * c.nx);
  if (withCorr && c.haveCorr && c.nTerms > 0) {
    distCorrPrepare(c);
    const long long rowLen = static_cast<long long>(c.nx) * B;
    const long long mine = static_cast<long long>(c.myRows) * rowLen;
    TBT_CUDA_CHECK(cudaMemcpyAsync(c.dXhalo + rowLen, x, mine * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    if (P > 1) {
      commSection(c, [&] {
        c.comm->groupStart();
        const size_t n = static_cast<size_t>(rowLen) * 2;
        if (me > 0) {
          c.comm->send(x, n, me - 1, s);
          c.comm->recv(c.dXhalo, n, me - 1, s);
        }
        if (me < P - 1) {
          c.comm->send(x + mine - rowLen, n, me + 1, s);
          c.comm->recv(c.dXhalo + rowLen + mine, n, me + 1, s);
        }
        c.comm->groupEnd(s);
      });
    }
    if (c.nTargetsLoc > 0) {
      CorrTables t{c.dTermInfoLoc, c.dTargetListLoc, c.dTargetPtrLoc, c.nTargetsLoc, c.maxTermsLoc};
      launchCorrVectorOn(c, t, c.dXhalo, c.dYcorrLoc, nrhs, s);
    }
    addRows<<<gridFor(mine, sms), 256, 0, s>>>(y, c.dYcorrLoc, mine);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace tbt
