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
//    The edge/corner correction needs neighbour rows: x is all-gathered
//    (P2P sends of each rank's slab) and each rank adds its rows of it.
// Replaces applyA / apply (proj/src/linsolve.cpp:260-290,373-388), which has
// no distributed counterpart ("Non-goals: distributed").
#include <dlfcn.h>

#include <algorithm>
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

// dst[(row * nsel + j) * B + b] = src[row * srcRow + col[j] * B + b]
__global__ void gatherColumns(const double2* __restrict__ src, double2* __restrict__ dst, int rows, int nsel,
                              const int* __restrict__ col, int B, long long srcRow) {
  const long long total = static_cast<long long>(rows) * nsel * B;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(q % B);
    const long long rj = q / B;
    const int j = static_cast<int>(rj % nsel), row = static_cast<int>(rj / nsel);
    dst[q] = src[row * srcRow + static_cast<long long>(col[j]) * B + b];
  }
}

// dst[row * dstRow + col[j] * B + b] = src[(row * nsel + j) * B + b]
__global__ void scatterColumns(const double2* __restrict__ src, double2* __restrict__ dst, int rows, int nsel,
                               const int* __restrict__ col, int B, long long dstRow) {
  const long long total = static_cast<long long>(rows) * nsel * B;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(q % B);
    const long long rj = q / B;
    const int j = static_cast<int>(rj % nsel), row = static_cast<int>(rj / nsel);
    dst[row * dstRow + static_cast<long long>(col[j]) * B + b] = src[q];
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
  for (void* p : {static_cast<void*>(c.dColsOfRank), static_cast<void*>(c.dTrow), static_cast<void*>(c.dTcol),
                  static_cast<void*>(c.dSend), static_cast<void*>(c.dRecv), static_cast<void*>(c.dXfull)})
    if (p) cudaFree(p);
  c.dColsOfRank = nullptr;
  c.dTrow = c.dTcol = c.dSend = c.dRecv = c.dXfull = nullptr;
  if (c.comm) nccl().commDestroy(c.comm);
  c.comm = nullptr;
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
  const int* myColDev = c.dColsOfRank + c.colsOffset[me];

  // 1. Row FFTs (level 0) of the local rows -> dTrow[r][s0][b].
  FftPass fa;
  fa.in = x;
  fa.out = c.dTrow;
  fa.lines = c.myRows;
  fa.in_line_stride = static_cast<long long>(c.nx) * B;
  fa.in_point_stride = B;
  fa.out_line_stride = static_cast<long long>(c.L0) * B;
  fa.out_point_stride = B;
  fa.n = c.L0;
  fa.n_in = c.nx;
  fa.n_out = c.L0;
  fa.batch = B;
  fa.tw = c.dTw0;
  launchFftPass(fa, s);

  // 2. All-to-all: my rows x columns of q  ->  rank q.
  long long off = 0;
  std::vector<long long> sendOff(P + 1, 0), recvOff(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    const int nq = static_cast<int>(c.colsOfRank[q].size());
    const long long cnt = static_cast<long long>(c.myRows) * nq * B;
    if (cnt > 0)
      gatherColumns<<<gridFor(cnt, sms), 256, 0, s>>>(c.dTrow, c.dSend + off, c.myRows, nq,
                                                        c.dColsOfRank + c.colsOffset[q], B,
                                                        static_cast<long long>(c.L0) * B);
    off += cnt;
    sendOff[q + 1] = off;
    recvOff[q + 1] = recvOff[q] + static_cast<long long>(c.rowStart[q + 1] - c.rowStart[q]) * myCols * B;
  }
  TBT_CUDA_CHECK(cudaGetLastError());
  commSection(c, [&] {
    TBT_NCCL_CHECK(nccl().groupStart());
    for (int q = 0; q < P; ++q) {
      const size_t sc = static_cast<size_t>(sendOff[q + 1] - sendOff[q]) * 2;
      const size_t rc = static_cast<size_t>(recvOff[q + 1] - recvOff[q]) * 2;
      if (sc) TBT_NCCL_CHECK(nccl().send(c.dSend + sendOff[q], sc, ncclDouble, q, c.comm, s));
      if (rc) TBT_NCCL_CHECK(nccl().recv(c.dRecv + recvOff[q], rc, ncclDouble, q, c.comm, s));
    }
    TBT_NCCL_CHECK(nccl().groupEnd());
  });
  // Received blocks are [rows of q][my columns][b] in row order: exactly
  // dTcol[r][j][b] for r = 0..ny-1 (rank slabs are contiguous and ordered).
  const double2* tcol = c.dRecv;

  // 3. Column FFTs (level 1) of my columns -> xhat_local[s1][j][b].
  FftPass fb;
  fb.in = tcol;
  fb.out = c.dXhat;
  fb.lines = myCols;
  fb.in_line_stride = B;
  fb.in_point_stride = static_cast<long long>(myCols) * B;
  fb.out_line_stride = B;
  fb.out_point_stride = static_cast<long long>(myCols) * B;
  fb.n = c.L1;
  fb.n_in = c.ny;
  fb.n_out = c.L1;
  fb.batch = B;
  fb.tw = c.dTw1;
  launchFftPass(fb, s);

  // 4. Bin-pair products on the local pairs.
  if (c.npairs > 0) launchBinProduct(c, nrhs);

  // 5. Inverse column FFTs, keep the ny element rows -> dTcol[r][j][b].
  FftPass ib;
  ib.in = c.dYhat;
  ib.out = c.dTcol;
  ib.lines = myCols;
  ib.in_line_stride = B;
  ib.in_point_stride = static_cast<long long>(myCols) * B;
  ib.out_line_stride = B;
  ib.out_point_stride = static_cast<long long>(myCols) * B;
  ib.n = c.L1;
  ib.n_in = c.L1;
  ib.n_out = c.ny;
  ib.batch = B;
  ib.inverse = 1;
  ib.tw = c.dTw1;
  launchFftPass(ib, s);

  // 6. All-to-all back: rows of rank q x my columns -> q; from q: my rows x
  //    columns of q.
  commSection(c, [&] {
    TBT_NCCL_CHECK(nccl().groupStart());
    for (int q = 0; q < P; ++q) {
      const long long rows = c.rowStart[q + 1] - c.rowStart[q];
      const size_t sc = static_cast<size_t>(rows) * myCols * B * 2;
      const size_t rc = static_cast<size_t>(c.myRows) * c.colsOfRank[q].size() * B * 2;
      if (sc)
        TBT_NCCL_CHECK(nccl().send(c.dTcol + static_cast<long long>(c.rowStart[q]) * myCols * B, sc, ncclDouble, q,
                                c.comm, s));
      if (rc) TBT_NCCL_CHECK(nccl().recv(c.dSend + sendOff[q], rc, ncclDouble, q, c.comm, s));
    }
    TBT_NCCL_CHECK(nccl().groupEnd());
  });
  for (int q = 0; q < P; ++q) {
    const int nq = static_cast<int>(c.colsOfRank[q].size());
    const long long cnt = static_cast<long long>(c.myRows) * nq * B;
    if (cnt > 0)
      scatterColumns<<<gridFor(cnt, sms), 256, 0, s>>>(c.dSend + sendOff[q], c.dTrow, c.myRows, nq,
                                                         c.dColsOfRank + c.colsOffset[q], B,
                                                         static_cast<long long>(c.L0) * B);
  }
  TBT_CUDA_CHECK(cudaGetLastError());

  // 7. Inverse row FFTs of my rows, keep nx points, 1/L -> y (local slab).
  FftPass ia;
  ia.in = c.dTrow;
  ia.out = y;
  ia.lines = c.myRows;
  ia.in_line_stride = static_cast<long long>(c.L0) * B;
  ia.in_point_stride = B;
  ia.out_line_stride = static_cast<long long>(c.nx) * B;
  ia.out_point_stride = B;
  ia.n = c.L0;
  ia.n_in = c.L0;
  ia.n_out = c.nx;
  ia.batch = B;
  ia.inverse = 1;
  ia.scale = 1.0 / static_cast<double>(c.L);
  ia.tw = c.dTw0;
  launchFftPass(ia, s);

  // 8. Spatial terms: K (element-local) and the correction (needs x of the
  //    neighbouring rows: all-gather the slabs, then add my rows).
  launchAntisym(c, x, y, nrhs, c.myRows * c.nx);
  if (withCorr && c.haveCorr && c.nTerms > 0) {
    commSection(c, [&] {
      TBT_NCCL_CHECK(nccl().groupStart());
      const size_t mine = static_cast<size_t>(c.myRows) * c.nx * B * 2;
      for (int q = 0; q < P; ++q) {
        const size_t rc = static_cast<size_t>(c.rowStart[q + 1] - c.rowStart[q]) * c.nx * B * 2;
        if (mine) TBT_NCCL_CHECK(nccl().send(x, mine, ncclDouble, q, c.comm, s));
        if (rc)
          TBT_NCCL_CHECK(nccl().recv(c.dXfull + static_cast<long long>(c.rowStart[q]) * c.nx * B, rc, ncclDouble, q,
                                  c.comm, s));
      }
      TBT_NCCL_CHECK(nccl().groupEnd());
    });
    launchCorrVector(c, c.dXfull, c.dYcorr, nrhs, s);
    const long long cnt = static_cast<long long>(c.myRows) * c.nx * B;
    addRows<<<gridFor(cnt, sms), 256, 0, s>>>(y, c.dYcorr + static_cast<long long>(c.myRow0) * c.nx * B, cnt);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace tbt
