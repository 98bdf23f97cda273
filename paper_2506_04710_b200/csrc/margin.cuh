// Margin operator state shared by margin.cu (B / B^T / C apply) and
// schur.cu (the Schur-complement driver).
#pragma once

#include <vector>

#include "tbt_internal.cuh"

namespace tbt {

struct MarginOp {
  int e[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long nM = 0;
  int Ly = 1, Lx = 1;
  int emSide[2] = {0, 0}, emRow[2] = {0, 0}, emCorner[4] = {0, 0, 0, 0};
  long long sideStart[2] = {0, 0}, rowStart[2] = {0, 0}, cornerStart[4] = {0, 0, 0, 0};
  double2* gSide[2] = {nullptr, nullptr};  // [Ly][em][nx*m]
  double2* gRow[2] = {nullptr, nullptr};   // [ny][Lx][em][m]
  double2* rawSide[2] = {nullptr, nullptr};  // uploaded generators (tbt_gen.h layout), kept for schur.cu
  double2* rawRow[2] = {nullptr, nullptr};
  double2* corner[4] = {nullptr, nullptr, nullptr, nullptr};  // [em][nA] row-major
  double2* C = nullptr;                    // [nM][nM] row-major
  // SemiSparse representations (reference bFull, toeplitz.hpp:90-93): B is
  // one dense nM x nA matrix applied by dense products (linsolve.cpp:294,
  // 318); no Toeplitz / corner regions then.
  double2* bDense = nullptr;               // [nM][nA] row-major
  double2* twY = nullptr;
  double2* twX = nullptr;
  std::vector<double2> diag;               // C's diagonal (host)
  // Work buffers for max_nrhs columns.
  double2 *xs = nullptr, *ys = nullptr;        // [nM][K]
  double2 *hatY = nullptr, *hatZy = nullptr;   // [Ly][nx][K][m]
  double2 *hatX = nullptr, *hatZx = nullptr;   // [Lx][ny][K][m]
  double2* hatMs[2] = {nullptr, nullptr};       // [Ly][em][K]
  double2* hatMr[2] = {nullptr, nullptr};       // [Lx][em][K]
  double2 *zA = nullptr, *zA2 = nullptr;       // [ne][K][m]
  double2* cornerPart = nullptr;               // [corner rows][K][element blocks]
  // Single-column fused path (B and B^T from one read of every array).
  double2* hatMsOut[2] = {nullptr, nullptr};    // [Ly][em]
  double2* hatMrOut[2] = {nullptr, nullptr};    // [Lx][em]
  double2 *bpartS = nullptr, *bpartR = nullptr; // B partials per (bin, row, chunk)
  double2* cornerT = nullptr;                   // [passes][nA] B^T corner contribution
  double2* ysC = nullptr;                       // [nM] C xM (one column)
  int chunkS = 1, chunkR = 1;                   // q-chunks per bin
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;
  // Side / row branches of the single-column apply run beside the corner
  // branch on the ctx stream (forked and joined with events).
  cudaStream_t branch[2] = {nullptr, nullptr};
  cudaEvent_t evFork = nullptr, evJoin[2] = {nullptr, nullptr};

  double2* alloc(size_t count) {
    void* p = nullptr;
    TBT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double2)));
    if (poisonBuffers()) memsetSync(p, 0xFF, std::max<size_t>(count, 1) * sizeof(double2), stream);
    allocs.push_back(p);
    return static_cast<double2*>(p);
  }
  ~MarginOp() {
    for (void* p : allocs) cudaFree(p);
    for (int b = 0; b < 2; ++b) {
      if (branch[b]) cudaStreamDestroy(branch[b]);
      if (evJoin[b]) cudaEventDestroy(evJoin[b]);
    }
    if (evFork) cudaEventDestroy(evFork);
  }
  bool anySide() const { return emSide[0] + emSide[1] > 0; }
  bool anyRow() const { return emRow[0] + emRow[1] > 0; }
};


}  // namespace tbt
