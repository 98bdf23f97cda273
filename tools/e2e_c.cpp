// e2e floor without Python: tbt_apply on pinned host buffers in a C++ loop
// (C2 by default), plus the per-call split.
//   g++ -O2 -std=c++17 -I include tools/e2e_c.cpp -L paper_2506_04710_b200 -ltbt \
//       -Wl,-rpath,$PWD/paper_2506_04710_b200 -L/usr/local/cuda/lib64 -lcudart -o tools/e2e_c
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tbt.h"
#include "tbt_gen.h"

int main(int argc, char** argv) {
  const int nx = 32, ny = 32, m = 64, rank = 8;
  const long long nb = tbtgen_num_blocks(nx, ny);
  std::vector<double> gen(static_cast<size_t>(nb) * m * m * 2);
  tbtgen_blocks(nx, ny, m, 2, gen.data(), 0);
  std::vector<double> d(40 * m * 2), u(40 * m * rank * 2), v(u.size());
  tbtgen_correction(m, rank, 2, 0.1, d.data(), u.data(), v.data());
  tbt_desc desc{nx, ny, m, 1, 0, 0};
  tbt_ctx* ctx = nullptr;
  if (tbt_create(&desc, &ctx) || tbt_set_generators(ctx, gen.data(), nb) ||
      tbt_set_correction(ctx, rank, d.data(), u.data(), v.data()) || tbt_precompute(ctx)) {
    std::printf("setup failed: %s\n", tbt_last_error());
    return 1;
  }
  const long long n = tbt_size_a(ctx);
  double *x = nullptr, *y = nullptr;
  cudaMallocHost(&x, n * 16);
  cudaMallocHost(&y, n * 16);
  tbtgen_rhs_normal(n, 1, 3, x);
  for (int i = 0; i < 20; ++i) tbt_apply(ctx, x, y, 1, TBT_HOST);
  const int iters = argc > 1 ? std::atoi(argv[1]) : 2000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) tbt_apply(ctx, x, y, 1, TBT_HOST);
  auto t1 = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
  std::printf("C2 e2e tbt_apply (pinned, C++ loop): %.1f us per call, %.0f matvec/s\n", us, 1e6 / us);
  tbt_destroy(ctx);
  return 0;
}
