// Drives the C++ mirror include/tbt.hpp the way a reference caller would
// (tbt::ToeplitzMatvec / tbt::iterativeSolve in place of arraymom's),
// linked against the product library: config C1 generators from tbt_gen.h,
// one apply (also through applyMany) and one GMRES(30) solve. Writes x, A x and the solution as raw
// complex128 to argv[1] for tests/test_abi.py to check against the oracle.
// Without a usable device the constructor throws tbt::DeviceError: the demo
// prints "no device" and exits 0 (there is no CPU fallback).
#include <cstdio>
#include <fstream>

#include "tbt.hpp"
#include "tbt_gen.h"

int main(int argc, char** argv) {
  const int nx = 4, ny = 4, m = 24;
  const long long nb = tbtgen_num_blocks(nx, ny);
  std::vector<tbt::Complex> gen(static_cast<size_t>(nb) * m * m);
  tbtgen_blocks(nx, ny, m, 0, reinterpret_cast<double*>(gen.data()), 0);
  try {
    tbt::ToeplitzMatvec op(nx, ny, m, gen);
    op.precompute();
    tbt::Vector x(static_cast<size_t>(op.size()));
    tbtgen_rhs_normal(op.size(), 1, 42, reinterpret_cast<double*>(x.data()));
    const tbt::Vector y = op.apply(x);
    const std::vector<tbt::Vector> ys = op.applyMany({x, y, x});
    if (ys.size() != 3 || ys[0] != y || ys[2] != y) {
      std::printf("applyMany mismatch\n");
      return 1;
    }
    tbt::SolverOptions opt;
    opt.restart = 30;
    const tbt::SolveResult r = tbt::iterativeSolve(op, {x}, opt);
    std::ofstream out(argc > 1 ? argv[1] : "mirror_demo.bin", std::ios::binary);
    const tbt::Vector* outs[3] = {&x, &y, &r.current[0]};
    for (const tbt::Vector* v : outs)
      out.write(reinterpret_cast<const char*>(v->data()), static_cast<std::streamsize>(v->size() * 16));
    std::printf("ok %d iterations residual %.3e\n", r.iterations[0], r.residual[0]);
  } catch (const tbt::DeviceError& e) {
    std::printf("no device: %s\n", e.what());
  }
  return 0;
}
