// tbt.hpp - header-only C++ mirror of the reference's operator / solver API
// (proj/include/arraymom/linsolve.hpp:40-95) over the C ABI of tbt.h.
// A reference caller swaps `arraymom::ToeplitzMatvec` for `tbt::ToeplitzMatvec`
// and `arraymom::iterativeSolve` for `tbt::iterativeSolve`.
#pragma once

#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tbt.h"

namespace tbt {

using Complex = std::complex<double>;  // common.hpp:28
using Vector = std::vector<Complex>;

struct UserError : std::runtime_error {  // common.hpp:40-43
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {  // common.hpp:47-50
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(tbt_status s) {
  if (s == TBT_OK) return;
  const std::string msg = tbt_last_error();
  if (s == TBT_USER_ERROR) throw UserError(msg);
  if (s == TBT_NUMERIC_ERROR) throw NumericError(msg);
  throw DeviceError(msg);
}

struct SolverOptions {  // linsolve.hpp:47-53
  double tol = 1e-8;
  int maxIter = 2000;
  int restart = 60;
  bool precondition = true;
  int threads = 1;  // columns run in lockstep on the device
};

struct SolveResult {  // linsolve.hpp:40-45
  std::vector<Vector> current;  // one vector per column
  std::vector<double> residual;
  std::vector<int> iterations;
  std::string solver = "gmres";
};

// ToeplitzMatvec (linsolve.hpp:59-77). Generators: ToeplitzRep::aGen in the
// Sparse order (toeplitz.hpp:72-74), each m x m column-major.
class ToeplitzMatvec {
 public:
  ToeplitzMatvec(int nx, int ny, int m, const std::vector<Complex>& generators, int maxNrhs = 1,
                 int device = 0) {
    tbt_desc d{nx, ny, m, maxNrhs, device, 0};
    check(tbt_create(&d, &ctx_));
    const long long nb = static_cast<long long>(nx) * ny + static_cast<long long>(nx - 1) * (ny - 1);
    if (static_cast<long long>(generators.size()) != nb * m * m) {
      tbt_destroy(ctx_);
      throw UserError("ToeplitzMatvec: generator count mismatch");
    }
    check(tbt_set_generators(ctx_, reinterpret_cast<const double*>(generators.data()), nb));
  }
  ~ToeplitzMatvec() { tbt_destroy(ctx_); }
  ToeplitzMatvec(const ToeplitzMatvec&) = delete;
  ToeplitzMatvec& operator=(const ToeplitzMatvec&) = delete;

  // Optional edge/corner terms (tbt_gen.h layout), then the spectra.
  void setCorrection(int rank, const Complex* d, const Complex* u, const Complex* v) {
    check(tbt_set_correction(ctx_, rank, reinterpret_cast<const double*>(d), reinterpret_cast<const double*>(u),
                             reinterpret_cast<const double*>(v)));
  }
  // Margin coupling B / B^T / C (ToeplitzRep::bSideGen, bRowGen, bCorner
  // and the margin blocks; layouts in tbt_gen.h). apply / diagonal /
  // iterativeSolve then act on sizeA() + sizeM() unknowns.
  void setMargin(const int e[9], const Complex* bSide, const Complex* bRow, const Complex* bCorner,
                 const Complex* c) {
    check(tbt_set_margin(ctx_, e, reinterpret_cast<const double*>(bSide), reinterpret_cast<const double*>(bRow),
                         reinterpret_cast<const double*>(bCorner), reinterpret_cast<const double*>(c)));
  }
  void precompute() { check(tbt_precompute(ctx_)); }

  Vector apply(const Vector& x) const { return run(tbt_apply, x, size()); }     // linsolve.hpp:64
  Vector applyA(const Vector& x) const { return run(tbt_apply_a, x, sizeA()); } // linsolve.hpp:65
  Vector applyB(const Vector& xA) const { return run(tbt_apply_b, xA, sizeA(), sizeM()); }   // linsolve.hpp:66
  Vector applyBT(const Vector& xM) const { return run(tbt_apply_bt, xM, sizeM(), sizeA()); } // linsolve.hpp:67
  Vector applyC(const Vector& xM) const { return run(tbt_apply_c, xM, sizeM(), sizeM()); }   // linsolve.hpp:68
  // Many independent applies on host vectors, copies overlapped with the
  // applies (tbt_apply_many; the reference runs them one column per thread,
  // linsolve.cpp:572). Each vector must have length size().
  std::vector<Vector> applyMany(const std::vector<Vector>& xs) const {
    const long n = sizeA();
    std::vector<Complex> xb(static_cast<size_t>(n) * xs.size()), yb(xb.size());
    for (size_t i = 0; i < xs.size(); ++i) {
      if (static_cast<long>(xs[i].size()) != n) throw UserError("applyMany: vector length mismatch");
      std::copy(xs[i].begin(), xs[i].end(), xb.begin() + static_cast<long>(i) * n);
    }
    check(tbt_apply_many(ctx_, reinterpret_cast<const double*>(xb.data()), reinterpret_cast<double*>(yb.data()),
                         static_cast<long long>(xs.size())));
    std::vector<Vector> ys;
    for (size_t i = 0; i < xs.size(); ++i)
      ys.emplace_back(yb.begin() + static_cast<long>(i) * n, yb.begin() + static_cast<long>(i + 1) * n);
    return ys;
  }
  Vector diagonal() const {                                                      // linsolve.hpp:69
    Vector d(static_cast<size_t>(size()));
    check(tbt_diagonal(ctx_, reinterpret_cast<double*>(d.data())));
    return d;
  }
  long sizeA() const { return static_cast<long>(tbt_size_a(ctx_)); }
  long sizeM() const { return static_cast<long>(tbt_size_m(ctx_)); }
  long size() const { return sizeA() + sizeM(); }
  tbt_ctx* handle() const { return ctx_; }

 private:
  using Fn = tbt_status (*)(tbt_ctx*, const double*, double*, int, int);
  Vector run(Fn fn, const Vector& x, long n, long nOut = -1) const {
    if (static_cast<long>(x.size()) != n) throw UserError("matvec: vector length mismatch");
    Vector y(static_cast<size_t>(nOut < 0 ? n : nOut));
    check(fn(ctx_, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data()), 1, TBT_HOST));
    return y;
  }
  tbt_ctx* ctx_ = nullptr;
};

namespace detail {
using SolveFn = tbt_status (*)(tbt_ctx*, const double*, double*, int, const tbt_gmres_opts*, tbt_gmres_stats*, int);
inline SolveResult solveColumns(SolveFn fn, ToeplitzMatvec& op, const std::vector<Vector>& V,
                                const SolverOptions& opt) {
  const int p = static_cast<int>(V.size());
  const long n = op.size();
  std::vector<Complex> b(static_cast<size_t>(n) * p), x(b.size());
  for (int c = 0; c < p; ++c) {
    if (static_cast<long>(V[c].size()) != n) throw UserError("solve: excitation length mismatch");
    std::copy(V[c].begin(), V[c].end(), b.begin() + static_cast<long>(c) * n);
  }
  tbt_gmres_opts o{opt.tol, opt.maxIter, opt.restart, opt.precondition ? 1 : 0, 0, 0, 1};
  std::vector<int> its(p), conv(p), hlen(p);
  std::vector<double> res(p);
  tbt_gmres_stats st{its.data(), res.data(), conv.data(), nullptr, hlen.data(), 0};
  const tbt_status s =
      fn(op.handle(), reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(x.data()), p, &o, &st,
         TBT_HOST);
  SolveResult out;
  for (int c = 0; c < p; ++c)
    out.current.emplace_back(x.begin() + static_cast<long>(c) * n, x.begin() + static_cast<long>(c + 1) * n);
  out.residual = res;
  out.iterations = its;
  check(s);
  return out;
}
}  // namespace detail

// iterativeSolve (linsolve.hpp:88-89): columns of V, throws NumericError if
// any column did not converge (linsolve.cpp:591).
inline SolveResult iterativeSolve(ToeplitzMatvec& op, const std::vector<Vector>& V, const SolverOptions& opt) {
  return detail::solveColumns(tbt_gmres, op, V, opt);
}

// schurSolve (linsolve.hpp:93-95, linsolve.cpp:595-682): V vanishes on the
// margin rows; NumericError on an unconverged inner solve or a singular S.
inline SolveResult schurSolve(ToeplitzMatvec& op, const std::vector<Vector>& V, const SolverOptions& opt) {
  return detail::solveColumns(tbt_schur_solve, op, V, opt);
}

// toeplitzMatvec (linsolve.hpp:80-81): one-shot apply.
inline Vector toeplitzMatvec(ToeplitzMatvec& op, const Vector& x) { return op.apply(x); }

}  // namespace tbt
