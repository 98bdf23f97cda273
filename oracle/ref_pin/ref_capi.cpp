// C entry points into the reference's OWN operator and solvers, compiled
// unchanged from /root/reference/proj/src/{linsolve,toeplitz,mesh,
// array_model,fft}.cpp against the functional Eigen-subset shim
// (oracle/eigen_shim) by oracle/Makefile into oracle/_ref/libref_linsolve.so.
//
// TEST INFRASTRUCTURE ONLY. It pins the CPU oracle (oracle/oracle.cpp) and the
// ZTOE1 parser of the product to reference outputs (tests/test_ref_pin.py,
// golden fixtures tests/golden/ref_c1.npz), and bench.py --impl reference
// times its applyA. Nothing on the product path links or loads it.
//
// linsolve.cpp is #included (not compiled separately) so that this unit can
// call its file-local restarted GMRES (`gmres`, linsolve.cpp:425-515)
// directly: the public iterativeSolve discards the partial solution when a
// column does not converge (:582-591), and the BASELINE configs C2-C5 do not
// converge within the budgets the tests use.
#include "src/linsolve.cpp"

#include <atomic>
#include <cstring>
#include <memory>
#include <string>

namespace arraymom {

// The EFIE kernel (src/kernel.cpp) is outside the pinned path: representations
// come from ZTOE1 files, never from a mesh. assemble()/assembleDenseParts()
// reach these two symbols and fail loudly if called.
void KernelParams::validate() const {
  throw UserError("ref pin: EFIE assembly (kernel.cpp) is not part of the pinned path");
}
ImpedanceBlock computeBlock(const DesignatedData&, const DesignatedData&, const Vec3&, const Vec3&,
                            const std::vector<std::pair<int, int>>&, const KernelParams&, int) {
  throw UserError("ref pin: EFIE assembly (kernel.cpp) is not part of the pinned path");
}

}  // namespace arraymom

namespace {

using arraymom::ArrayModel;
using arraymom::Complex;
using arraymom::MatrixXc;
using arraymom::ToeplitzMatvec;
using arraymom::ToeplitzRep;
using arraymom::VectorXc;

thread_local std::string g_err;

struct RefOp {
  ToeplitzRep rep;
  ArrayModel model;
  std::unique_ptr<ToeplitzMatvec> mv;
};

// The part layout of buildArray (array_model.cpp:207-234) without its mesh
// conformity checks: parts in component order 5,2,8,6,4,3,9,1,7, row-major
// bottom-left first; edgeStart accumulates partEdgeCount. The components
// carry e[c] placeholder edges each (only the counts matter on this path).
ArrayModel modelFor(const ToeplitzRep& rep) {
  ArrayModel m;
  const int nx = rep.nx, ny = rep.ny;
  m.nx = nx;
  m.ny = ny;
  m.comps.dx = 1.0;
  m.comps.dy = 1.0;
  for (int c = 1; c <= 9; ++c) {
    auto& d = m.comps.comps[c - 1];
    for (int k = 1; k <= rep.e[c - 1]; ++k) d.globalEdges.push_back(k);
  }
  const int pn = nx * ny + 2 * nx + 2 * ny + 4;
  m.offsets.resize(3, pn);
  m.partTable.resize(3, pn);
  int p = 0;
  auto place = [&](int row, int col, int comp) {
    m.offsets.col(p) = arraymom::Vec3(static_cast<double>(col), static_cast<double>(row), 0.0);
    m.partTable(0, p) = row;
    m.partTable(1, p) = col;
    m.partTable(2, p) = comp;
    ++p;
  };
  for (int r = 1; r <= ny; ++r)
    for (int c = 1; c <= nx; ++c) place(r, c, 5);
  for (int r = 1; r <= ny; ++r) place(r, 0, 2);
  for (int r = 1; r <= ny; ++r) place(r, nx + 1, 8);
  for (int c = 1; c <= nx; ++c) place(ny + 1, c, 6);
  for (int c = 1; c <= nx; ++c) place(0, c, 4);
  place(ny + 1, 0, 3);
  place(ny + 1, nx + 1, 9);
  place(0, 0, 1);
  place(0, nx + 1, 7);
  m.edgeStart.resize(pn);
  long acc = 0;
  for (int q = 1; q <= pn; ++q) {
    m.edgeStart[q - 1] = acc;
    acc += m.partEdgeCount(q);
  }
  return m;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const arraymom::UserError& e) {
    g_err = e.what();
    return 1;
  } catch (const arraymom::NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

VectorXc toVec(const double* p, long n) {
  VectorXc v(n);
  std::memcpy(static_cast<void*>(v.data()), p, sizeof(Complex) * static_cast<size_t>(n));
  return v;
}
void fromMat(const MatrixXc& m, double* out) {
  std::memcpy(out, m.data(), sizeof(Complex) * static_cast<size_t>(m.size()));
}
MatrixXc toMat(const double* p, long rows, long cols) {
  MatrixXc m(rows, cols);
  std::memcpy(static_cast<void*>(m.data()), p, sizeof(Complex) * static_cast<size_t>(rows * cols));
  return m;
}

}  // namespace

extern "C" {

const char* refp_last_error() { return g_err.c_str(); }

// loadBlockCache (toeplitz.cpp:754-815) + the array model + ToeplitzMatvec
// (linsolve.cpp:352-353: spectra, Toe1D margin spectra, C block cache).
int refp_load(const char* path, void** out) {
  return guarded([&] {
    auto op = std::make_unique<RefOp>();
    op->rep = arraymom::loadBlockCache(path);
    op->model = modelFor(op->rep);
    op->mv = std::make_unique<ToeplitzMatvec>(op->rep, op->model);
    *out = op.release();
  });
}

int refp_save(void* h, const char* path) {
  return guarded([&] { arraymom::saveBlockCache(static_cast<RefOp*>(h)->rep, path); });
}

void refp_destroy(void* h) { delete static_cast<RefOp*>(h); }

int refp_sizes(void* h, long long* nA, long long* nM, int* mode) {
  auto* op = static_cast<RefOp*>(h);
  *nA = op->mv->sizeA();
  *nM = op->mv->sizeM();
  *mode = static_cast<int>(op->rep.mode);
  return 0;
}

int refp_edge_start(void* h, long long* out) {
  auto* op = static_cast<RefOp*>(h);
  for (size_t p = 0; p < op->model.edgeStart.size(); ++p) out[p] = op->model.edgeStart[p];
  return static_cast<int>(op->model.edgeStart.size());
}

// which: 0 apply (linsolve.cpp:373-388), 1 applyA (:260-290), 2 applyB
// (:292-314), 3 applyBT (:316-334), 4 applyC (:336-349).
int refp_apply(void* h, int which, const double* x, double* y) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    const long nA = op->mv->sizeA(), nM = op->mv->sizeM();
    VectorXc r;
    switch (which) {
      case 0: r = op->mv->apply(toVec(x, nA + nM)); break;
      case 1: r = op->mv->applyA(toVec(x, nA)); break;
      case 2: r = op->mv->applyB(toVec(x, nA)); break;
      case 3: r = op->mv->applyBT(toVec(x, nM)); break;
      case 4: r = op->mv->applyC(toVec(x, nM)); break;
      default: throw arraymom::UserError("refp_apply: bad selector");
    }
    fromMat(r, y);
  });
}

// Column-wise applyA over ncols vectors with up to `threads` workers, one
// column per task (parallelFor, mesh.cpp:27-53): the CPU arm of the bench.
int refp_apply_a_cols(void* h, const double* x, double* y, int ncols, int threads) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    const long nA = op->mv->sizeA();
    arraymom::parallelFor(ncols, threads, [&](long lo, long hi) {
      for (long c = lo; c < hi; ++c) {
        const VectorXc r = op->mv->applyA(toVec(x + 2 * nA * c, nA));
        fromMat(r, y + 2 * nA * c);
      }
    });
  });
}

int refp_diagonal(void* h, double* d) {
  return guarded([&] { fromMat(static_cast<RefOp*>(h)->mv->diagonal(), d); });
}

// One restarted GMRES solve through the reference's own gmres()
// (linsolve.cpp:425-515) with the Jacobi preconditioner of iterativeSolve
// (:556-563) or, a_only = 1, schurSolve's element-block one on applyA
// (:605-611, :640-647). Returns x, iterations, final true residual,
// convergence and the operator applications counted through the plug-in.
int refp_gmres(void* h, const double* b, double* x, int a_only, int precondition, double tol, int max_iter,
               int restart, int* iterations, double* residual, int* converged, long long* matvecs) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    const long nA = op->mv->sizeA(), nM = op->mv->sizeM();
    const long n = a_only ? nA : nA + nM;
    VectorXc invDiag;
    if (precondition) {
      const VectorXc d = op->mv->diagonal();
      invDiag = VectorXc(n);
      for (long i = 0; i < n; ++i) invDiag(i) = (std::abs(d(i)) > 0.0) ? 1.0 / d(i) : Complex{1.0, 0.0};
    }
    std::atomic<long long> count{0};
    const auto fn = [&](const VectorXc& v) -> VectorXc {
      ++count;
      return a_only ? op->mv->applyA(v) : op->mv->apply(v);
    };
    VectorXc xv;
    const arraymom::GmresOutcome res =
        arraymom::gmres(fn, toVec(b, n), xv, precondition ? &invDiag : nullptr, tol, max_iter, restart);
    fromMat(xv, x);
    *iterations = res.iterations;
    *residual = res.residual;
    *converged = res.converged ? 1 : 0;
    *matvecs = count.load();
  });
}

// The public solvers (linsolve.cpp:532-682). V, X: n x p column-major.
// kind: 0 iterativeSolve, 1 schurSolve, 2 denseSolve. On NumericError the
// status is 2 and X is untouched (the reference discards partial results).
int refp_solve(void* h, int kind, const double* V, int p, double tol, int max_iter, int restart, int precondition,
               int threads, double* X, int* iterations, double* residual) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    const long n = op->mv->sizeA() + op->mv->sizeM();
    arraymom::ExcitationSet ex;
    ex.v = toMat(V, n, p);
    arraymom::SolverOptions opt;
    opt.tol = tol;
    opt.maxIter = max_iter;
    opt.restart = restart;
    opt.precondition = precondition != 0;
    opt.threads = threads;
    arraymom::SolveResult r;
    if (kind == 0)
      r = arraymom::iterativeSolve(op->rep, op->model, ex, opt);
    else if (kind == 1)
      r = arraymom::schurSolve(op->rep, op->model, ex, opt);
    else
      r = arraymom::denseSolve(op->rep, op->model, ex);
    fromMat(r.current, X);
    for (int c = 0; c < p; ++c) {
      iterations[c] = r.iterations[static_cast<size_t>(c)];
      residual[c] = r.residual[static_cast<size_t>(c)];
    }
  });
}

// reconstructFull (toeplitz.cpp:514-532): the dense part-ordered matrix.
int refp_reconstruct_full(void* h, double* z) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    fromMat(arraymom::reconstructFull(op->rep, op->model).z, z);
  });
}

// buildExcitation (linsolve.cpp:28-50): the feed rows of the given ports.
int refp_excitation(void* h, int feed_local_edge, const int* ports, int nports, long long* rows) {
  return guarded([&] {
    auto* op = static_cast<RefOp*>(h);
    const arraymom::ExcitationSet ex =
        arraymom::buildExcitation(op->model, feed_local_edge, std::vector<int>(ports, ports + nports));
    for (int c = 0; c < nports; ++c) rows[c] = ex.feedRows[static_cast<size_t>(c)];
  });
}

}  // extern "C"
