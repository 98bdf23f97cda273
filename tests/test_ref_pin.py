"""Pins the CPU oracle to the reference ITSELF.

oracle/_ref/libref_linsolve.so is the reference's own src/linsolve.cpp,
toeplitz.cpp, fft.cpp (+ mesh / array_model / partition) compiled unchanged
against a functional Eigen-subset shim (oracle/eigen_shim, oracle/Makefile).
Every case writes a ZTOE1 block cache with the test-side writer, lets the
reference read it with its own loadBlockCache (toeplitz.cpp:754-815) and
compares its ToeplitzMatvec / gmres / iterativeSolve / schurSolve /
denseSolve with the oracle restatement (oracle/oracle.cpp) on the same data.

The committed fixtures tests/golden/ref_pin.npz (made by
tests/golden/make_ref_golden.py from the same library) keep the pin where
the library is absent."""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import CONFIGS, ToeplitzRep, gen, read_ztoe1
from paper_2506_04710_b200.toeplitz import Margin
from ztoe1_writer import assemble_c, random_c_records, write_ztoe1, write_ztoe1_dense

GOLDEN = Path(__file__).resolve().parent / "golden" / "ref_pin.npz"

needs_ref = pytest.mark.skipif(oracle.ref_linsolve() is None,
                               reason="oracle/_ref/libref_linsolve.so not built (reference tree absent)")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def random_blocks(nx, ny, m, seed):
    """Arbitrary canonical blocks (non-symmetric self block included)."""
    rng = np.random.default_rng(seed)
    nb = nx * ny + (nx - 1) * (ny - 1)
    g = rng.standard_normal((nb, m, m)) + 1j * rng.standard_normal((nb, m, m))
    g[0] += (3 + 3j) * np.eye(m)
    return np.ascontiguousarray(g)


def a_only_case(tmp_path, nx, ny, m, g):
    e = [0] * 9
    e[4] = m
    path = tmp_path / f"a_{nx}_{ny}_{m}.ztoe1"
    write_ztoe1(str(path), nx, ny, e, g)
    return oracle.RefOperator(path), oracle.Oracle(nx, ny, m, g)


def margin_case(tmp_path, nx, ny, m, e, seed=4):
    rng = np.random.default_rng(seed)
    g = gen.blocks_raw(nx, ny, m, seed)
    mg = gen.margin(nx, ny, e, seed + 3)
    recs = random_c_records(nx, ny, e, rng)
    path = tmp_path / f"m_{nx}_{ny}_{m}.ztoe1"
    write_ztoe1(str(path), nx, ny, e, g, mg, recs)
    C = assemble_c(nx, ny, e, recs)
    margin = Margin(list(e), mg.bside, mg.brow, mg.bcorner, np.asfortranarray(C).ravel(order="F"))
    return oracle.RefOperator(path), oracle.Oracle.from_rep(ToeplitzRep(nx, ny, m, g, None, margin)), path


A_SHAPES = [(4, 4, 24, "gen"), (5, 3, 4, "rand"), (1, 6, 3, "rand"), (7, 1, 2, "rand"), (3, 3, 8, "rand"),
            (2, 5, 5, "rand"), (1, 1, 3, "rand"), (9, 6, 7, "gen")]


@needs_ref
@pytest.mark.parametrize("nx,ny,m,kind", A_SHAPES)
def test_apply_a_matches_reference(tmp_path, nx, ny, m, kind):
    g = gen.blocks_raw(nx, ny, m, 11) if kind == "gen" else random_blocks(nx, ny, m, nx * 100 + ny * 10 + m)
    R, O = a_only_case(tmp_path, nx, ny, m, g)
    X = gen.rhs_normal(nx * ny * m, 3, 7)
    for c in range(3):
        x = np.ascontiguousarray(X[:, c])
        yr, yo = R.applyA(x), O.applyA(x)
        assert rel(yo, yr) <= 1e-14, (nx, ny, m, rel(yo, yr))
        assert np.array_equal(R.apply(x), yr)  # nM = 0: apply == applyA (linsolve.cpp:380-383)
    assert np.array_equal(R.diagonal(), O.diagonal())


@needs_ref
def test_dense_reconstruction_matches_reference(tmp_path):
    """reconstructFull (toeplitz.cpp:514-532) vs the oracle's dense A."""
    g = random_blocks(3, 4, 5, 9)
    R, O = a_only_case(tmp_path, 3, 4, 5, g)
    assert np.array_equal(R.dense(), O.dense())


@needs_ref
@pytest.mark.parametrize("name,max_iter", [("C1", 2000), ("C2", 60)])
def test_gmres_matches_reference(tmp_path, name, max_iter):
    """The reference's own gmres (linsolve.cpp:425-515): C1 to convergence,
    C2 over a budget (it stalls): identical iteration and
    operator-application counts, same solution and final residual."""
    cfg = CONFIGS[name]
    g = gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed)
    R, O = a_only_case(tmp_path, cfg.nx, cfg.ny, cfg.m, g)
    b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    r = R.gmres(b, tol=cfg.tol, max_iter=max_iter, restart=cfg.restart)
    o = O.gmres(b, tol=cfg.tol, max_iter=max_iter, restart=cfg.restart)
    assert r["iterations"] == o["iterations"][0]
    assert r["converged"] == bool(o["converged"][0])
    assert rel(o["x"], r["x"]) <= 1e-12
    assert abs(r["residual"] - o["residual"][0]) <= 1e-12 * max(r["residual"], 1e-300) + 1e-15
    # one application per inner iteration + one per restart cycle (+ the final check)
    assert r["matvecs"] >= r["iterations"]


@needs_ref
def test_iterative_solve_matches_reference(tmp_path):
    """iterativeSolve (linsolve.cpp:551-593) over 3 columns, 2 threads."""
    cfg = CONFIGS["C1"]
    g = gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed)
    R, O = a_only_case(tmp_path, cfg.nx, cfg.ny, cfg.m, g)
    V = gen.rhs_normal(cfg.n, 3, 21)
    r = R.solve("iterative", V, tol=1e-8, restart=30, threads=2)
    o = O.gmres(V, tol=1e-8, max_iter=2000, restart=30)
    assert r["iterations"] == o["iterations"]
    assert rel(o["x"], r["x"]) <= 1e-12
    d = R.solve("dense", V)
    assert rel(d["x"], r["x"]) < 1e-7


@needs_ref
def test_nonconvergence_is_numeric_error(tmp_path):
    """The reference throws NumericError for an unconverged column (:591)."""
    cfg = CONFIGS["C1"]
    R, _ = a_only_case(tmp_path, cfg.nx, cfg.ny, cfg.m, gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed))
    with pytest.raises(oracle.RefError) as ei:
        R.solve("iterative", gen.rhs_normal(cfg.n, 1, 2), tol=1e-12, max_iter=5, restart=30)
    assert ei.value.status == 2 and "did not converge" in str(ei.value)


MARGIN_SHAPES = [(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]), (3, 2, 5, [0, 2, 1, 0, 5, 3, 0, 1, 2]),
                 (1, 3, 5, [1, 2, 1, 2, 5, 2, 1, 2, 1]), (5, 4, 8, [0, 2, 0, 3, 8, 1, 0, 2, 1])]


@needs_ref
@pytest.mark.parametrize("nx,ny,m,e", MARGIN_SHAPES)
def test_margin_operator_matches_reference(tmp_path, nx, ny, m, e):
    """apply / applyB / applyBT / applyC / diagonal with margin parts
    (linsolve.cpp:54-134, 292-408): Toe1D spectra, corners, C blocks."""
    R, O, _ = margin_case(tmp_path, nx, ny, m, e)
    assert (R.nA, R.n) == (O.nA, O.n)
    x = gen.rhs_normal(R.n, 1, 5)[:, 0]
    assert rel(O.apply(x), R.apply(x)) <= 1e-14
    assert rel(O.applyA(x[:R.nA]), R.applyA(x[:R.nA])) <= 1e-14
    assert np.array_equal(R.diagonal(), O.diagonal())
    # the reference's own edge offsets (buildArray order) are the C-ABI layout
    es = R.edge_start()
    assert es[nx * ny] == R.nA and es[nx * ny - 1] == R.nA - m


@needs_ref
def test_margin_gmres_and_schur_match_reference(tmp_path):
    nx, ny, m, e = 4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]
    R, O, _ = margin_case(tmp_path, nx, ny, m, e)
    b = gen.rhs_normal(R.n, 1, 9)[:, 0]
    r = R.gmres(b, tol=1e-8, max_iter=300, restart=30)
    o = O.gmres(b, tol=1e-8, max_iter=300, restart=30)
    assert r["iterations"] == o["iterations"][0]
    assert rel(o["x"], r["x"]) <= 1e-12
    # schurSolve needs excitations that vanish on margin rows (:603-604)
    V = np.zeros((R.n, 2), complex)
    V[:R.nA] = gen.rhs_normal(R.nA, 2, 10)
    rs = R.solve("schur", V, tol=1e-10, restart=30)
    os_ = O.schur(V, tol=1e-10, restart=30)
    assert rs["iterations"] == os_["iterations"]
    assert rel(os_["x"], rs["x"]) <= 1e-10
    with pytest.raises(oracle.RefError) as ei:
        R.solve("schur", gen.rhs_normal(R.n, 1, 3))
    assert ei.value.status == 1


@needs_ref
def test_ztoe1_written_by_reference_parses(tmp_path):
    """The product's ZTOE1 reader (csrc/io.cu, host only) on a file the
    reference's own saveBlockCache wrote (toeplitz.cpp:701-752)."""
    nx, ny, m, e = 3, 2, 5, [0, 2, 1, 0, 5, 3, 0, 1, 2]
    R, O, src = margin_case(tmp_path, nx, ny, m, e)
    out = tmp_path / "by_reference.ztoe1"
    R.save(out)
    mine = read_ztoe1(str(src))
    theirs = read_ztoe1(str(out))
    assert np.array_equal(mine.generators, theirs.generators)
    for k in ("bside", "brow", "bcorner", "c"):
        assert np.array_equal(getattr(mine.margin, k), getattr(theirs.margin, k))


@needs_ref
def test_semisparse_and_full_modes(tmp_path):
    """The reference's SemiSparse (aLevel1 + dense B, C) and Full storage
    modes give the same operator as Sparse on the same matrix."""
    nx, ny, m, e = 3, 3, 4, [1, 2, 1, 2, 4, 1, 1, 2, 1]
    R, O, _ = margin_case(tmp_path, nx, ny, m, e)
    Z = R.dense()
    nA, n = R.nA, R.n
    # aLevel1[i] = block row of element row i+1 against element row 1
    a1 = [Z[i * nx * m:(i + 1) * nx * m, 0:nx * m] for i in range(ny)]
    semi = tmp_path / "semi.ztoe1"
    write_ztoe1_dense(str(semi), nx, ny, e, 1, a_level1=a1, b_full=Z[nA:, :nA], c_full=Z[nA:, nA:])
    full = tmp_path / "full.ztoe1"
    write_ztoe1_dense(str(full), nx, ny, e, 0, z_full=Z)
    x = gen.rhs_normal(n, 1, 6)[:, 0]
    y = R.apply(x)
    for p in (semi, full):
        Rm = oracle.RefOperator(p)
        assert rel(Rm.apply(x), y) <= 1e-14
        assert np.array_equal(Rm.diagonal(), R.diagonal())


def test_golden_reference_outputs():
    """Oracle vs outputs of the reference library committed as fixtures
    (tests/golden/make_ref_golden.py): runs without the library."""
    z = np.load(GOLDEN)
    cfg = CONFIGS["C1"]
    g = gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed)
    O = oracle.Oracle(cfg.nx, cfg.ny, cfg.m, g)
    assert rel(O.applyA(z["c1_x"]), z["c1_y"]) <= 1e-14
    assert np.array_equal(O.diagonal(), z["c1_diag"])
    o = O.gmres(z["c1_b"], tol=cfg.tol, max_iter=2000, restart=cfg.restart)
    assert o["iterations"][0] == int(z["c1_gmres_iterations"])
    assert rel(o["x"], z["c1_gmres_x"]) <= 1e-12
    # a random-block shape with a non-symmetric self block
    gr = random_blocks(5, 3, 4, 534)
    Or = oracle.Oracle(5, 3, 4, gr)
    assert rel(Or.applyA(z["r_x"]), z["r_y"]) <= 1e-14


# ---- the CUDA path against the reference itself (through the C ABI)

@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_gpu_matches_reference(gpu, tmp_path, name):
    from paper_2506_04710_b200 import SolverOptions, ToeplitzMatvec
    cfg = CONFIGS[name]
    g = gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed)
    R, _ = a_only_case(tmp_path, cfg.nx, cfg.ny, cfg.m, g)
    op = ToeplitzMatvec.from_ztoe1(str(tmp_path / f"a_{cfg.nx}_{cfg.ny}_{cfg.m}.ztoe1"))
    x = gen.rhs_normal(cfg.n, 1, 17)[:, 0]
    assert rel(op.apply(x), R.applyA(x)) <= 1e-11
    assert np.array_equal(op.diagonal(), R.diagonal())
    b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    budget = 2000 if name == "C1" else 60
    r = R.gmres(b, tol=cfg.tol, max_iter=budget, restart=cfg.restart)
    res = op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=budget, restart=cfg.restart), raise_on_fail=False)
    assert res.iterations[0] == r["iterations"]
    assert res.matvecs == r["matvecs"]
    # operator applications are counted by the solver, not inferred from the history
    res0 = op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=budget, restart=cfg.restart), raise_on_fail=False,
                    hist_cap=0)
    assert res0.matvecs == r["matvecs"] and res0.iterations == res.iterations
    assert rel(res.current[:, 0] if res.current.ndim == 2 else res.current, r["x"]) <= 1e-8


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,e", MARGIN_SHAPES[:2])
def test_gpu_margin_matches_reference(gpu, tmp_path, nx, ny, m, e):
    from paper_2506_04710_b200 import ToeplitzMatvec
    R, _, path = margin_case(tmp_path, nx, ny, m, e)
    op = ToeplitzMatvec.from_ztoe1(str(path))
    x = gen.rhs_normal(R.n, 1, 5)[:, 0]
    assert rel(op.apply(x), R.apply(x)) <= 1e-11
    assert rel(op.applyB(x[:R.nA]), R.applyB(x[:R.nA])) <= 1e-11
    assert rel(op.applyBT(x[R.nA:]), R.applyBT(x[R.nA:])) <= 1e-11
    assert rel(op.applyC(x[R.nA:]), R.applyC(x[R.nA:])) <= 1e-11
    assert np.array_equal(op.diagonal(), R.diagonal())
