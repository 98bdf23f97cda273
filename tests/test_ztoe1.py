"""Row f3: reference ZTOE1 block caches (saveBlockCache format,
proj/src/toeplitz.cpp:700-815) and the persisted spectrum.

CPU: the loader (csrc/io.cu, tbt_ztoe1_read) against the test-side writer
and an independent restatement of partBlock's C assembly
(tests/ztoe1_writer.py); malformed files raise user errors. GPU: an operator
built straight from a ZTOE1 file against the oracle, and a TBTS1 spectrum
round trip."""
import os

import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import Config, ToeplitzRep, UserError, gen, read_ztoe1
from ztoe1_writer import assemble_c, random_c_records, write_ztoe1

CASES = [(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]), (3, 2, 5, [0, 2, 1, 0, 5, 3, 0, 1, 2]), (2, 2, 4, [0] * 4 + [4] + [0] * 4)]


def make_file(tmp_path, nx, ny, m, e, seed=1):
    rng = np.random.default_rng(seed)
    g = gen.blocks_raw(nx, ny, m, seed)
    mg = gen.margin(nx, ny, e, seed + 3)
    recs = random_c_records(nx, ny, e, rng)
    path = str(tmp_path / f"rep_{nx}_{ny}_{m}.ztoe1")
    write_ztoe1(path, nx, ny, e, g, mg, recs)
    C = assemble_c(nx, ny, e, recs)
    return path, g, mg, C


@pytest.mark.parametrize("nx,ny,m,e", CASES)
def test_ztoe1_parse(tmp_path, nx, ny, m, e):
    path, g, mg, C = make_file(tmp_path, nx, ny, m, e)
    rep = read_ztoe1(path)
    assert (rep.nx, rep.ny, rep.m) == (nx, ny, m)
    assert np.array_equal(rep.generators, g)
    if mg.size(nx, ny) == 0:
        assert rep.margin is None
        return
    assert rep.margin.e == e
    assert np.array_equal(rep.margin.bside, mg.bside)
    assert np.array_equal(rep.margin.brow, mg.brow)
    assert np.array_equal(rep.margin.bcorner, mg.bcorner)
    nM = mg.size(nx, ny)
    assert np.array_equal(rep.margin.c.reshape(nM, nM).T, C)  # column-major in the ABI


def test_ztoe1_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.ztoe1"
    p.write_bytes(b"NOPE!" + bytes(60))
    with pytest.raises(UserError):
        read_ztoe1(str(p))
    path, *_ = make_file(tmp_path, 3, 2, 5, [0, 2, 1, 0, 5, 3, 0, 1, 2])
    data = open(path, "rb").read()
    short = tmp_path / "short.ztoe1"
    short.write_bytes(data[:len(data) // 2])
    with pytest.raises(UserError):
        read_ztoe1(str(short))
    semi = bytearray(data)
    semi[5] = 1  # SemiSparse mode
    other = tmp_path / "semi.ztoe1"
    other.write_bytes(bytes(semi))
    with pytest.raises(UserError):
        read_ztoe1(str(other))


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,e", CASES)
def test_gpu_from_ztoe1(gpu, tmp_path, nx, ny, m, e):
    from paper_2506_04710_b200 import ToeplitzMatvec
    from paper_2506_04710_b200.toeplitz import Margin
    path, g, mg, C = make_file(tmp_path, nx, ny, m, e)
    op = ToeplitzMatvec.from_ztoe1(path, max_nrhs=2)
    nM = mg.size(nx, ny)
    margin = Margin(e, mg.bside, mg.brow, mg.bcorner, np.asfortranarray(C).ravel(order="F")) if nM else None
    o = oracle.Oracle.from_rep(ToeplitzRep(nx, ny, m, g, None, margin))
    assert op.size() == o.n
    X = gen.rhs_normal(o.n, 2, 3)
    Y = op.apply(X)
    for c in range(2):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert np.linalg.norm(Y[:, c] - ref) / np.linalg.norm(ref) < 1e-11


@pytest.mark.gpu
def test_gpu_spectra_cache_roundtrip(gpu, tmp_path):
    from paper_2506_04710_b200 import ToeplitzMatvec
    rep = ToeplitzRep.synthetic(Config("sc", 6, 5, 16, 1, 4, 2, "normal", 20))
    cache = str(tmp_path / "spec.tbts")
    op1 = ToeplitzMatvec(rep, spectra_cache=cache)  # K1, then written
    assert os.path.exists(cache)
    op2 = ToeplitzMatvec(rep, spectra_cache=cache)  # loaded, K1 skipped
    x = gen.rhs_normal(op1.size(), 1, 8)[:, 0]
    assert np.array_equal(op1.apply(x), op2.apply(x))
    assert np.array_equal(op1.diagonal(), op2.diagonal())
    o = oracle.Oracle.from_rep(rep)
    assert np.linalg.norm(op2.apply(x) - o.apply(x)) / np.linalg.norm(o.apply(x)) < 1e-11
    other = ToeplitzRep.synthetic(Config("sc", 5, 5, 16, 1, 4, 2, "normal", 20))
    with pytest.raises(UserError):
        ToeplitzMatvec(other, spectra_cache=cache)
    # same shape, other generators (another sweep frequency / seed): rejected by the key
    reseeded = ToeplitzRep.synthetic(Config("sc", 6, 5, 16, 1, 4, 9, "normal", 20))
    with pytest.raises(UserError, match="generator key"):
        ToeplitzMatvec(reseeded, spectra_cache=cache)
