"""The seeded generator (include/tbt_gen.h): deterministic, thread-invariant,
the reference's canonical block order/count, BASELINE's distribution."""
import numpy as np
import pytest

from paper_2506_04710_b200 import gen


def test_block_count_and_order():
    assert gen.num_blocks(4, 6) == 39  # SPEC.md acceptance 3 / PAPER section II-C
    assert gen.num_blocks(1, 1) == 1
    nx, ny = 4, 3
    shifts = [gen.block_shift(nx, ny, t) for t in range(gen.num_blocks(nx, ny))]
    # toeplitz.cpp:305-312: i = 0..ny-1, j from (i==0 ? 0 : 1-nx) to nx-1
    want = [(0, j) for j in range(nx)] + [(i, j) for i in range(1, ny) for j in range(1 - nx, nx)]
    assert shifts == want
    with pytest.raises(IndexError):
        gen.block_shift(nx, ny, len(want))


def test_deterministic_and_thread_invariant():
    a = gen.blocks_raw(5, 4, 7, 3, nthreads=1)
    b = gen.blocks_raw(5, 4, 7, 3, nthreads=8)
    assert np.array_equal(a, b)
    c = gen.blocks_raw(5, 4, 7, 4, nthreads=1)
    assert not np.array_equal(a, c)


def test_block_structure_and_distribution():
    nx, ny, m = 8, 8, 32
    raw = gen.blocks_raw(nx, ny, m, 0)
    z0 = raw[0].T
    assert np.array_equal(z0, z0.T)  # reciprocal self block
    assert np.allclose(np.diag(z0) - (2 + 2j), np.diag(z0 - (2 + 2j) * np.eye(m)))
    # entries exp(-j pi R)/(1+R) (u + j v)/sqrt(m): |.|^2 averages 2/(m (1+R)^2)
    for t in [1, 5, 20, 60]:
        i, j = gen.block_shift(nx, ny, t)
        R = np.hypot(i, j)
        blk = raw[t]
        ms = np.mean(np.abs(blk) ** 2) * m * (1 + R) ** 2
        assert 1.6 < ms < 2.4, (t, ms)
        # common phase exp(-j pi R) times a zero-mean complex normal
        w = np.exp(-1j * np.pi * R) / (1 + R)
        u = (blk / w * np.sqrt(m)).ravel()
        assert abs(np.mean(u.real)) < 0.15 and abs(np.mean(u.imag)) < 0.15
        assert 0.8 < np.var(u.real) < 1.2 and 0.8 < np.var(u.imag) < 1.2


def test_correction_shapes_and_scale():
    d, u, v = gen.correction(16, 4, 1, 0.1)
    assert d.shape == (40, 16) and u.shape == (40, 4, 16) and v.shape == (40, 4, 16)
    assert 0.05 < np.sqrt(np.mean(np.abs(d) ** 2)) < 0.15
    d2, u2, v2 = gen.correction(16, 4, 1, 0.1)
    assert np.array_equal(d, d2) and np.array_equal(u, u2)


def test_rhs_kinds():
    x = gen.rhs_delta_steered(32, 32, 64, 2)
    assert np.count_nonzero(x) == 32 * 32
    per = x.reshape(32, 32, 64)
    assert np.all(np.count_nonzero(per, axis=2) == 1)
    c = 5
    assert np.allclose(per[3, c][per[3, c] != 0], np.exp(-1j * np.pi * c * 0.5))
    V, rows = gen.rhs_ports(3, 2, 4, 9)
    assert V.shape == (24, 6) and np.array_equal(np.nonzero(V)[0], rows)
    assert np.all(rows // 4 == np.arange(6))
    N = gen.rhs_normal(100, 3, 1)
    assert N.shape == (100, 3)


def test_components():
    # array_model.hpp:26-29 numbering, bottom-left = 1, top-right = 9
    assert [gen.component(4, 3, 0, c) for c in range(4)] == [1, 4, 4, 7]
    assert [gen.component(4, 3, 1, c) for c in range(4)] == [2, 5, 5, 8]
    assert [gen.component(4, 3, 2, c) for c in range(4)] == [3, 6, 6, 9]


def test_block_lines_match_blocks():
    """tbtgen_block_lines (row a / column a of every canonical block) draws
    the same values as tbtgen_blocks; oracle.sampled_apply builds on it."""
    nx, ny, m = 4, 3, 5
    g = gen.blocks(nx, ny, m, 9)  # [t, a, b]
    for a in range(m):
        rows, cols = gen.block_lines(nx, ny, m, 9, a)
        assert np.array_equal(rows, g[:, a, :]) and np.array_equal(cols, g[:, :, a])


def test_sampled_apply_matches_full_apply():
    import oracle
    nx, ny, m = 5, 4, 6
    o = oracle.Oracle(nx, ny, m, gen.blocks_raw(nx, ny, m, 3))
    x = gen.rhs_normal(nx * ny * m, 1, 4)[:, 0]
    y = o.applyA(x).reshape(nx * ny, m)
    ys, tf, tr = oracle.sampled_apply(nx, ny, m, 3, [0, 4, 5], x)
    assert np.array_equal(ys, y[:, [0, 4, 5]].T) and tf >= 0 and tr >= 0
