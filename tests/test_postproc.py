"""Row f4: port network and far-field contractions (proj/src/postproc.cpp).

CPU: the oracle's restatement against independent numpy formulas. GPU: the
device kernels through the C ABI against the oracle, on C3-like shapes
(18 x 9 array, 162 ports) and with margin parts."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import Config, ToeplitzRep, UserError, gen, tarc


def numpy_port_network(cur, feed, length, z0):
    I = cur[feed, :]
    Y = I / length / length
    Z = np.linalg.inv(Y)
    Z0 = np.diag(z0)
    core = (Z - Z0) @ np.linalg.inv(Z + Z0)
    S = core * np.sqrt(z0[None, :] / z0[:, None])
    return Y, Z, S


def numpy_farfield(nx, ny, e, tensors, dirs, dx, dy, k, eta, cur, W):
    parts = [(5, (c - 1) * dx, (r - 1) * dy) for r in range(1, ny + 1) for c in range(1, nx + 1)]
    parts += [(2, 0.0, (r - 1) * dy) for r in range(1, ny + 1)] + [(8, (nx - 1) * dx, (r - 1) * dy) for r in range(1, ny + 1)]
    parts += [(6, (c - 1) * dx, (ny - 1) * dy) for c in range(1, nx + 1)] + [(4, (c - 1) * dx, 0.0) for c in range(1, nx + 1)]
    parts += [(3, 0.0, (ny - 1) * dy), (9, (nx - 1) * dx, (ny - 1) * dy), (1, 0.0, 0.0), (7, (nx - 1) * dx, 0.0)]
    comb = cur @ W
    co = np.zeros((len(dirs), W.shape[1]), complex)
    cx = np.zeros_like(co)
    row = 0
    for comp, ox, oy in parts:
        n = e[comp - 1]
        if n:
            seg = comb[row:row + n]
            ph = np.exp(1j * k * (dirs[:, 0] * ox + dirs[:, 1] * oy))[:, None]
            co += ph * (tensors[comp - 1][0] @ seg)
            cx += ph * (tensors[comp - 1][1] @ seg)
        row += n
    return -1j * k * eta * co, -1j * k * eta * cx


def synth(nx, ny, e, ndir, p, seed=0):
    rng = np.random.default_rng(seed)
    ntot = nx * ny * e[4] + ny * (e[1] + e[7]) + nx * (e[5] + e[3]) + e[2] + e[8] + e[0] + e[6]
    cn = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    tensors = [(cn(ndir, e[c]), cn(ndir, e[c])) if e[c] else None for c in range(9)]
    d = rng.standard_normal((ndir, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return tensors, d, cn(ntot, p), ntot


@pytest.mark.parametrize("p", [1, 5, 24])
def test_oracle_port_network_vs_numpy(p):
    rng = np.random.default_rng(p)
    n = 200
    cur = rng.standard_normal((n, p)) + 1j * rng.standard_normal((n, p))
    feed = rng.choice(n, p, replace=False)
    z0 = rng.uniform(25, 75, p)
    r = oracle.port_network(cur, feed, 0.01, z0)
    Y, Z, S = numpy_port_network(cur, feed, 0.01, z0)
    for a, b in ((r["y"], Y), (r["z"], Z), (r["s"], S)):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-10
    with pytest.raises(ArithmeticError):
        oracle.port_network(np.zeros((n, p), complex), feed, 0.01, z0)


@pytest.mark.parametrize("nx,ny,e", [(3, 2, [0, 0, 0, 0, 4, 0, 0, 0, 0]), (4, 3, [2, 3, 1, 4, 6, 2, 3, 5, 1])])
def test_oracle_farfield_vs_numpy(nx, ny, e):
    tensors, d, cur, ntot = synth(nx, ny, e, 17, 3)
    W = np.eye(3)
    co, cx = oracle.array_farfield(nx, ny, e, tensors, d, 0.5, 0.7, 2.1, 376.7, cur, W)
    rco, rcx = numpy_farfield(nx, ny, e, tensors, d, 0.5, 0.7, 2.1, 376.7, cur, W)
    assert np.linalg.norm(co - rco) / np.linalg.norm(rco) < 1e-12
    assert np.linalg.norm(cx - rcx) / np.linalg.norm(rcx) < 1e-12


def test_tarc():
    s = np.array([[0.1, 0.2j], [0.2j, 0.3]])
    a = np.array([1.0, 1j])
    assert abs(tarc(s, a) - np.linalg.norm(s @ a) / np.linalg.norm(a)) < 1e-15
    with pytest.raises(UserError):
        tarc(s, np.zeros(2))


@pytest.mark.gpu
@pytest.mark.parametrize("p", [3, 162])
def test_gpu_port_network(gpu, p):
    from paper_2506_04710_b200 import ToeplitzMatvec, port_network
    rep = ToeplitzRep.synthetic(Config("pn", 18, 9, 8, 1, 4, 1, "normal", 20))
    op = ToeplitzMatvec(rep)
    rng = np.random.default_rng(p)
    n = op.size()
    cur = rng.standard_normal((n, p)) + 1j * rng.standard_normal((n, p))
    feed = np.sort(rng.choice(n, p, replace=False))
    z0 = rng.uniform(25, 75, p)
    g = port_network(op, cur, feed, 0.02, z0)
    r = oracle.port_network(cur, feed, 0.02, z0)
    for key in ("y", "z", "s"):
        assert np.linalg.norm(g[key] - r[key]) / np.linalg.norm(r[key]) < 1e-10, key


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,e,q", [(18, 9, [0, 0, 0, 0, 16, 0, 0, 0, 0], 1),
                                       (18, 9, [0, 0, 0, 0, 16, 0, 0, 0, 0], 162),
                                       (4, 3, [2, 3, 1, 4, 6, 2, 3, 5, 1], 5)])
def test_gpu_farfield(gpu, nx, ny, e, q):
    from paper_2506_04710_b200 import ToeplitzMatvec, array_farfield
    rep = ToeplitzRep.synthetic(Config("ff", nx, ny, e[4], 1, 4, 1, "normal", 20))
    if sum(e) != e[4]:
        rep.margin = gen.margin(nx, ny, e, 3)
    op = ToeplitzMatvec(rep)
    tensors, d, cur, ntot = synth(nx, ny, e, 41, q, seed=q)
    W = np.eye(q) if q > 1 else np.array([[1.0 + 0.5j]])
    co, cx = array_farfield(op, tensors, e, d, 0.5, 0.7, 2.1, 376.7, cur, W)
    rco, rcx = oracle.array_farfield(nx, ny, e, tensors, d, 0.5, 0.7, 2.1, 376.7, cur, W)
    assert np.linalg.norm(co - rco) / np.linalg.norm(rco) < 1e-12
    assert np.linalg.norm(cx - rcx) / np.linalg.norm(rcx) < 1e-12
