"""Test-side ZTOE1 writer and partBlock restatement (row f3 fixtures).

Writes block caches in the reference's on-disk format (restated from
saveBlockCache / loadBlockCache, proj/src/toeplitz.cpp:700-815): "ZTOE1",
u8 mode, i32 nx, ny, e[9], records {u8 tag, i32 i0, i1, i2, i64 rows,
cols, column-major complex128}, tag 255. Also assembles the dense margin
block C from the C records by partBlock's rules (:506-573), independently
of the loader in paper_2506_04710_b200/csrc/io.cu."""
import struct

import numpy as np

EDGE = (2, 8, 6, 4)
CORNER = (3, 9, 1, 7)


def _rec(f, tag, i0, i1, i2, mat):
    mat = np.asarray(mat, dtype=np.complex128)
    f.write(struct.pack("<Biiiqq", tag, i0, i1, i2, mat.shape[0], mat.shape[1]))
    f.write(np.asfortranarray(mat).tobytes(order="F"))


def random_c_records(nx, ny, e, rng):
    e2, e8, e6, e4 = e[1], e[7], e[5], e[3]
    cn = lambda r, c: (rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c))) * 0.05  # noqa: E731
    ct = sum(e[c - 1] for c in CORNER)
    recs = {
        "c11": [cn(e2, e2) + (2 + 2j) * np.eye(e2) * (k == 0) for k in range(ny)],
        "c21": [cn(e8, e2) for _ in range(2 * ny - 1)],
        "c22": [cn(e8, e8) + (2 + 2j) * np.eye(e8) * (k == 0) for k in range(ny)],
        "c33": [cn(e6, e6) + (2 + 2j) * np.eye(e6) * (k == 0) for k in range(nx)],
        "c43": [cn(e4, e6) for _ in range(2 * nx - 1)],
        "c44": [cn(e4, e4) + (2 + 2j) * np.eye(e4) * (k == 0) for k in range(nx)],
        "c31": cn(nx * e6, ny * e2), "c41": cn(nx * e4, ny * e2),
        "c32": cn(nx * e6, ny * e8), "c42": cn(nx * e4, ny * e8),
        "c5x": [cn(ct, n) for n in (ny * e2, ny * e8, nx * e6, nx * e4)],
        "c55": {(a, b): cn(e[CORNER[a] - 1], e[CORNER[b] - 1]) + (2 + 2j) * np.eye(e[CORNER[a] - 1], e[CORNER[b] - 1]) * (a == b)
                for a in range(4) for b in range(a, 4)},
    }
    return recs


def assemble_c(nx, ny, e, recs):
    """Dense margin block from the C records (partBlock, toeplitz.cpp:506-573)."""
    parts = []
    for g, comp in enumerate(EDGE, start=1):
        for a in range(1, (ny if g <= 2 else nx) + 1):
            parts.append((g, a, e[comp - 1]))
    for a, comp in enumerate(CORNER, start=1):
        parts.append((5, a, e[comp - 1]))
    offs = np.cumsum([0] + [p[2] for p in parts])
    nM = int(offs[-1])
    C = np.zeros((nM, nM), complex)
    eg = {g: e[EDGE[g - 1] - 1] for g in range(1, 5)}
    crs = np.cumsum([0] + [e[c - 1] for c in CORNER])

    def blk(gi, a, gj, b):
        toe = {1: "c11", 2: "c22", 3: "c33", 4: "c44"}
        if gi == gj and gi <= 4:
            st = recs[toe[gi]]
            return st[a - b] if a >= b else st[b - a].T
        if (gi, gj) == (2, 1):
            return recs["c21"][(a - b) + ny - 1]
        if (gi, gj) == (1, 2):
            return recs["c21"][(b - a) + ny - 1].T
        if (gi, gj) == (4, 3):
            return recs["c43"][(a - b) + nx - 1]
        if (gi, gj) == (3, 4):
            return recs["c43"][(b - a) + nx - 1].T
        rect = {(3, 1): "c31", (4, 1): "c41", (3, 2): "c32", (4, 2): "c42"}
        if (gi, gj) in rect:
            m = recs[rect[(gi, gj)]]
            return m[(a - 1) * eg[gi]:a * eg[gi], (b - 1) * eg[gj]:b * eg[gj]]
        if (gj, gi) in rect:
            return blk(gj, b, gi, a).T
        if gi == 5 and gj != 5:
            m = recs["c5x"][gj - 1]
            return m[crs[a - 1]:crs[a], (b - 1) * eg[gj]:b * eg[gj]]
        if gi != 5 and gj == 5:
            return blk(gj, b, gi, a).T
        return recs["c55"][(a - 1, b - 1)] if a <= b else recs["c55"][(b - 1, a - 1)].T

    for i, (gi, a, si) in enumerate(parts):
        for j, (gj, b, sj) in enumerate(parts):
            if si and sj:
                C[offs[i]:offs[i + 1], offs[j]:offs[j + 1]] = blk(gi, a, gj, b)
    return C


def write_ztoe1(path, nx, ny, e, gen_raw, margin=None, recs=None, mode=2):
    """gen_raw: (nb, m, m) column-major blocks (gen.blocks_raw order);
    margin: a Margin (bside / brow / bcorner in tbt_gen.h layout), or None
    for an A-only cache (margin components empty: the loader zero-fills
    records that are absent, toeplitz.cpp:766)."""
    m = e[4]
    with open(path, "wb") as f:
        f.write(b"ZTOE1")
        f.write(struct.pack("<B", mode))
        f.write(struct.pack("<ii", nx, ny))
        f.write(struct.pack("<9i", *e))
        t = 0
        for j in range(nx):
            _rec(f, 1, 0, j, 0, gen_raw[t].T)  # raw [t][b][a] -> block (a, b)
            t += 1
        for i in range(1, ny):
            for j in range(2 * nx - 1):
                _rec(f, 1, i, j, 0, gen_raw[t].T)
                t += 1
        if margin is None:
            f.write(struct.pack("<B", 255))
            return
        off = 0
        for r in range(2):
            em = e[EDGE[r] - 1]
            for j in range(2 * ny - 1):
                n = em * nx * m
                _rec(f, 2, r, j, 0, margin.bside[off:off + n].reshape(nx * m, em).T)
                off += n
        off = 0
        for r in range(2):
            em = e[EDGE[2 + r] - 1]
            for j in range(ny):
                for k in range(2 * nx - 1):
                    n = em * m
                    _rec(f, 3, r, j, k, margin.brow[off:off + n].reshape(m, em).T)
                    off += n
        off = 0
        nA = nx * ny * m
        for c in range(4):
            em = e[CORNER[c] - 1]
            _rec(f, 4, c, 0, 0, margin.bcorner[off:off + em * nA].reshape(nA, em).T)
            off += em * nA
        for r, key in enumerate(("c11", "c21", "c22", "c33", "c43", "c44")):
            for k, mat in enumerate(recs[key]):
                _rec(f, 5, r, k, 0, mat)
        for r, key in enumerate(("c31", "c41", "c32", "c42")):
            _rec(f, 6, r, 0, 0, recs[key])
        for g in range(4):
            _rec(f, 7, g, 0, 0, recs["c5x"][g])
        for (a, b), mat in recs["c55"].items():
            _rec(f, 8, a, b, 0, mat)
        f.write(struct.pack("<B", 255))


def write_ztoe1_dense(path, nx, ny, e, mode, a_level1=None, b_full=None, c_full=None, z_full=None):
    """SemiSparse (mode 1: ny first-level A blocks, each (nx*m)^2, plus dense
    B and C) or Full (mode 0: the whole matrix) caches, tags 9-12
    (toeplitz.cpp:730-745)."""
    with open(path, "wb") as f:
        f.write(b"ZTOE1")
        f.write(struct.pack("<B", mode))
        f.write(struct.pack("<ii", nx, ny))
        f.write(struct.pack("<9i", *e))
        if mode == 1:
            for i, blk in enumerate(a_level1):
                _rec(f, 9, i, 0, 0, blk)
            if b_full is not None and b_full.size:
                _rec(f, 10, 0, 0, 0, b_full)
            if c_full is not None and c_full.size:
                _rec(f, 11, 0, 0, 0, c_full)
        elif mode == 0:
            _rec(f, 12, 0, 0, 0, z_full)
        f.write(struct.pack("<B", 255))
