"""The C-ABI boundary without a GPU: libtbt.so loads, exports every symbol
declared in include/*.h, carries sm_100a code, and fails loudly (no CPU
fallback) when no device is present."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2506_04710_b200 import ToeplitzMatvec, ToeplitzRep, _lib
from paper_2506_04710_b200.toeplitz import DeviceError

REPO = Path(__file__).resolve().parents[1]


def declared_functions():
    names = []
    for h in (REPO / "include").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*[\w\s\*]*?\b(tbt\w*)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if not n.startswith("TBT_")))


def test_every_declared_symbol_exported():
    L = _lib.lib()
    decl = declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) <= set(_lib.SIGNATURES), set(decl) - set(_lib.SIGNATURES)


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not Path("/usr/local/cuda/bin/cuobjdump").exists(),
                    reason="no cuobjdump")
def test_library_is_sm100a():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    rep = ToeplitzRep(2, 2, 3, __import__("numpy").zeros((5, 3, 3), complex))
    with pytest.raises(DeviceError):
        ToeplitzMatvec(rep)
    assert _lib.last_error()


def test_cpp_mirror_compiles(tmp_path):
    """include/tbt.hpp (the C++ mirror a reference maintainer would include)
    compiles against the C ABI header."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    src = tmp_path / "use_hpp.cpp"
    src.write_text('#include "tbt.hpp"\n'
                   'int main() {\n'
                   '  std::vector<tbt::Complex> gen(1);\n'
                   '  try { tbt::ToeplitzMatvec op(1, 1, 1, gen); int e[9] = {0};\n'
                   '        e[4] = 1; op.setMargin(e, nullptr, nullptr, nullptr, nullptr);\n'
                   '        op.precompute(); (void)op.apply(tbt::Vector(op.size()));\n'
                   '        (void)op.applyB(tbt::Vector(op.sizeA())); (void)op.applyBT(tbt::Vector(op.sizeM()));\n'
                   '        (void)op.applyC(tbt::Vector(op.sizeM())); (void)tbt::toeplitzMatvec(op, tbt::Vector(op.size()));\n'
                   '        tbt::SolverOptions so; std::vector<tbt::Vector> V(1, tbt::Vector(op.size()));\n'
                   '        (void)tbt::iterativeSolve(op, V, so); (void)tbt::schurSolve(op, V, so); }\n'
                   '  catch (const std::exception&) {}\n'
                   '  return 0;\n'
                   '}\n')
    r = subprocess.run([gxx, "-std=c++17", "-fsyntax-only", "-I", str(REPO / "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _build_mirror_demo(tmp_path):
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    repo = Path(__file__).resolve().parents[1]
    exe = tmp_path / "mirror_demo"
    lib_dir = repo / "paper_2506_04710_b200"
    subprocess.run([gxx, "-std=c++17", "-O2", f"-I{repo / 'include'}", str(repo / "tests" / "cpp" / "mirror_demo.cpp"),
                    f"-L{lib_dir}", "-ltbt", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_mirror_links_and_runs(tmp_path):
    """The C++ mirror linked against libtbt.so and run (on a CPU-only host
    the constructor must report the missing device, not fall back)."""
    import subprocess
    import torch
    exe = _build_mirror_demo(tmp_path)
    r = subprocess.run([str(exe), str(tmp_path / "out.bin")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    if not torch.cuda.is_available():
        assert r.stdout.startswith("no device")


@pytest.mark.gpu
def test_gpu_cpp_mirror_matches_oracle(gpu, tmp_path):
    import subprocess

    import numpy as np

    import oracle
    from paper_2506_04710_b200 import CONFIGS, ToeplitzRep
    exe = _build_mirror_demo(tmp_path)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
    v = np.fromfile(out, dtype=np.complex128).reshape(3, -1)
    x, y, sol = v
    cfg = CONFIGS["C1"]
    rep = ToeplitzRep.synthetic(cfg)
    o = oracle.Oracle(cfg.nx, cfg.ny, cfg.m, rep.generators)  # no correction in the demo
    assert np.linalg.norm(y - o.applyA(x)) / np.linalg.norm(y) < 1e-11
    ref = o.gmres(x, tol=1e-8, max_iter=2000, restart=30)
    assert np.linalg.norm(sol - ref["x"]) / np.linalg.norm(ref["x"]) < 1e-8
