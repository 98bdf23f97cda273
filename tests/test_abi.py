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
