"""The C-ABI library builds, loads and exports every symbol include/frsvt.h
declares; argument validation runs before any device work (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "frsvt.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("frsvt_", "rpca_"))))


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def test_header_and_binding_agree(P):
    decl = _declared()
    assert len(decl) >= 15
    assert sorted(P._abi.SYMBOLS) == decl


def test_library_exports_every_symbol(P):
    out = subprocess.run(["nm", "-D", "--defined-only", P.library_path], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for name in _declared():
        assert name in exported, name


def test_struct_layouts_match_header(P, tmp_path):
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "frsvt.h"\n'
                 'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(frsvt_config), sizeof(frsvt_info),'
                 ' sizeof(rpca_state), offsetof(rpca_state, iter), offsetof(frsvt_info, mu));}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    A = P._abi
    assert got == [ctypes.sizeof(A.FrsvtConfig), ctypes.sizeof(A.FrsvtInfo), ctypes.sizeof(A.RpcaState),
                   A.RpcaState.iter.offset, A.FrsvtInfo.mu.offset]


def test_validation_before_device_work(P):
    lib = P.lib
    A = P._abi
    h = ctypes.c_void_p()
    cfg = A.FrsvtConfig(dtype=0, m_local=100, n=50, m_global=100, row0=0, l=60, q=1,
                        range_propagation=1, seed=1, nranks=1, rank=0)
    assert lib.frsvt_create(ctypes.byref(cfg), None, ctypes.byref(h)) == 1  # l > n
    cfg.l = 10
    cfg.dtype = 7
    assert lib.frsvt_create(ctypes.byref(cfg), None, ctypes.byref(h)) == 1
    cfg.dtype = 0
    cfg.q = -1
    assert lib.frsvt_create(ctypes.byref(cfg), None, ctypes.byref(h)) == 1
    cfg.q = 1
    cfg.nranks = 2
    assert lib.frsvt_create(ctypes.byref(cfg), None, ctypes.byref(h)) == 1  # no nccl id
    assert h.value is None
    assert lib.frsvt_apply(None, None, 0, 1.0, None, 0, None) == 1
    assert lib.rpca_alm_step(None, None, 0, None) == 1
    assert P.status_string(lib, 5).startswith("non-finite")
    assert lib.frsvt_kernel_launches(None) == -1


def test_product_path_has_no_oracle_or_fallback():
    """The package never imports the oracle and has no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_1509_00296_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "import synth" not in src and "from synth" not in src, f
