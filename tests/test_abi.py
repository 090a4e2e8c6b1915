"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and
exports every symbol include/dgtau.h declares (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dglib():
    import paper_2210_03523_b200 as dg

    dg.build()
    return dg


def _declared():
    src = open(os.path.join(ROOT, "include", "dgtau.h")).read()
    return sorted(set(re.findall(r"\b(dg_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(dglib):
    L = dglib.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(dglib.EXPORTS) <= set(names)


def test_sm100a_cubin_present(dglib):
    out = subprocess.run(["cuobjdump", "--list-elf", dglib._SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product():
    """The product never imports / links / calls the oracle."""
    pkg = os.path.join(ROOT, "paper_2210_03523_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "dgsem_oracle" not in txt and "liboracle" not in txt, f


def test_no_gpu_raises_cleanly(dglib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import workloads as W

    with pytest.raises(dglib.DGError):
        dglib.Solver(W.cube_mesh(2))
    # the C side refuses too (no CPU fallback)
    ctx = ctypes.c_void_p()
    p = dglib._Params()
    p.physics, p.flux, p.gamma = 0, 0, 1.4
    rc = dglib.lib().dg_create(ctypes.byref(p), ctypes.byref(ctx))
    assert rc != 0
