"""CPU-side boundary checks: the C-ABI library loads and exports every symbol
include/cusci.h declares; host-only entry points behave; the binding refuses
to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "cusci.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^(?!typedef)\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    from paper_2604_15768_b200 import build
    build.build()
    from paper_2604_15768_b200._lib import lib
    return lib()


def test_header_symbols_exported(L):
    names = header_functions()
    assert len(names) >= 17, names
    for n in names:
        assert hasattr(L, n), f"libcusci.so does not export {n}"
    from paper_2604_15768_b200._lib import EXPORTS
    assert sorted(EXPORTS) == names


def test_bound_closed_form(L):
    import paper_2604_15768_b200 as P
    assert P.gen_coupled_bound(P.Space(12, 2, 2), 1) == 92
    assert P.gen_coupled_bound(P.Space(26, 5, 5), 10) == 22400
    assert P.gen_coupled_bound(P.Space(56, 7, 7), 1) == 30723
    assert P.gen_coupled_bound(P.Space(96, 8, 8), 1) == 146720
    assert P.gen_coupled_bound(P.Space(120, 12, 12), 1) == 481824


def test_null_args_rejected_without_gpu(L):
    assert L.cusci_init(None, 0, 0, 1, None, None, None, None, None) == 1
    ctx = ctypes.c_void_p()
    assert L.cusci_init(ctypes.byref(ctx), 0, 2, 2, None, None, None, None, None) == 1  # rank >= world
    assert L.cusci_init(ctypes.byref(ctx), 0, 0, 2, None, None, None, None, None) == 1  # world>1 needs id
    assert L.gen_coupled(None, None, None, 0, None, 0.0, None) == 1
    assert L.dedup_global(None, None, None, 0, None) == 1
    assert L.merge_space(None, None, None, 0, None) == 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback():
    import paper_2604_15768_b200 as P
    with pytest.raises(RuntimeError, match="CUDA"):
        P.Context(0)


def test_sass_is_sm100a():
    """The library carries sm_100a SASS (cuobjdump), compiled in-tree."""
    import subprocess
    from paper_2604_15768_b200 import build
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
