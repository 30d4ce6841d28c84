"""The drop-in boundary: libbt_b200.so loads, exports exactly the symbols
include/blocktet_b200.h declares, and fails loudly without a GPU."""
import ctypes
import os
import re

import pytest
import torch

import paper_2308_01792_b200 as bt
from paper_2308_01792_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "blocktet_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(bt_[a-z0-9_]+)\s*\(", text))


def test_every_declared_symbol_is_exported():
    decl = declared_symbols()
    assert len(decl) >= 50
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert decl == set(_lib.SIGNATURES), decl ^ set(_lib.SIGNATURES)


def test_version_and_mesh_generator_are_host_only():
    assert b"sm_100a" in _lib.lib.bt_version()
    from pyoracle import cubes_mesh_text
    for n, p, s in ((1, 0.0, 0), (2, 0.1, 0), (4, 0.1, 0), (3, 0.1, 7)):
        assert bt.cubes_mesh_text(n, p, s) == cubes_mesh_text(n, p, s)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    h = ctypes.c_void_p()
    st = _lib.lib.bt_grid_create(bt.ref_tet_text().encode(), 2, 3, 0, ctypes.byref(h))
    assert st == 6  # BT_CUDA_ERROR
    assert b"no CUDA device" in _lib.lib.bt_last_error()


def test_error_mapping():
    with pytest.raises(bt.InvalidArgument):
        bt.compute_stencil(bt.FormId.div_k_grad(bt.Coefficient.constant(1.0)), None, 2)
    with pytest.raises(bt.InvalidArgument):
        bt.FormId.div_k_grad(None)
