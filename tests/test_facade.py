"""The C++ facade (include/blocktet_b200.hpp) over the C ABI: it compiles
against the in-tree library, keeps the reference's exception types, fails
loudly without CUDA, and on the GPU gives the oracle's results through the
reference-shaped API (apply_stencil, v_cycle)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import paper_2308_01792_b200 as bt
from oracle.pyoracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2308_01792_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("facade") / "facade_check")
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), "-o", out, "-L", LIBDIR, "-lbt_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def mesh_file(tmp_path):
    p = tmp_path / "cube_kuhn.mesh"
    p.write_text(bt.cube_kuhn_text())
    return str(p)


def test_facade_index_and_exceptions(exe):
    r = subprocess.run([exe, "index"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "ok"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_facade_fails_loudly_without_cuda(exe, tmp_path):
    r = subprocess.run([exe, "nogpu", mesh_file(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("raised")


@pytest.mark.gpu
def test_facade_apply_and_vcycle_match_oracle(exe, tmp_path):
    r = subprocess.run([exe, "apply", mesh_file(tmp_path), str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    load = lambda n: np.fromfile(str(tmp_path / n), dtype=np.float64)
    l = 4
    o = Oracle(bt.cube_kuhn_text(), 2, l)
    x = o.random_fill(l, 0)
    assert np.array_equal(load("x.bin"), x)  # inputs bit-exact
    y = o.apply_stencil(l, x, bc=0)
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    assert rel(load("y.bin"), y) <= 1e-12
    o.make_hierarchy(form=0, kernel=1)
    sm = bt.SmootherConfig.chebyshev(2)
    sm.nu1 = sm.nu2 = 2
    rhs = load("rhs.bin")
    u, _ = o.vcycles(l, sm.as_array(), rhs, np.zeros_like(rhs), 3, 2, 1e-14, 20)
    assert rel(load("u.bin"), u) <= 1e-12


@pytest.mark.gpu
def test_facade_reference_shaped_call_sites(tmp_path):
    """tests/cpp/facade_kats.cpp: reference-style call sites (Grid from
    parse_mesh, values[l][cell][entry], at(), groups(), cg over a callable)
    against the reference tests' known answers."""
    out = str(tmp_path / "facade_kats")
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_kats.cpp"), "-o", out, "-L", LIBDIR, "-lbt_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert r.stdout.strip().endswith("ok")


def test_facade_kats_compile(tmp_path):
    """The reference-shaped call sites compile against the facade (no GPU needed)."""
    out = str(tmp_path / "facade_kats.o")
    cmd = ["g++", "-std=c++17", "-O1", "-c", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_kats.cpp"), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
