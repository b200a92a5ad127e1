"""CPU-side checks of the boundary: the C-ABI library builds/loads and exports every symbol
include/rsfde.h declares, the binding declares the same set, and the product path refuses
to run without a GPU (no CPU fallback).  No compute call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsfde.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsfde_[a-z_]+)\s*\(", src)))


def _lib_path():
    from paper_2404_10221_b200 import _lib
    return _lib.LIB_PATH


@pytest.fixture(scope="module")
def lib():
    path = _lib_path()
    if not os.path.exists(path):
        from paper_2404_10221_b200.build import build
        build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for required in ("rsfde_setup", "rsfde_matvec", "rsfde_precond_apply", "rsfde_gmres_step",
                     "rsfde_solve_steps", "rsfde_destroy", "rsfde_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_covers_every_declared_symbol():
    from paper_2404_10221_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_version_string(lib):
    lib.rsfde_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.rsfde_version()


def test_library_contains_sm100a_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib_path()], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_10221_b200 import inputs as I
    from paper_2404_10221_b200.solver import RsfdeSolver
    with pytest.raises(RuntimeError):
        RsfdeSolver.from_problem(I.config_c1(n=31, M=2))


def test_setup_without_device_returns_cuda_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_10221_b200 import _lib as L
    L.load()
    prob = L.rsfde_problem()
    prob.d = 1
    prob.n[0] = 31
    prob.alpha[0] = 1.5
    prob.kappa[0] = 1.0
    prob.tau_t = 0.1
    prob.M = 2
    import numpy as np
    a = np.ones(2)
    prob.e.a_half = a.ctypes.data_as(L.DP)
    prob.e.b_half = a.ctypes.data_as(L.DP)
    ctx = ctypes.c_void_p()
    st = L.load().rsfde_setup(ctypes.byref(ctx), ctypes.byref(prob), None)
    assert st == L.E_CUDA and not ctx.value


def test_oracle_is_not_imported_by_the_product_path():
    import pathlib
    pat = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b)", re.M)
    for f in pathlib.Path(ROOT, "paper_2404_10221_b200").rglob("*.py"):
        assert not pat.search(f.read_text()), f


def test_team_chunking_host_bookkeeping(monkeypatch):
    # rsfde_team_chunking (host only): pieces tile the all-to-all block, sub-slabs keep >= 2 planes,
    # at most 256 segments per x1 pencil; one rank never chunks; bad arguments fail with the same
    # codes as rsfde_team_partition
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import team_chunking, team_partition
    monkeypatch.delenv("RSFDE_TEAM_CHUNKS", raising=False)
    for n, P, req, expect in [((511, 511, 511), 8, 0, (4, 16)), ((511, 511, 511), 2, 0, (4, 64)),
                              ((511, 511, 511), 4, 8, (8, 16)), ((255, 255, 255), 8, 4, (4, 8)),
                              ((15, 7, 5), 8, 4, (1, 2)), ((7, 7, 7), 2, 4, (2, 2)), ((511, 511, 511), 1, 4, (1, 512))]:
        ch = team_chunking(n, P, req)
        part = team_partition(n, P, 0)
        assert (ch["nchunk"], ch["sc"]) == expect, (n, P, req, ch)
        assert ch["nchunk"] * ch["sc"] == part["s"] and ch["nchunk"] * ch["piece"] == part["block"]
        assert P * ch["nchunk"] <= 256 and (ch["sc"] >= 2 or ch["nchunk"] == 1)
    monkeypatch.setenv("RSFDE_TEAM_CHUNKS", "2")
    assert team_chunking((511, 511, 511), 8)["nchunk"] == 2      # requested <= 0: the environment value
    assert team_chunking((511, 511, 511), 8, 8)["nchunk"] == 8   # an explicit request wins
    with pytest.raises(L.RsfdeError):
        team_chunking((510, 511, 511), 8)                        # nranks must divide n1 + 1
    with pytest.raises(L.RsfdeError):
        team_chunking((511, 511, 511), 9)
