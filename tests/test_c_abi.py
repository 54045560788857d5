"""CPU checks of the drop-in boundary: the sm_100a library loads, exports
every entry point include/cqrrpt_gpu.h declares, and its host-side argument
validation mirrors the reference's exceptions (no GPU work is issued)."""
import ctypes
import os
import re

import pytest

import paper_2311_08316_b200 as pkg
from paper_2311_08316_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cqrrpt_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(cqrrpt_gpu_[a-z0-9_]+)\s*\(", src)
    return sorted(set(n for n in names if not n.endswith("_fn")))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the same surface
    assert set(names) <= set(_lib.SYMBOLS) | {"cqrrpt_gpu_ctx_init"}


def test_library_is_sm100a_only():
    so = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_sketch_rows_and_flop_model_host_entry_points():
    assert pkg.sketch_rows_for(1.25, 50) == 63  # test_cqrrpt.cc:253-260
    assert pkg.sketch_rows_for(3.0, 500) == 1500
    assert pkg.sketch_rows_for(1.25, 100) == 125  # test_sketch.cc default d
    assert abs(pkg.flop_model(1000, 100, 100, 125, 0.0) - 3.227e7) <= 3.227e4  # test_cqrrpt.cc:315-319
    assert pkg.flop_model(500, 64, 0, 80, 77.0) == 77.0
    with pytest.raises(ValueError):
        pkg.flop_model(100, 10, 11, 20, 0.0)  # test_cqrrpt.cc:343-346


def _call(m=100, n=10, lda=100, d_factor=1.25, nnz=4, eps=1e-4, a=1, r=1, ldr=10, j=1):
    lib = _lib.load()
    k, k0 = ctypes.c_int64(-7), ctypes.c_int64(-7)
    ctx = _lib.new_ctx()
    rc = lib.cqrrpt_gpu_dgeqpt(m, n, a, lda, d_factor, nnz, 0, eps, r, ldr, j, ctypes.byref(k), ctypes.byref(k0),
                               ctypes.byref(ctx))
    return rc, k.value, k0.value


def test_dgeqpt_argument_errors_mirror_reference_exceptions():
    # check_config (cqrrpt.cc:38-42): gamma < 1, eps_tol <= u
    assert _call(d_factor=0.5)[0] == -5
    assert _call(eps=1.1102230246251565e-16 / 2)[0] == -8
    # sample_sketch (sketch.cc:54,74-75): nnz outside [1, d]
    assert _call(nnz=0)[0] == -6
    assert _call(nnz=14)[0] == -6  # d = ceil(1.25*10) = 13
    assert _call(lda=50)[0] == -4
    assert _call(ldr=5)[0] == -10
    assert _call(m=-1)[0] == -1
    # n == 0 returns an empty factorization without touching the device (cqrrpt.cc:319-324)
    rc, k, k0 = _call(n=0)
    assert rc == 0 and k == 0 and k0 == 0


def test_python_config_mirrors_reference_defaults():
    cfg = pkg.CqrrptConfig()
    assert cfg.gamma == 1.25 and cfg.nnz_per_col == 4 and cfg.eps_tol == 1e-4  # cqrrpt.hh:92-102
    assert cfg.family == pkg.SketchFamily.saso and cfg.cond_method == pkg.CondMethod.identity_deviation
    assert cfg.stage1_enabled and cfg.validate_output
    with pytest.raises(ValueError):
        pkg.check_config(pkg.CqrrptConfig(gamma=0.5))
    with pytest.raises(ValueError):
        pkg.check_config(pkg.CqrrptConfig(eps_tol=1e-17))


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np
    with pytest.raises(RuntimeError):
        pkg.cqrrpt(np.ones((10, 3)), pkg.CqrrptConfig())


def test_trsm_engine_choice(monkeypatch):
    """cqrrpt_gpu_trsm_engine (a host-only query): the INT8 tensor-core engine
    from m >= 131072 rows and k >= 768 columns, DMMA below; CQRRPT_GPU_TRSM
    forces either."""
    from paper_2311_08316_b200 import kernels
    monkeypatch.delenv("CQRRPT_GPU_TRSM", raising=False)
    assert kernels.trsm_engine(4194304, 2048) == "int8"  # C5-2048
    assert kernels.trsm_engine(131072, 1024) == "int8"   # C2
    assert kernels.trsm_engine(4194304, 512) == "dmma"   # k = 512: DMMA measured faster
    assert kernels.trsm_engine(16384, 256) == "dmma"     # C1
    monkeypatch.setenv("CQRRPT_GPU_TRSM", "dmma")
    assert kernels.trsm_engine(4194304, 2048) == "dmma"
    monkeypatch.setenv("CQRRPT_GPU_TRSM", "oz")
    assert kernels.trsm_engine(1000, 300) == "int8"
