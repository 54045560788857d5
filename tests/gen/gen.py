"""TEST INFRASTRUCTURE: the BASELINE inputs rebuilt on the GPU
box bit-for-bit equal to the reference generators' output.

The Gaussian draws come from the oracle's restated counter RNG on the host
(oracle/cqrrpt_oracle.c gaussian_block, testmat.cc:17-25, OpenMP over
columns); the serial O(m n^2) linear algebra of gen_spectral / gen_exact_rank
(householder_qr, accumulate_q, apply_q_left, matmul; linalg.cc:52-197) runs on
the device in the reference's exact operation order (tests/gen/gen_gpu.cu).
Every full-size input is checked against the sha256 of the reference's own
input bytes recorded by tests/golden/make_fullsize_golden.py before use.

Only tests/ import this module.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRC = os.path.join(HERE, "gen_gpu.cu")
LIB = os.path.join(HERE, "_build", "libgen_gpu.so")

SALT_LEFT, SALT_RIGHT = 0x6C656674, 0x72696768  # testmat.cc:79-93 ("left", "righ")
SALT_A, SALT_B = 0xAAAA, 0xBBBB                  # testmat.cc:145-151


def build() -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    nvcc = "/usr/local/cuda/bin/nvcc"
    host = ["-ccbin", "/usr/bin/g++"] if os.path.exists("/usr/bin/g++") else []
    cmd = [nvcc] + host + ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", SRC, "-o", LIB]
    subprocess.run(cmd, check=True)
    return LIB


def _lib():
    if not os.path.exists(LIB):
        build()
    L = ctypes.CDLL(LIB)
    i64, vp = ctypes.c_int64, ctypes.c_void_p
    L.gen_householder_reduce.argtypes = [vp, i64, i64, vp, vp]
    L.gen_accumulate_q.argtypes = [vp, i64, vp, i64, vp, vp]
    L.gen_apply_q_left.argtypes = [vp, i64, i64, vp, vp, i64, vp]
    L.gen_matmul.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, vp]
    return L


def _check(rc, what):
    if rc:
        raise RuntimeError(f"{what}: CUDA error {rc}")


def to_device(a):
    """Column-major host array -> column-major CUDA tensor (stride (1, m))."""
    import torch
    a = np.asfortranarray(a)
    return torch.from_numpy(a.T).to("cuda").t()


def sha256_device(t) -> str:
    """sha256 of a column-major (m x n) CUDA tensor's bytes in column-major
    order (the reference DenseMatrix layout)."""
    host = t.t().contiguous().cpu().numpy()  # (n, m) row-major = column-major bytes
    return hashlib.sha256(host.tobytes()).hexdigest()


def gen_spectral(oracle, m, n, sigma, seed):
    """gen_spectral(m, n, SpectrumSpec::explicit_list(sigma), seed)
    (testmat.cc:79-93, restated as orc_gen_spectral_list), on the device."""
    import torch
    L = _lib()
    st = torch.cuda.current_stream().cuda_stream
    left = to_device(oracle.gaussian_block(m, n, oracle.mix_seed(seed, SALT_LEFT)))
    betas = torch.zeros(n, dtype=torch.float64, device="cuda")
    _check(L.gen_householder_reduce(left.data_ptr(), m, n, betas.data_ptr(), st), "householder (left)")
    vb = to_device(oracle.gaussian_block(n, n, oracle.mix_seed(seed, SALT_RIGHT)))
    vbet = torch.zeros(n, dtype=torch.float64, device="cuda")
    _check(L.gen_householder_reduce(vb.data_ptr(), n, n, vbet.data_ptr(), st), "householder (right)")
    v = torch.eye(n, dtype=torch.float64, device="cuda").t().contiguous().t()
    _check(L.gen_accumulate_q(vb.data_ptr(), n, vbet.data_ptr(), n, v.data_ptr(), st), "accumulate_q")
    sig = torch.as_tensor(np.ascontiguousarray(sigma, dtype=np.float64), device="cuda")
    out = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()  # column-major m x n
    out[:n, :] = sig[:, None] * v.t()  # out(i, j) = sigma_i V(j, i)
    _check(L.gen_apply_q_left(left.data_ptr(), m, n, betas.data_ptr(), out.data_ptr(), n, st), "apply_q_left")
    torch.cuda.synchronize()
    return out


def gen_exact_rank(oracle, m, n, r, seed):
    """gen_exact_rank (testmat.cc:145-151): A (m x r) B (r x n), on the device."""
    import torch
    L = _lib()
    st = torch.cuda.current_stream().cuda_stream
    a = to_device(oracle.gaussian_block(m, r, oracle.mix_seed(seed, SALT_A)))
    b = to_device(oracle.gaussian_block(r, n, oracle.mix_seed(seed, SALT_B)))
    out = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    _check(L.gen_matmul(m, r, n, a.data_ptr(), m, b.data_ptr(), r, out.data_ptr(), st), "matmul")
    torch.cuda.synchronize()
    return out


def add_noise(oracle, ab, noise, seed=1):
    """C3 / C3b: ab + (noise ||ab||_F / sqrt(mn)) G with
    G = gen_gaussian(m, n, seed), in make_fullsize_golden.py's operation order
    (numpy sum of squares on the host; scale * G rounded, then added)."""
    import torch
    m, n = ab.shape
    h = ab.t().contiguous().cpu().numpy()
    fro = float(np.sqrt(np.sum(h * h)))
    del h
    scale = noise * fro / np.sqrt(float(m) * float(n))
    g = to_device(oracle.gen_gaussian(m, n, seed))
    out = ab.clone()
    out += g * scale
    del g
    torch.cuda.synchronize()
    return out
