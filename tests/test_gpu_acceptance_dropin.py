"""The reference's OWN acceptance suite (tests/acceptance.cc + src/verify.cc,
unmodified) linked against the GPU drop-in (paper_2311_08316_b200/dropin/
cqrrpt_dropin.cc defines cqrrpt::cqrrpt and cqrrpt::cqrrpt_core over the C
ABI; oracle/Makefile weakens the reference's two definitions so every call
site binds to ours). Each check that calls cqrrpt()/cqrrpt_core() must print
its PASS line: thm2.1 (cqrrpt_core, Gaussian operator, validate at 1e-13, k =
100), cor3.1 (cqrrpt_core under small distortion), stability (cond 1e10
polynomial decay, loss/recon <= 1e-12 where plain CholeskyQR fails), rank
(exact rank 17), pivots-low / pivots-high (pivot quality against the
reference QRCP), plus sketch-struct (operator structure, unchanged path).
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")
CHECKS = ["thm2.1", "cor3.1", "stability", "rank", "pivots-low", "pivots-high", "sketch-struct"]


@pytest.mark.parametrize("check", CHECKS)
def test_reference_acceptance_through_gpu_dropin(cuda, check):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/acceptance_gpu not built (needs /root/reference at build time)")
    r = subprocess.run([EXE, "--only", check], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    print(out)
    lines = [ln for ln in out.splitlines() if f"] {check}" in ln]
    assert lines, out
    assert lines[0].startswith("[ PASS ]"), out
