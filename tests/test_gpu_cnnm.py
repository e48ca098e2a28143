"""GPU parity of the CNNM baseline (cnnm_solve, solver.cpp:161-170; SURVEY
§8f-4) against the oracle's literal restatement (numpy thin SVD per
iteration), on the reference's own cnnm test cases (test_solver.cpp:151-193),
BASELINE config 1 and the paper's runtime-ordering criterion
(test_acceptance.cpp:288-300).

Tolerances: both sides fp64; the GPU thresholds singular values through the
Gram, so L agrees to rel-L2 1e-7, the objective trace to rel
1e-7 and the residual / l_change traces to rel 1e-6 (abs 1e-12, the rounding
floor of these relative quantities) over fixed iteration counts.
"""
import numpy as np
import pytest

from oracle import icnnm_oracle as O
from paper_2604_17001_b200 import synth

pytestmark = pytest.mark.gpu

FIXED = dict(tol_primal=1e-300, tol_change=1e-300)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _cos(m, period):
    return np.cos(2.0 * np.pi * np.arange(m) / period)


def test_reference_cnnm_cases(gpu):                      # test_solver.cpp:151-168
    M = synth.Rng(35).random_tensor((8, 8))
    L, rep = gpu.cnnm_solve(M, np.ones_like(M), (3, 3), gpu.SolverConfig(max_iters=300))
    assert _rel(L, M) < 1e-3
    Lo, ro = O.cnnm_solve(M, np.ones_like(M), (3, 3), O.SolverConfig(max_iters=300))
    assert _rel(L, Lo) < 1e-7 and rep.iterations == ro.iterations
    L0 = _cos(32, 8)
    mask = synth.reference_bernoulli_mask((32,), 0.75, 5)
    L2, rep2 = gpu.cnnm_solve(L0, mask, (8,))
    assert _rel(L2, L0) < 1e-3
    Lo2, ro2 = O.cnnm_solve(L0, mask, (8,))
    assert _rel(L2, Lo2) < 1e-6
    assert abs(rep2.iterations - ro2.iterations) <= 1


def test_exact_basis_icnnm_and_cnnm_agree(gpu):          # test_solver.cpp:170-193
    L0 = _cos(32, 8)
    B = gpu.learn_ensemble_basis([L0], (8,))
    mask = synth.reference_bernoulli_mask((32,), 0.75, 11)
    li, _ = gpu.icnnm_solve(L0, mask, B, gpu.SolverConfig(engine="ffma"))
    lc, _ = gpu.cnnm_solve(L0, mask, (8,))
    assert np.linalg.norm(li - lc) / np.linalg.norm(L0) < 1e-4


@pytest.mark.parametrize("dims,ks,iters", [((8, 8), (3, 3), 120), ((12, 10, 8), (3, 3, 2), 80),
                                          ((9, 7, 16), (2, 3, 4), 60)])
def test_cnnm_trace_matches_oracle(gpu, dims, ks, iters):
    r = synth.Rng(900 + len(dims))
    X = r.random_tensor(dims)
    mask = synth.reference_bernoulli_mask(dims, 0.6, 17)
    for fill in ("zero", "mean"):
        cfg = dict(max_iters=iters, init_fill=fill, **FIXED)
        L, rep = gpu.cnnm_solve(X * mask, mask, ks, gpu.SolverConfig(**cfg))
        Lo, ro = O.cnnm_solve(X * mask, mask, ks, O.SolverConfig(**cfg))
        assert rep.iterations == ro.iterations == iters
        assert _rel(L, Lo) < 1e-7
        np.testing.assert_allclose(rep.objective, ro.objective, rtol=1e-7)
        # residual / l_change are relative quantities: below ~1e-12 they are
        # rounding noise on both sides
        np.testing.assert_allclose(rep.primal_residual, ro.primal_residual, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(rep.l_change, ro.l_change, rtol=1e-6, atol=1e-12)


def test_cnnm_config1_matches_oracle(gpu):
    """BASELINE config 1 (32x32x8, kernel 5x5x3, 200 iterations) through the
    CNNM baseline: the recovered video against the oracle."""
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    cfg = dict(max_iters=w.iters, **FIXED)
    L, rep = gpu.cnnm_solve(X * mask, mask, w.kernel, gpu.SolverConfig(**cfg))
    Lo, ro = O.cnnm_solve(X * mask, mask, w.kernel, O.SolverConfig(**cfg))
    assert _rel(L, Lo) < 1e-6
    assert abs(synth.psnr(X, L) - O.psnr(X, Lo)) < 0.01
    np.testing.assert_allclose(rep.objective, ro.objective, rtol=1e-6)


def test_cnnm_errors(gpu):
    X = np.ones((6, 6))
    with pytest.raises(ValueError, match="empty sampling set"):
        gpu.cnnm_solve(X, np.zeros_like(X), (2, 2))
    with pytest.raises(ValueError, match="0 or 1"):
        gpu.cnnm_solve(X, np.full_like(X, 0.5), (2, 2))
    with pytest.raises(ValueError, match="non-finite"):
        gpu.cnnm_solve(np.full_like(X, np.nan), np.ones_like(X), (2, 2))
    with pytest.raises(ValueError, match="lambda"):
        gpu.cnnm_solve(X, np.ones_like(X), (2, 2), gpu.SolverConfig(lambda_=-1.0))
    with pytest.raises(ValueError, match="KernelShape"):
        gpu.cnnm_solve(X, np.ones_like(X), (7, 2))


def test_runtime_ordering(gpu):                          # test_acceptance.cpp:288-300
    """ICNNM (pre-learned basis, column shrink) is faster per solve than the
    CNNM baseline (an SVD per iteration) at 40 iterations."""
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    cfg = gpu.SolverConfig(max_iters=40, **FIXED)
    gpu.icnnm_solve(X * mask, mask, B, cfg)
    gpu.cnnm_solve(X * mask, mask, w.kernel, cfg)
    ti = tc = 0.0
    for _ in range(5):
        _, ri = gpu.icnnm_solve(X * mask, mask, B, cfg)
        _, rc = gpu.cnnm_solve(X * mask, mask, w.kernel, cfg)
        ti += ri.wall_time_seconds
        tc += rc.wall_time_seconds
    assert ti < tc


def test_cli_cnnm_matches_api(gpu, tmp_path):
    import json
    import subprocess
    from paper_2604_17001_b200 import io as pio
    from paper_2604_17001_b200._lib import CLI_PATH
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    pio.write_tnsr(str(tmp_path / "M.tnsr"), X * mask)
    pio.write_tnsr(str(tmp_path / "mask.tnsr"), mask)
    (tmp_path / "cfg.json").write_text(json.dumps({"max_iters": 30, "tol_primal": 1e-300,
                                                   "tol_change": 1e-300}))
    out = subprocess.run([CLI_PATH, "cnnm", "--input", str(tmp_path / "M.tnsr"), "--mask",
                          str(tmp_path / "mask.tnsr"), "--kernel", "5,5,3", "--config",
                          str(tmp_path / "cfg.json"), "--out", str(tmp_path / "L.tnsr"),
                          "--report", str(tmp_path / "rep.json")], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    L = pio.read_tnsr(str(tmp_path / "L.tnsr"))
    rep = json.loads((tmp_path / "rep.json").read_text())
    Lp, rp = gpu.cnnm_solve(X * mask, mask, w.kernel, gpu.SolverConfig(max_iters=30, **FIXED))
    # cuBLAS / cuSOLVER are not bit-reproducible across processes (algorithm
    # selection), so the CLI and the in-process call agree to fp64 rounding
    np.testing.assert_allclose(L, Lp, rtol=1e-12, atol=1e-14)
    assert rep["iterations"] == 30
    np.testing.assert_allclose(rep["objective"], rp.objective, rtol=1e-12)
