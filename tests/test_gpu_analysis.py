"""GPU parity of the recovery-theory diagnostics against the
oracle's restatement of core/src/analysis.cpp, on the reference's own test
cases (test_analysis.cpp, test_acceptance.cpp criteria 4/5/11) and on
BASELINE-shaped video tensors.

Tolerances (fp64 on both sides; the GPU is matrix-free, the oracle uses FFT
convolutions and a dense SVD like the reference):
  r_K, support, r0, certified: exact
  sigma^K: |gpu - oracle| <= 1e-10 * max(sigma)
  alpha_K: rel 1e-9;  mu_K_I: rel 1e-12;  mu1, mu2, tau: rel 1e-8
"""
import numpy as np
import pytest

from oracle import icnnm_oracle as O
from analysis_cases import (Rng, basis_from_matrix, cosine_1d, cosine_2d, one_missing_mask,
                            random_orthogonal)

pytestmark = pytest.mark.gpu


def _A():
    from paper_2604_17001_b200 import analysis
    return analysis


def _gb(b):
    """oracle basis -> product EigenBasis"""
    from paper_2604_17001_b200 import EigenBasis
    return EigenBasis(tuple(b.kernel_shape), np.asarray(b.K), np.asarray(b.eigenvalues))


def _check_diag(d, ref, coherence=True):
    assert d.r_K == ref["r_K"]
    assert d.support_I == list(ref["support_I"])
    assert d.alpha_K == pytest.approx(ref["alpha_K"], rel=1e-9)
    assert d.mu_K_I == pytest.approx(ref["mu_K_I"], rel=1e-12)
    if coherence:
        assert d.r0 == ref["r0"]
        for key in ("mu1", "mu2", "tau"):
            assert getattr(d, key) == pytest.approx(ref[key], rel=1e-8), key
        for key in ("rho_min_noiseless", "rho_min_noisy", "error_bound_factor", "cnnm_bound",
                    "icnnm_ideal_bound"):
            assert getattr(d, key) == pytest.approx(ref[key], rel=1e-7, abs=1e-12), key
        assert d.certified == ref["certified"]
    assert d.rho0 == ref["rho0"]


def test_sigma_matches_oracle_random_bases(gpu):
    A = _A()
    r = Rng(42)
    for _ in range(10):
        L0 = r.random_tensor((6, 6))
        b = basis_from_matrix((2, 2), random_orthogonal(4, r))
        s = A.relative_eigenvalues(L0, _gb(b))
        so = O.relative_eigenvalues(L0, b)
        assert np.max(np.abs(s - so)) <= 1e-10 * so.max()
        assert A.relative_conv_rank(L0, _gb(b)) == O.relative_conv_rank(L0, b)


def test_own_basis_recovers_conv_rank(gpu):              # test_analysis.cpp:43-50
    A = _A()
    L0 = O.synth_low_conv_rank((16, 16), (4, 4), 4, Rng(99))
    b = O.learn_ensemble_basis([L0], (4, 4))
    rk, sup = A.relative_conv_rank(L0, _gb(b))
    assert rk == O.conv_spectrum(L0, (4, 4)).rank == 4
    assert sup == O.relative_conv_rank(L0, b)[1]


def test_zero_tensor_empty_support_and_errors(gpu):      # :52-59, :111-116, :154-170
    A = _A()
    b = _gb(basis_from_matrix((2, 2), random_orthogonal(4, Rng(41))))
    assert A.relative_conv_rank(np.zeros((5, 5)), b) == (0, [])
    with pytest.raises(ValueError, match="r_K = 0"):
        A.spectral_corr_coeff(np.zeros((4, 4)), b)
    with pytest.raises(ValueError, match="zero tensor"):
        A.conv_coherence(np.zeros((4, 4)), (2, 2))
    with pytest.raises(ValueError, match="zero target"):
        A.analyze_recovery(np.zeros((4, 4)), b, np.ones((4, 4)))
    with pytest.raises(ValueError, match="empty support"):
        A.active_coherence(b, [])
    with pytest.raises(ValueError, match="0 or 1"):
        A.analyze_recovery(np.ones((4, 4)), b, np.full((4, 4), 0.5))
    with pytest.raises(ValueError, match="mask dims"):
        A.analyze_recovery(np.ones((4, 4)), b, np.ones((4, 5)))
    bad = _gb(basis_from_matrix((2, 2), np.ones((4, 4))))
    with pytest.raises(ValueError, match="orthogonal"):
        A.relative_eigenvalues(np.ones((4, 4)), bad)


def test_alpha_matches_oracle_and_bounds(gpu):           # :87-109
    A = _A()
    r = Rng(43)
    for _ in range(100):
        L0 = r.random_tensor((6, 6))
        b = basis_from_matrix((2, 2), random_orthogonal(4, r))
        rk, _ = A.relative_conv_rank(L0, _gb(b))
        alpha = A.spectral_corr_coeff(L0, _gb(b))
        assert 1.0 - 1e-8 <= alpha <= np.sqrt(rk) + 1e-8
        assert alpha == pytest.approx(O.spectral_corr_coeff(L0, b), rel=1e-9)


def test_exact_basis_alpha_one(gpu):                     # :79-85
    A = _A()
    L0 = O.synth_low_conv_rank((32,), (8,), 4, Rng(5))
    b = O.learn_ensemble_basis([L0], (8,))
    assert abs(A.spectral_corr_coeff(L0, _gb(b)) - 1.0) < 1e-6


def test_active_coherence_cases(gpu):                    # :118-142
    A = _A()
    ident = _gb(basis_from_matrix((2, 2), np.eye(4)))
    assert A.active_coherence(ident, [0, 1]) == pytest.approx(2.0)
    assert A.active_coherence(ident, [0]) == pytest.approx(4.0)
    H = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]]) / 2.0
    assert A.active_coherence(_gb(basis_from_matrix((2, 2), H)), [0, 1, 2]) == pytest.approx(1.0)


def test_conv_coherence_constant_tensor(gpu):            # :144-152
    cc = _A().conv_coherence(np.full((6, 6), 0.7), (2, 2))
    assert cc.rank == 1
    assert cc.mu1 == pytest.approx(1.0, rel=1e-10)
    assert cc.mu2 == pytest.approx(1.0, rel=1e-10)
    assert cc.tau == pytest.approx(1.0, rel=1e-10)


@pytest.mark.parametrize("seed", [46, 111])               # :154-170; acceptance criterion 11
def test_conv_coherence_random_dims_match_oracle(gpu, seed):
    A = _A()
    r = Rng(seed)
    for _ in range(50):
        dims = r.random_dims()
        kd = r.random_kernel_dims(dims)
        L = r.random_tensor(dims)
        cc = A.conv_coherence(L, kd)
        co = O.conv_coherence(L, kd)
        assert cc.rank == co.rank
        assert cc.mu1 == pytest.approx(co.mu1, rel=1e-8)
        assert cc.mu2 == pytest.approx(co.mu2, rel=1e-8)
        assert cc.tau == pytest.approx(co.tau, rel=1e-8)
        m, k = float(L.size), float(np.prod(kd))
        assert 1.0 - 1e-8 <= cc.mu1 <= m / cc.rank + 1e-8
        assert 1.0 - 1e-8 <= cc.mu2 <= k / cc.rank + 1e-8


def test_thresholds_plug_in(gpu):                        # :172-199
    A = _A()
    t = A.thresholds(A.ThresholdInputs(1, 1.0, 1.0, 1.0, 1.0, 1, 16, 16, 0.9))
    assert t.rho_min_noiseless == pytest.approx(0.5, rel=1e-12) and t.certified
    t = A.thresholds(A.ThresholdInputs(2, 1.0, 1.0, 1.0, 1.0, 2, 8, 32, 0.9))
    ref = O.thresholds(O.ThresholdInputs(2, 1.0, 1.0, 1.0, 1.0, 2, 8, 32, 0.9))
    for key in ("rho_min_noiseless", "rho_min_noisy", "error_bound_factor", "cnnm_bound",
                "icnnm_ideal_bound"):
        assert getattr(t, key) == ref[key]


def test_ideal_case_collapse(gpu):                       # :244-256
    A = _A()
    L0 = O.synth_low_conv_rank((16, 16), (4, 4), 4, Rng(77))
    b = O.learn_ensemble_basis([L0], (4, 4))
    mask = np.ones((16, 16))
    d = A.analyze_recovery(L0, _gb(b), mask)
    assert d.r_K == d.r0
    assert abs(d.alpha_K - 1.0) < 1e-6
    assert abs(d.mu_K_I - d.mu2) < 1e-6
    assert d.rho0 == 1.0
    _check_diag(d, O.analyze_recovery(L0, b, mask))


def test_diagnostics_scale_invariant(gpu):               # :258-275
    A = _A()
    r = Rng(48)
    L0 = r.random_tensor((8, 8))
    b = basis_from_matrix((3, 3), random_orthogonal(9, r))
    mask = np.ones((8, 8))
    d1 = A.analyze_recovery(L0, _gb(b), mask)
    d2 = A.analyze_recovery(-41.5 * L0, _gb(b), mask)
    assert d1.r_K == d2.r_K
    assert d1.alpha_K == pytest.approx(d2.alpha_K, rel=1e-8)
    assert d1.mu_K_I == pytest.approx(d2.mu_K_I, rel=1e-10)
    for key in ("mu1", "mu2", "tau"):
        assert getattr(d1, key) == pytest.approx(getattr(d2, key), rel=1e-7)
    _check_diag(d1, O.analyze_recovery(L0, b, mask))


def test_acceptance_ideal_diagnostics(gpu):              # criterion 4
    A = _A()
    for trial in range(5):
        L0 = O.synth_low_conv_rank((12, 12), (3, 3), 3 + trial, Rng(400 + trial))
        b = O.learn_ensemble_basis([L0], (3, 3))
        mask = one_missing_mask((12, 12), 7)
        d = A.analyze_recovery(L0, _gb(b), mask)
        c = A.conv_coherence(L0, (3, 3))
        assert d.r_K == d.r0
        assert abs(d.alpha_K - 1.0) < 1e-6
        assert abs(d.mu_K_I - c.mu2) < 1e-6
        _check_diag(d, O.analyze_recovery(L0, b, mask))


@pytest.mark.parametrize("case", ["1d", "2d"])
def test_acceptance_certified_instances(gpu, case):      # criterion 5
    A = _A()
    if case == "1d":
        L0, ks, mask = cosine_1d(32, 8), (8,), one_missing_mask((32,), 13)
    else:
        L0, ks, mask = cosine_2d(16, 4), (4, 4), one_missing_mask((16, 16), 37)
    b = O.learn_ensemble_basis([L0], ks)
    d = A.analyze_recovery(L0, _gb(b), mask)
    assert d.certified
    _check_diag(d, O.analyze_recovery(L0, b, mask))


@pytest.mark.parametrize("dims,ks", [((20, 24, 16), (3, 3, 2)), ((24, 24, 16), (5, 5, 3)),
                                     ((9, 13, 11), (4, 2, 3))])
def test_video_tensors_match_oracle(gpu, dims, ks):
    """BASELINE-recipe video (held-out target, basis learned on training
    clips, exact-rate mask): the full diagnostics record against the oracle."""
    from paper_2604_17001_b200 import synth
    A = _A()
    H, W, T = dims
    L0 = synth.synth_video(H, W, T, 3, 2, 7001)
    refs = [synth.synth_video(H, W, T, 3, 2, 7100 + i) for i in range(3)]
    b = O.learn_ensemble_basis(refs, ks)
    mask = synth.reference_bernoulli_mask(dims, 0.3, 11)
    d = A.analyze_recovery(L0, _gb(b), mask)
    _check_diag(d, O.analyze_recovery(L0, b, mask))
    import json
    j = json.loads(A.diagnostics_to_json(d))
    assert j["r_K"] == d.r_K and j["support_I"] == d.support_I and j["certified"] == d.certified


@pytest.mark.slow
def test_config2_sigma_alpha_match_oracle(gpu):
    """BASELINE config 2 (128x128x32, 9x9x5): sigma^K and alpha_K at full
    size against the oracle's FFT path; conv_coherence checked through its
    invariants (the dense 524288 x 405 SVD is out of the oracle's reach)."""
    from paper_2604_17001_b200 import synth
    A = _A()
    w = synth.WORKLOADS[2]
    X = w.target()
    from paper_2604_17001_b200 import learn_ensemble_basis
    b = learn_ensemble_basis(w.training(), w.kernel)
    ob = O.EigenBasis(tuple(w.kernel), b.K, b.eigenvalues)
    s = A.relative_eigenvalues(X, b)
    so = O.relative_eigenvalues(X, ob)
    assert np.max(np.abs(s - so)) <= 1e-10 * so.max()
    assert A.spectral_corr_coeff(X, b) == pytest.approx(O.spectral_corr_coeff(X, ob), rel=1e-9)
    d = A.analyze_recovery(X, b, w.mask())
    assert d.r_K == O.relative_conv_rank(X, ob)[0]
    k = b.K.shape[0]
    assert 1 <= d.r0 <= k and d.tau >= 1.0
    assert 1.0 - 1e-8 <= d.mu1 <= X.size / d.r0 + 1e-8
    assert 1.0 - 1e-8 <= d.mu2 <= k / d.r0 + 1e-8


def test_cli_analyze_matches_api(gpu, tmp_path):
    """`icnnm_b200 analyze` (tools/icnnm_cli.cpp:100-108,174-179) on the
    reference's TNSR/EBAS files equals the library call; errors are
    {"error": ...} with exit code 1."""
    import json
    import subprocess
    from paper_2604_17001_b200 import io as pio, synth
    from paper_2604_17001_b200._lib import CLI_PATH
    A = _A()
    dims, ks = (20, 24, 16), (3, 3, 2)
    L0 = synth.synth_video(*dims, 3, 2, 7001)
    b = gpu.learn_ensemble_basis([synth.synth_video(*dims, 3, 2, 7100)], ks)
    mask = synth.reference_bernoulli_mask(dims, 0.3, 11)
    pio.write_tnsr(str(tmp_path / "L0.tnsr"), L0)
    pio.write_tnsr(str(tmp_path / "mask.tnsr"), mask)
    pio.write_ebas(str(tmp_path / "b.ebas"), b)
    args = [CLI_PATH, "analyze", "--target", str(tmp_path / "L0.tnsr"), "--basis",
            str(tmp_path / "b.ebas"), "--mask", str(tmp_path / "mask.tnsr"), "--out",
            str(tmp_path / "d.json")]
    out = subprocess.run(args, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    j = json.loads((tmp_path / "d.json").read_text())
    d = A.analyze_recovery(L0, b, mask)
    assert j["r_K"] == d.r_K and j["support_I"] == d.support_I and j["r0"] == d.r0
    for key in ("alpha_K", "mu_K_I", "mu1", "mu2", "tau", "rho0", "rho_min_noiseless"):
        assert j[key] == getattr(d, key), key
    pio.write_tnsr(str(tmp_path / "bad.tnsr"), np.full(dims, 0.5))
    out = subprocess.run(args[:6] + ["--mask", str(tmp_path / "bad.tnsr"), "--out",
                                     str(tmp_path / "d2.json")], capture_output=True, text=True)
    assert out.returncode == 1 and json.loads(out.stderr)["error"].startswith("SamplingMask")
