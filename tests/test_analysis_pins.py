"""Pin the oracle's recovery-theory diagnostics (oracle.analyze_recovery & co.,
restating core/src/analysis.cpp) against the reference's own known-answer
tests: /root/reference/proj/tests/test_analysis.cpp and the analysis
criteria of test_acceptance.cpp (4, 5, 7, 11).  Inputs are rebuilt from the
same mt19937_64 streams (synth.Rng); test helpers live in analysis_cases.py
so the GPU parity tests (test_gpu_analysis.py) replay the very same cases.
"""
import numpy as np
import pytest

from oracle import icnnm_oracle as O
from analysis_cases import (Rng, basis_from_matrix, cosine_1d, cosine_2d, one_missing_mask,
                            random_orthogonal)


def test_own_basis_recovers_conv_rank():                 # test_analysis.cpp:43-50
    L0 = O.synth_low_conv_rank((16, 16), (4, 4), 4, Rng(99))
    basis = O.learn_ensemble_basis([L0], (4, 4))
    rk, sup = O.relative_conv_rank(L0, basis)
    assert rk == O.conv_spectrum(L0, (4, 4)).rank
    assert len(sup) == rk


def test_zero_tensor_empty_support():                    # :52-59
    basis = basis_from_matrix((2, 2), random_orthogonal(4, Rng(41)))
    rk, sup = O.relative_conv_rank(np.zeros((5, 5)), basis)
    assert rk == 0 and sup == []


def test_rank_matches_column_norm_oracle():              # :61-77
    r = Rng(42)
    for _ in range(10):
        L0 = r.random_tensor((6, 6))
        basis = basis_from_matrix((2, 2), random_orthogonal(4, r))
        rk, _ = O.relative_conv_rank(L0, basis)
        norms = np.linalg.norm(O.conv_matrix(L0, (2, 2)) @ basis.K, axis=0)
        assert rk == int(np.sum(norms > 1e-8 * norms.max()))


def test_exact_basis_alpha_one():                        # :79-85
    L0 = O.synth_low_conv_rank((32,), (8,), 4, Rng(5))
    basis = O.learn_ensemble_basis([L0], (8,))
    assert abs(O.spectral_corr_coeff(L0, basis) - 1.0) < 1e-6


def test_alpha_bounds_and_explicit_oracle():             # :87-109
    r = Rng(43)
    for _ in range(100):
        L0 = r.random_tensor((6, 6))
        basis = basis_from_matrix((2, 2), random_orthogonal(4, r))
        rk, sup = O.relative_conv_rank(L0, basis)
        alpha = O.spectral_corr_coeff(L0, basis)
        assert alpha >= 1.0 - 1e-8
        assert alpha <= np.sqrt(rk) + 1e-8
        AK = O.conv_matrix(L0, (2, 2)) @ basis.K
        B = AK[:, sup] / np.linalg.norm(AK[:, sup], axis=0)
        assert alpha == pytest.approx(np.linalg.svd(B, compute_uv=False)[0], rel=1e-7)


def test_alpha_zero_target_is_error():                   # :111-116
    basis = basis_from_matrix((2, 2), random_orthogonal(4, Rng(44)))
    with pytest.raises(ValueError):
        O.spectral_corr_coeff(np.zeros((4, 4)), basis)


def test_active_coherence_cases():                       # :118-142
    ident = basis_from_matrix((2, 2), np.eye(4))
    assert O.active_coherence(ident, [0, 1]) == pytest.approx(2.0)
    assert O.active_coherence(ident, [0]) == pytest.approx(4.0)
    H = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]]) / 2.0
    assert O.active_coherence(basis_from_matrix((2, 2), H), [0, 1, 2]) == pytest.approx(1.0)
    r = Rng(45)
    for _ in range(50):
        rb = basis_from_matrix((2, 2), random_orthogonal(4, r))
        n = int(r.uniform_int(1, 4)[0])
        mu = O.active_coherence(rb, list(range(n)))
        assert 1.0 - 1e-10 <= mu <= 4.0 / n + 1e-10
    with pytest.raises(ValueError):
        O.active_coherence(ident, [])


def test_conv_coherence_constant_tensor():               # :144-152
    cc = O.conv_coherence(np.full((6, 6), 0.7), (2, 2))
    assert cc.rank == 1
    assert cc.mu1 == pytest.approx(1.0, rel=1e-10)
    assert cc.mu2 == pytest.approx(1.0, rel=1e-10)
    assert cc.tau == pytest.approx(1.0, rel=1e-10)


def test_conv_coherence_range_bounds():                  # :154-170
    r = Rng(46)
    for _ in range(50):
        dims = r.random_dims()
        kd = r.random_kernel_dims(dims)
        L = r.random_tensor(dims)
        cc = O.conv_coherence(L, kd)
        m, k = float(L.size), float(np.prod(kd))
        assert 1.0 - 1e-8 <= cc.mu1 <= m / k * cc.tau ** 2 + 1e-8
        assert 1.0 - 1e-8 <= cc.mu2 <= cc.tau ** 2 + 1e-8
    with pytest.raises(ValueError):
        O.conv_coherence(np.zeros((4, 4)), (2, 2))


def test_thresholds_plug_in():                           # :172-199
    t = O.thresholds(O.ThresholdInputs(1, 1.0, 1.0, 1.0, 1.0, 1, 16, 16, 0.9))
    assert t["rho_min_noiseless"] == pytest.approx(0.5, rel=1e-12)
    assert t["certified"]
    t = O.thresholds(O.ThresholdInputs(2, 1.0, 1.0, 1.0, 1.0, 2, 8, 32, 0.9))
    assert t["rho_min_noiseless"] == pytest.approx(1.0 - 8.0 / (2.0 * 1.0 * 2.0 * 32.0), rel=1e-12)
    assert t["rho_min_noisy"] == pytest.approx(1.0 - 0.64 * 8.0 / ((0.64 + 1.0) * 2.0 * 32.0),
                                               rel=1e-12)
    assert t["error_bound_factor"] == pytest.approx((18.0 * np.sqrt(8.0) + 2.0) * (1.0 + np.sqrt(2.0)),
                                                    rel=1e-12)


def test_thresholds_monotone():                          # :201-222
    base = O.ThresholdInputs(2, 1.5, 1.2, 1.0, 1.0, 2, 16, 256, 0.0)
    t0 = O.thresholds(base)["rho_min_noiseless"]
    import dataclasses
    for bump in (1.1, 1.5, 3.0):
        assert O.thresholds(dataclasses.replace(base, alpha_K=base.alpha_K * bump))["rho_min_noiseless"] > t0
        assert O.thresholds(dataclasses.replace(base, mu_K_I=base.mu_K_I * bump))["rho_min_noiseless"] > t0
    assert O.thresholds(dataclasses.replace(base, r_K=3))["rho_min_noiseless"] > t0


def test_ideal_bound_never_exceeds_baseline():           # :224-242
    r = Rng(47)
    for _ in range(1000):
        mu1, mu2 = r.uniform(1.0, 50.0, 1)[0], r.uniform(1.0, 50.0, 1)[0]
        r0 = int(r.uniform_int(1, 20)[0])
        t = O.thresholds(O.ThresholdInputs(r0, 1.0, mu2, mu1, mu2, r0, 16, 1024, 0.0))
        assert t["icnnm_ideal_bound"] <= t["cnnm_bound"]


def test_ideal_case_collapse():                          # :244-256
    L0 = O.synth_low_conv_rank((16, 16), (4, 4), 4, Rng(77))
    basis = O.learn_ensemble_basis([L0], (4, 4))
    d = O.analyze_recovery(L0, basis, np.ones((16, 16)))
    assert d["r_K"] == d["r0"]
    assert abs(d["alpha_K"] - 1.0) < 1e-6
    assert abs(d["mu_K_I"] - d["mu2"]) < 1e-6
    assert d["rho0"] == 1.0


def test_diagnostics_scale_invariant():                  # :258-275
    r = Rng(48)
    L0 = r.random_tensor((8, 8))
    basis = basis_from_matrix((3, 3), random_orthogonal(9, r))
    mask = np.ones((8, 8))
    d1 = O.analyze_recovery(L0, basis, mask)
    d2 = O.analyze_recovery(-41.5 * L0, basis, mask)
    assert d1["r_K"] == d2["r_K"]
    assert d1["alpha_K"] == pytest.approx(d2["alpha_K"], rel=1e-8)
    assert d1["mu_K_I"] == pytest.approx(d2["mu_K_I"], rel=1e-10)
    for key in ("mu1", "mu2", "tau"):
        assert d1[key] == pytest.approx(d2[key], rel=1e-7)


# --- test_acceptance.cpp --------------------------------------------------------
def test_acceptance_ideal_diagnostics():                 # criterion 4, :152-168
    for trial in range(5):
        L0 = O.synth_low_conv_rank((12, 12), (3, 3), 3 + trial, Rng(400 + trial))
        basis = O.learn_ensemble_basis([L0], (3, 3))
        d = O.analyze_recovery(L0, basis, one_missing_mask((12, 12), 7))
        c = O.conv_coherence(L0, (3, 3))
        assert d["r_K"] == d["r0"]
        assert abs(d["alpha_K"] - 1.0) < 1e-6
        assert abs(d["mu_K_I"] - c.mu2) < 1e-6


@pytest.mark.parametrize("case", ["1d", "2d"])
def test_acceptance_certified_instances(case):           # criterion 5, :177-209
    if case == "1d":
        L0, ks, mask = cosine_1d(32, 8), (8,), one_missing_mask((32,), 13)
    else:
        L0, ks, mask = cosine_2d(16, 4), (4, 4), one_missing_mask((16, 16), 37)
    basis = O.learn_ensemble_basis([L0], ks)
    d = O.analyze_recovery(L0, basis, mask)
    assert d["certified"]


def test_acceptance_bound_ordering():                    # criterion 7, :236-256
    r = Rng(107)
    for _ in range(1000):
        u = lambda: float(r.uniform(0.0, 1.0, 1)[0])
        k = 4 + int(u() * 60)
        m = k * (2 + int(u() * 30))
        r0 = 1 + int(u() * float(k - 1))
        mu1 = 1.0 + u() * 4.0
        mu2 = 1.0 + u() * 4.0
        rho0 = u()
        t = O.thresholds(O.ThresholdInputs(r0, 1.0, mu2, mu1, mu2, r0, k, m, rho0))
        assert t["icnnm_ideal_bound"] <= t["cnnm_bound"]


def test_acceptance_coherence_ranges():                  # criterion 11, :326-343
    r = Rng(111)
    for _ in range(50):
        dims = r.random_dims()
        kd = r.random_kernel_dims(dims)
        L = r.random_tensor(dims)
        c = O.conv_coherence(L, kd)
        m, k, rr = float(L.size), float(np.prod(kd)), float(c.rank)
        assert 1.0 - 1e-8 <= c.mu1 <= m / rr + 1e-8
        assert 1.0 - 1e-8 <= c.mu2 <= k / rr + 1e-8
        assert c.tau >= 1.0 - 1e-8
