"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): index maps and integer-valued
operator outputs bit-exact; fp32 operators within 1e-5 relative of the fp64
oracle; recovered tensors within relative L2 1e-4 and PSNR within 0.01 dB
after a fixed iteration count.  Inputs of the reference's own known-answer
tests are rebuilt from libstdc++'s mt19937_64 streams (synth.Rng).
"""
import numpy as np
import pytest

from oracle import icnnm_oracle as O

pytestmark = pytest.mark.gpu

FIXED = dict(tol_primal=1e-300, tol_change=1e-300)
ENGINES = ["ffma", "tf32x3", "f16x3"]


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _ab_lib():
    """The experiments build of the library (environment A/B knobs); the
    product build ignores the environment, so knob tests run against it."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "build", "ab", "libicnnm_b200_ab.so")
    if not os.path.exists(path):
        pytest.skip("experiments build missing (make -C paper_2604_17001_b200/csrc EXPERIMENTS=1)")
    return path


def _rand_orth(k, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((k, k)))
    return q


# --------------------------------------------------------------------------
# operators
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dims,ks", [((32, 32, 8), (5, 5, 3)), ((7, 5, 9), (3, 2, 4)),
                                     ((5, 4), (3, 3)), ((12,), (5,)), ((3, 3, 3), (3, 3, 3)),
                                     ((20, 33, 17), (9, 1, 5)), ((6, 6, 40), (1, 6, 13))])
@pytest.mark.parametrize("engine", ENGINES)
def test_forward_index_map_bit_exact(gpu, dims, ks, engine):
    """K = I on integer-valued L: A(L) must equal conv_matrix exactly
    (pins the corner-anchored periodic index map, conv_op.cpp:35-46)."""
    rng = np.random.default_rng(1)
    L = rng.integers(-8, 9, size=dims).astype(np.float64)
    k = int(np.prod(ks))
    out = gpu.BasisConvolver(dims, ks, np.eye(k), engine=engine).apply(L)
    np.testing.assert_array_equal(out, O.conv_matrix(L, ks))


@pytest.mark.parametrize("dims,ks", [((32, 32, 8), (5, 5, 3)), ((16, 16, 32), (9, 9, 5)),
                                     ((9, 7, 11), (3, 4, 2)), ((6, 5), (2, 3)),
                                     ((24, 24, 16), (13, 13, 7))])
@pytest.mark.parametrize("engine", ENGINES)
def test_forward_matches_basis_convolver(gpu, dims, ks, engine):
    rng = np.random.default_rng(2)
    L = rng.uniform(-1, 1, size=dims)
    k = int(np.prod(ks))
    K = _rand_orth(k, 3)
    got = gpu.BasisConvolver(dims, ks, K, engine=engine).apply(L)
    ref = O.BasisConvolver(dims, ks, K).apply(L)
    # fp32 FFMA: ~1e-7; TF32x3 (tensor-core fp32 accumulate): ~1e-6 at k ~ 1e3
    assert _rel(got, ref) < (1e-6 if engine == "ffma" else 1e-5)


@pytest.mark.parametrize("dims,ks", [((32, 32, 8), (5, 5, 3)), ((5, 6, 7), (2, 3, 4)),
                                     ((4, 4), (2, 2)), ((10,), (4,)), ((8, 8, 16), (8, 8, 3)),
                                     ((20, 20, 16), (9, 9, 5)),
                                     # k = 245: the adjoint runs on CTA pairs with resident B
                                     # halves (even and odd brick counts: dummy tail brick)
                                     ((16, 24, 16), (7, 7, 5)), ((12, 12, 8), (7, 7, 5)),
                                     ((20, 12, 24), (7, 7, 5))])
@pytest.mark.parametrize("engine", ENGINES)
def test_adjoint_bit_exact_on_integers(gpu, dims, ks, engine):
    """conv_adjoint (conv_op.cpp:57-77) on integer W: exact in fp32."""
    rng = np.random.default_rng(4)
    m, k = int(np.prod(dims)), int(np.prod(ks))
    W = rng.integers(-4, 5, size=(m, k)).astype(np.float64)
    np.testing.assert_array_equal(gpu.conv_adjoint(W, ks, dims, engine=engine),
                                  O.conv_adjoint(W, ks, dims))


def test_adjointness_and_composition(gpu):
    """<A(L), W> = <L, A*(W)> and A*A = k Id (test_tensor_core.cpp:124-146)."""
    r = gpu.synth.Rng(14)
    for _ in range(20):
        dims = r.random_dims()
        kd = r.random_kernel_dims(dims)
        L = r.random_tensor(dims)
        m, k = L.size, int(np.prod(kd))
        W = np.random.default_rng(k * m).uniform(-1, 1, size=(m, k))
        adj = gpu.conv_adjoint(W, kd, dims)
        A = O.conv_matrix(L, kd)
        lhs = float(np.sum(A * W))
        rhs = float(np.sum(L * adj))
        assert abs(lhs - rhs) < 1e-5 * (np.linalg.norm(W) * np.linalg.norm(L) + 1.0)
        comp = gpu.conv_adjoint(A, kd, dims)
        assert np.linalg.norm(comp - k * L) < 1e-5 * k * np.linalg.norm(L)


def test_adjoint_zero_and_shape_errors(gpu):
    dims, ks = (4, 4), (2, 2)
    assert np.linalg.norm(gpu.conv_adjoint(np.zeros((16, 4)), ks, dims)) == 0.0
    with pytest.raises(gpu.InvalidArgument):
        gpu.conv_adjoint(np.zeros((15, 4)), ks, dims)
    with pytest.raises(gpu.InvalidArgument):
        gpu.conv_adjoint(np.zeros((16, 5)), ks, dims)


def test_forward_rejects_bad_shapes(gpu):
    L = np.zeros((4, 4))
    with pytest.raises(gpu.InvalidArgument):
        gpu.BasisConvolver((4, 4), (5, 2), np.eye(10)).apply(L)
    with pytest.raises(gpu.InvalidArgument):
        gpu.BasisConvolver((4, 4), (2, 2), np.eye(3))


def test_prox_known_answers(gpu):
    """prox_l21 KATs (test_solver.cpp:50-80,99-109)."""
    W = np.random.default_rng(5).uniform(-1, 1, size=(10, 4))
    assert np.linalg.norm(gpu.prox_l21(W, 0.0) - W) == 0.0
    W = np.zeros((4, 2))
    W[0, 0] = 2.0
    W[1, 1] = 0.4
    Z = gpu.prox_l21(W, 0.5)
    assert abs(np.linalg.norm(Z[:, 0]) - 1.5) < 1e-12
    assert abs(Z[0, 0] - 1.5) < 1e-12
    assert np.linalg.norm(Z[:, 1]) == 0.0
    W = np.random.default_rng(6).uniform(-1, 1, size=(15, 8))
    Z = gpu.prox_l21(W, 0.4)
    np.testing.assert_allclose(np.linalg.norm(Z, axis=0),
                               np.maximum(0, np.linalg.norm(W, axis=0) - 0.4), rtol=1e-12,
                               atol=1e-15)
    np.testing.assert_allclose(Z, O.prox_l21(W, 0.4), rtol=1e-12, atol=1e-15)
    with pytest.raises(gpu.InvalidArgument):
        gpu.prox_l21(W, -1.0)


def test_gram_matches_explicit(gpu):
    """conv_gram == A^T A (test_spectral.cpp:29-41), fp64 accumulation."""
    r = gpu.synth.Rng(21)
    for _ in range(20):
        dims = r.random_dims()
        kd = r.random_kernel_dims(dims)
        L = r.random_tensor(dims)
        G = gpu.conv_gram(L, kd)
        A = O.conv_matrix(L, kd)
        E = A.T @ A
        assert np.max(np.abs(G - E)) < 1e-10 * (1.0 + np.linalg.norm(E))


def test_gram_large_kernel_matches_oracle(gpu):
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(48, 40, 24, 8, 2, 7)
    for ks in [(9, 9, 5), (13, 13, 7), (7, 7, 5)]:
        G = gpu.conv_gram(X, ks)
        E = O.conv_gram(X, ks)
        assert np.max(np.abs(G - E)) < 1e-10 * np.max(np.abs(E))


def test_gram_generic_kernel_and_mirror(gpu):
    """Frame kernels beyond the register-tiled Gram kernel's range (kt > 9)
    take the lag-per-thread kernel; both give an exactly symmetric Gram."""
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(20, 24, 40, 6, 1, 11)
    for ks in [(3, 4, 11), (5, 6, 9), (2, 3, 1), (1, 1, 7)]:
        G = gpu.conv_gram(X, ks)
        E = O.conv_gram(X, ks)
        assert np.max(np.abs(G - E)) < 1e-10 * np.max(np.abs(E)), ks
        if ks[2] <= 9:
            np.testing.assert_array_equal(G, G.T)


@pytest.mark.parametrize("cfgno", [1, 2, 3])
def test_learn_basis_matches_oracle(gpu, cfgno):
    """learn_ensemble_basis: eigenvalues + per-block projectors
    (test_spectral.cpp:112-137), at the kernels and training sets of BASELINE
    configs 1-3 (k = 75, 405, 1183)."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[cfgno]
    refs = w.training()
    got = gpu.learn_ensemble_basis(refs, w.kernel)
    ref = O.learn_ensemble_basis(refs, w.kernel)
    k = w.k
    # sigma = sqrt(lambda): compare lambda, whose rounding floor is ~eps*lambda_1
    np.testing.assert_allclose(got.eigenvalues ** 2, ref.eigenvalues ** 2, rtol=1e-8,
                               atol=1e-11 * ref.eigenvalues[0] ** 2)
    assert np.max(np.abs(got.K.T @ got.K - np.eye(k))) < 1e-10
    lam = ref.eigenvalues ** 2          # Gram eigenvalues
    l1 = lam[0]
    start = 0
    while start < k:
        end = start + 1
        while end < k and abs(lam[end] - lam[start]) < 1e-6 * l1:
            end += 1
        gap = min(lam[start - 1] - lam[start] if start > 0 else np.inf,
                  lam[end - 1] - lam[end] if end < k else np.inf)
        if lam[start] > 1e-8 * l1 and gap > 0:
            b = got.K[:, start:end]
            v = ref.K[:, start:end]
            # Davis-Kahan: ||P - P'|| <~ ||dG|| / gap with ||dG|| ~ 1e-13 lambda_1
            tol = max(1e-6, 1e-11 * l1 / gap)
            assert np.linalg.norm(b @ b.T - v @ v.T) < tol, (start, end, tol)
        start = end


def test_learn_basis_is_deterministic(gpu):
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    refs = w.training()
    a = gpu.learn_ensemble_basis(refs, w.kernel)
    b = gpu.learn_ensemble_basis(refs, w.kernel)
    np.testing.assert_array_equal(a.K, b.K)
    np.testing.assert_array_equal(a.eigenvalues, b.eigenvalues)


def test_learn_basis_degenerate_and_errors(gpu):
    b = gpu.learn_ensemble_basis([np.zeros((4, 4))], (2, 2))
    assert b.degenerate and np.array_equal(b.K, np.eye(4))
    with pytest.raises(gpu.InvalidArgument):
        gpu.learn_ensemble_basis([], (2, 2))
    with pytest.raises(gpu.InvalidArgument):
        gpu.learn_ensemble_basis([np.ones((4, 4)), np.ones((5, 4))], (2, 2))


def test_own_basis_l21_is_nuclear_norm(gpu):
    """l21(A K) with K the tensor's own basis == ||A||_* (test_spectral.cpp:99-110)."""
    r = gpu.synth.Rng(25)
    for _ in range(5):
        L = r.random_tensor((6, 6))
        b = gpu.learn_ensemble_basis([L], (3, 3))
        AK = gpu.BasisConvolver((6, 6), (3, 3), b.K).apply(L)
        l21 = np.sum(np.linalg.norm(AK, axis=0))
        nuc = np.sum(np.linalg.svd(O.conv_matrix(L, (3, 3)), compute_uv=False))
        assert abs(l21 - nuc) < 1e-5 * nuc


def test_objective_matches_explicit(gpu):
    """objective_icnnm vs explicit-matrix oracle (test_solver.cpp:195-216)."""
    r = gpu.synth.Rng(36)
    ref = r.random_tensor((5, 5))
    b = gpu.learn_ensemble_basis([ref], (2, 2))
    L = r.random_tensor((5, 5))
    M = r.random_tensor((5, 5))
    mask = gpu.synth.reference_bernoulli_mask((5, 5), 0.6, 3)
    fast = gpu.objective_icnnm(L, M, mask, b, 1000.0)
    A = O.conv_matrix(L, (2, 2))
    fit = np.sum(((L - M) * mask) ** 2)
    oracle = np.sum(np.linalg.norm(A @ b.K, axis=0)) + 0.5 * 1000.0 * 4.0 * fit
    assert abs(fast - oracle) < 1e-6 * (1.0 + oracle)
    z = np.zeros((5, 5))
    assert gpu.objective_icnnm(z, z, np.ones((5, 5)), b, 1000.0) == 0.0


# --------------------------------------------------------------------------
# solver
# --------------------------------------------------------------------------
def _oracle_basis(B):
    return O.EigenBasis(tuple(B.kernel_shape), B.K, B.eigenvalues, B.degenerate)


@pytest.mark.parametrize("engine", ENGINES)
def test_solve_config1_full_parity(gpu, engine):
    """BASELINE config 1 (32x32x8, 5x5x3, 200 iterations): GPU vs oracle."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    X = w.target()
    mask = w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    M = X * mask
    Lg, rg = gpu.icnnm_solve(M, mask, B, gpu.SolverConfig(max_iters=w.iters, engine=engine,
                                                          **FIXED))
    Lo, ro = O.icnnm_solve(M, mask, _oracle_basis(B),
                           O.SolverConfig(max_iters=w.iters, **FIXED))
    assert rg.iterations == w.iters and rg.termination == "max_iters"
    assert _rel(Lg, Lo) <= 1e-4
    assert abs(synth.psnr(X, Lg) - O.psnr(X, Lo)) <= 0.01
    np.testing.assert_allclose(rg.objective, ro.objective, rtol=1e-4)
    np.testing.assert_allclose(rg.l_change, ro.l_change, rtol=1e-2, atol=1e-6)
    # residual trace: fp32 identity estimate, exact while the
    # gap is resolvable, NaN below the fp32 floor -- never a spurious value
    res = np.array(rg.primal_residual)
    ok = ~np.isnan(res)
    assert ok[0]
    np.testing.assert_allclose(res[0], ro.primal_residual[0], rtol=2e-3)
    assert np.all(res[ok] < 1.0)


@pytest.mark.parametrize("dims,ks,iters,rate", [((24, 20, 16), (5, 3, 3), 150, 0.3),
                                                ((16, 16, 32), (9, 9, 5), 60, 0.2),
                                                ((20, 24), (4, 5), 100, 0.5),
                                                ((32, 32, 24), (13, 13, 7), 40, 0.3)])
@pytest.mark.parametrize("engine", ENGINES)
def test_solve_small_parity(gpu, dims, ks, iters, rate, engine):
    from paper_2604_17001_b200 import synth
    full = dims if len(dims) == 3 else (1,) + tuple(dims)
    X = synth.synth_video(*full, 8, 2, 11).reshape(dims)
    refs = [synth.synth_video(*full, 8, 2, 100 + i).reshape(dims) for i in range(3)]
    mask = synth.reference_bernoulli_mask(dims, rate, 9)
    B = gpu.learn_ensemble_basis(refs, ks)
    Lg, rg = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=iters, engine=engine,
                                                                  **FIXED))
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B),
                          O.SolverConfig(max_iters=iters, **FIXED))
    assert _rel(Lg, Lo) <= 1e-4
    assert abs(synth.psnr(X, Lg) - O.psnr(X, Lo)) <= 0.01


def test_solve_mean_fill_and_theta0(gpu):
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(16, 16, 8, 6, 1, 5)
    mask = synth.reference_bernoulli_mask(X.shape, 0.4, 2)
    B = gpu.learn_ensemble_basis([synth.synth_video(16, 16, 8, 6, 1, 6)], (3, 3, 3))
    for kw in [dict(init_fill="mean"), dict(theta0=3.0, theta_growth=1.1),
               dict(lambda_=50.0, theta_max=1e3)]:
        Lg, _ = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=80, **FIXED, **kw))
        Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B),
                              O.SolverConfig(max_iters=80, **FIXED, **kw))
        assert _rel(Lg, Lo) <= 1e-4, kw


def test_solve_fully_observed_returns_input(gpu):
    """test_solver.cpp:111-120: fully observed 8x8, kernel 3x3, 300 iters."""
    M = gpu.synth.Rng(33).random_tensor((8, 8))
    B = gpu.learn_ensemble_basis([M], (3, 3))
    L, _ = gpu.icnnm_solve(M, np.ones_like(M), B, gpu.SolverConfig(max_iters=300))
    assert _rel(L, M) < 1e-3


def test_solve_exact_cosine_recovery(gpu):
    """test_solver.cpp:122-138: rank-2 cosine, m=32, k=8, Bernoulli .75 seed 5."""
    L0 = np.cos(2 * np.pi * np.arange(32) / 8)
    B = gpu.learn_ensemble_basis([L0], (8,))
    mask = gpu.synth.reference_bernoulli_mask((32,), 0.75, 5)
    L, rep = gpu.icnnm_solve(L0 * mask, mask, B, gpu.SolverConfig())
    assert _rel(L, L0) < 1e-3
    Lo, ro = O.icnnm_solve(L0 * mask, mask, _oracle_basis(B), O.SolverConfig())
    assert ro.termination == "converged"
    assert _rel(L, Lo) < 1e-4


def test_solve_objective_trace_decreases(gpu):
    """test_solver.cpp:218-245: objective non-increasing after burn-in."""
    L0 = np.cos(2 * np.pi * np.arange(32) / 8)
    B = gpu.learn_ensemble_basis([L0], (8,))
    mask = gpu.synth.reference_bernoulli_mask((32,), 0.75, 7)
    _, rep = gpu.icnnm_solve(L0 * mask, mask, B, gpu.SolverConfig(max_iters=400, **FIXED))
    obj = rep.objective
    burn = len(obj) // 2
    for i in range(burn, len(obj) - 1):
        assert obj[i + 1] <= obj[i] * (1 + 1e-4) + 1e-6


def test_solve_errors(gpu):
    r = gpu.synth.Rng(34)
    M = r.random_tensor((4, 4))
    B = gpu.learn_ensemble_basis([M], (2, 2))
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(M, np.zeros((4, 4)), B)                   # empty mask
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(M, np.full((4, 4), 0.5), B)               # non-binary mask
    bad = M.copy()
    bad[0, 0] = np.nan
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(bad, np.ones((4, 4)), B)                  # non-finite
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(M, np.ones((4, 4)), B, gpu.SolverConfig(lambda_=-1))
    nonorth = gpu.EigenBasis((2, 2), B.K * 1.01, B.eigenvalues)
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(M, np.ones((4, 4)), nonorth)
    with pytest.raises(gpu.InvalidArgument):
        gpu.icnnm_solve(M, np.ones((5, 4)), B)


def test_handle_api_equals_one_shot(gpu):
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    cfg = gpu.SolverConfig(max_iters=50, **FIXED)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    with gpu.Solver(X.shape, B) as S:
        S.upload(X * mask, mask)
        r2 = S.run(cfg)
        L2 = S.download()
        assert S.last_launches >= 4 * 50
        r3 = S.run(cfg)  # re-run from the same staged problem
        L3 = S.download()
    assert _rel(L2, L1) < 1e-6 and _rel(L3, L1) < 1e-6
    assert r2.iterations == r3.iterations == 50


def test_device_cache_reuse_across_sizes_and_empty(gpu):
    """Device blocks freed by one call are reused by the next (icnnm_host.cu
    devcache): interleaved solves of two sizes and engines, a cache flush in
    between, and every result still equals the first solve of its problem."""
    from paper_2604_17001_b200 import synth
    probs = []
    for dims, rate, seed in [((32, 32, 8), 0.5, 3), ((24, 20, 16), 0.4, 4)]:
        w = synth.scaled(synth.WORKLOADS[1], dims, iters=30)
        X = w.target()
        mask = (np.random.default_rng(seed).random(dims) < rate).astype(np.float64)
        B = gpu.learn_ensemble_basis(w.training(), w.kernel)
        probs.append((X * mask, mask, B))
    ref = {}
    for rnd in range(3):
        for i, (M, mask, B) in enumerate(probs):
            for eng in ("f16x3", "ffma"):
                L, r = gpu.icnnm_solve(M, mask, B, gpu.SolverConfig(max_iters=30, engine=eng, **FIXED))
                assert r.iterations == 30 and np.all(np.isfinite(L))
                if (i, eng) not in ref:
                    ref[(i, eng)] = L
                else:
                    assert _rel(L, ref[(i, eng)]) < 1e-6
        if rnd == 1:
            gpu.empty_cache()


@pytest.mark.parametrize("engine", ENGINES)
def test_sharded_virtual_slabs_match_unsharded(gpu, engine):
    """H-sharded iteration (halo exchange + norm all-reduce) with G virtual
    slabs on one device equals the unsharded solve."""
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(48, 16, 16, 8, 2, 21)
    mask = synth.synth_mask(48, 16, 16, synth.MASK_IID, 0.3, 22)
    mask[20:30, 3:9, 4:12] = 0.0  # a missing box crossing slab boundaries
    B = gpu.learn_ensemble_basis([synth.synth_video(48, 16, 16, 8, 2, 23)], (5, 3, 3))
    cfg = gpu.SolverConfig(max_iters=60, engine=engine, **FIXED)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B), O.SolverConfig(max_iters=60, **FIXED))
    assert _rel(L1, Lo) < 1e-4
    for G in (1, 2, 3, 4):
        row0, rows, rep = gpu.sharded_solve(X * mask, mask, B, cfg, local_slabs=G)
        assert row0 == 0 and rows.shape == X.shape
        assert _rel(rows, L1) < 1e-5, G
        np.testing.assert_allclose(rep.objective, r1.objective, rtol=1e-5)


def test_sharded_virtual_slabs_k245_pairs(gpu):
    """The same with the 7x7x5 kernel (k = 245): the adjoint runs on CTA pairs
    with resident B halves, here on slab geometry (halo rows, no H wrap inside a
    slab) and through the sharded solve's separate pair-fold kernel."""
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(48, 24, 16, 8, 2, 31)
    mask = synth.synth_mask(48, 24, 16, synth.MASK_IID, 0.4, 32)
    B = gpu.learn_ensemble_basis([synth.synth_video(48, 24, 16, 8, 2, 33)], (7, 7, 5))
    cfg = gpu.SolverConfig(max_iters=30, engine="f16x3", **FIXED)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    for G in (1, 2, 3):
        row0, rows, rep = gpu.sharded_solve(X * mask, mask, B, cfg, local_slabs=G)
        assert row0 == 0 and rows.shape == X.shape
        assert _rel(rows, L1) < 1e-5, G
        np.testing.assert_allclose(rep.objective, r1.objective, rtol=1e-5)


# --------------------------------------------------------------------------
# BASELINE recipes at oracle-feasible sizes (same generator, mask kind and
# kernel box as configs 3-5; SURVEY §8c parity plan for the large configs)
# --------------------------------------------------------------------------
def _recipe(cfg, dims, iters):
    from paper_2604_17001_b200 import synth
    w = synth.scaled(synth.WORKLOADS[cfg], dims, iters=iters, n_train=3)
    if cfg == 3:   # frames 0..(5/6 T) observed, the tail missing (40 of 48)
        mask = synth.synth_mask(*dims, synth.MASK_T_PREFIX, int(dims[2] * 40 / 48), 0)
    elif cfg == 5:
        mask = synth.synth_mask(*dims, synth.MASK_IID_BOXES, 0.3, 3005, n_boxes=2)
    else:
        mask = w.mask()
    return w, w.target(), mask


@pytest.mark.parametrize("cfg,dims,iters", [(3, (24, 24, 24), 30), (4, (32, 32, 16), 60),
                                            (5, (32, 24, 18), 40)])
@pytest.mark.parametrize("engine", ENGINES)
def test_recipe_parity(gpu, cfg, dims, iters, engine):
    from paper_2604_17001_b200 import synth
    w, X, mask = _recipe(cfg, dims, iters)
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    Lg, _ = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=iters, engine=engine,
                                                                **FIXED))
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B),
                          O.SolverConfig(max_iters=iters, **FIXED))
    assert _rel(Lg, Lo) <= 1e-4
    miss = mask == 0
    assert _rel(Lg[miss], Lo[miss]) <= 1e-3          # the recovered (unobserved) entries
    assert abs(synth.psnr(X, Lg) - O.psnr(X, Lo)) <= 0.01


@pytest.mark.parametrize("engine", ENGINES)
def test_config5_sharded_recipe(gpu, engine):
    """Config 5's kernel (9x9x9) and mask recipe, H-sharded over 2 and 4 virtual
    slabs, against the fp64 oracle and the unsharded GPU solve."""
    from paper_2604_17001_b200 import synth
    w, X, mask = _recipe(5, (48, 24, 20), 30)
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    cfg = gpu.SolverConfig(max_iters=30, engine=engine, **FIXED)
    L1, _ = gpu.icnnm_solve(X * mask, mask, B, cfg)
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B), O.SolverConfig(max_iters=30, **FIXED))
    assert _rel(L1, Lo) <= 1e-4
    for G in (2, 4):
        _, rows, _ = gpu.sharded_solve(X * mask, mask, B, cfg, local_slabs=G)
        assert _rel(rows, Lo) <= 1e-4, G
        assert _rel(rows, L1) <= 1e-5, G


@pytest.mark.parametrize("engine", ["f16x3", "tf32x3"])
def test_config5_recipe_golden_sharded(gpu, engine):
    """Config 5's recipe (kernel 9x9x9, k = 729; 30% i.i.d. minus boxes) at
    128x128x64, 100 iterations, against the fp64 oracle golden
    (cfg5_128x128x64_it100.npz, blocked oracle): the unsharded solve, G = 1,
    2, 4, 8 virtual slabs, and G = 2 through the one-rank NCCL transport --
    the adjoint wrap across slab boundaries (conv_op.cpp:57-77) and the loop
    (solver.cpp:107-139) at the survey's size."""
    import os
    from paper_2604_17001_b200 import synth
    path = os.path.join(os.path.dirname(__file__), "golden", "cfg5_128x128x64_it100.npz")
    if not os.path.exists(path):
        pytest.skip("cfg5_128x128x64_it100.npz not generated")
    gd = np.load(path)
    w = synth.scaled(synth.WORKLOADS[5], (128, 128, 64), iters=100)
    assert tuple(gd["dims"]) == w.dims and tuple(gd["kernel"]) == w.kernel
    X, mask = w.target(), w.mask()
    B = gpu.EigenBasis(w.kernel, gd["K"], gd["eigenvalues"])
    Lo = gd["L"].astype(np.float64)
    miss = mask == 0
    cfg = gpu.SolverConfig(max_iters=100, engine=engine, **FIXED)

    def check(L, rep, tag):
        assert rep.iterations == 100, tag
        assert _rel(L, Lo) <= 1e-4, tag
        assert _rel(L[miss], Lo[miss]) <= 1e-3, tag
        assert abs(synth.psnr(X, L) - float(gd["psnr"])) <= 0.01, tag
        np.testing.assert_allclose(rep.objective, gd["objective"], rtol=1e-4)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    check(L1, r1, "unsharded")
    for G in (1, 2, 4, 8):
        row0, rows, rep = gpu.sharded_solve(X * mask, mask, B, cfg, local_slabs=G)
        assert row0 == 0 and rows.shape == X.shape
        check(rows, rep, f"G={G}")
    rows, rep = gpu.sharded_solve_local(X.shape, X * mask, mask, B, cfg, local_slabs=2,
                                        nccl_id=gpu.dist_unique_id())
    check(rows, rep, "G=2 NCCL one-rank, slab-local inputs")


def test_sharded_local_inputs_errors(gpu):
    """Slab-local inputs must be exactly the rank's rows; an invalid entry on
    any slab fails the call."""
    from paper_2604_17001_b200 import synth
    X = synth.synth_video(32, 16, 16, 4, 1, 5)
    mask = synth.synth_mask(32, 16, 16, synth.MASK_IID, 0.4, 6)
    B = gpu.learn_ensemble_basis([X], (5, 3, 3))
    cfg = gpu.SolverConfig(max_iters=5, **FIXED)
    assert gpu.sharded_rows(X.shape, (5, 3, 3), local_slabs=4) == (0, 32)
    with pytest.raises(gpu.InvalidArgument, match="owns rows"):
        gpu.sharded_solve_local(X.shape, (X * mask)[:16], mask[:16], B, cfg, local_slabs=4)
    bad = X * mask
    bad[20, 3, 3] = np.nan
    with pytest.raises(gpu.InvalidArgument, match="non-finite"):
        gpu.sharded_solve_local(X.shape, bad, mask, B, cfg, local_slabs=2,
                                nccl_id=gpu.dist_unique_id())
    L, _ = gpu.sharded_solve_local(X.shape, X * mask, mask, B, cfg, local_slabs=2)
    Lf, _ = gpu.icnnm_solve(X * mask, mask, B, cfg)
    assert _rel(L, Lf) <= 1e-5


@pytest.mark.parametrize("engine", ENGINES)
def test_exact_residual_trace(gpu, engine):
    """exact_residual=True reproduces the reference's primal_residual trace
    (solver.cpp:123-124) while it is above the fp32 resolution floor."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    Lg, rg = gpu.icnnm_solve(X * mask, mask, B,
                             gpu.SolverConfig(max_iters=120, engine=engine, exact_residual=True,
                                              **FIXED))
    Lo, ro = O.icnnm_solve(X * mask, mask, _oracle_basis(B),
                           O.SolverConfig(max_iters=120, **FIXED))
    assert _rel(Lg, Lo) <= 1e-4
    rgv, rov = np.array(rg.primal_residual), np.array(ro.primal_residual)
    assert not np.any(np.isnan(rgv))
    sel = rov > 1e-4
    assert sel.sum() > 10
    np.testing.assert_allclose(rgv[sel], rov[sel], rtol=2e-2)
    assert np.all(rgv[~sel] < 2e-4)


def test_exact_residual_stops_like_reference(gpu):
    """The exact residual drives the primal stopping test (solver.cpp:136-139)
    like the reference's on the cosine recovery case (tol_change disabled on
    both sides: fp32 cannot resolve l_change below ~1e-7)."""
    L0 = np.cos(2 * np.pi * np.arange(32) / 8)
    B = gpu.learn_ensemble_basis([L0], (8,))
    mask = gpu.synth.reference_bernoulli_mask((32,), 0.75, 5)
    cfg = gpu.SolverConfig(exact_residual=True, tol_primal=1e-5, tol_change=1e-300)
    L, rep = gpu.icnnm_solve(L0 * mask, mask, B, cfg)
    Lo, ro = O.icnnm_solve(L0 * mask, mask, _oracle_basis(B),
                           O.SolverConfig(tol_primal=1e-5, tol_change=1e-300))
    assert rep.termination == "converged" and ro.termination == "converged"
    assert abs(rep.iterations - ro.iterations) <= 3
    assert _rel(L, L0) < 1e-3


def test_default_config_converges_like_reference(gpu):
    """A drop-in caller's default SolverConfig (tol_primal 1e-7, tol_change
    1e-8, solver.hpp:35-37) stops where the reference does (solver.cpp:136-139):
    engine "auto" runs the fp64 engine for tolerances below the fp32 engines'
    resolution.  The reference's cosine case (test_solver.cpp:122-138) stops on
    l_change = 7.7e-9 at iteration 28."""
    L0 = np.cos(2 * np.pi * np.arange(32) / 8)
    B = gpu.learn_ensemble_basis([L0], (8,))
    mask = gpu.synth.reference_bernoulli_mask((32,), 0.75, 5)
    L, rep = gpu.icnnm_solve(L0 * mask, mask, B, gpu.SolverConfig())
    Lo, ro = O.icnnm_solve(L0 * mask, mask, _oracle_basis(B), O.SolverConfig())
    assert rep.termination == "converged" and ro.termination == "converged"
    assert abs(rep.iterations - ro.iterations) <= 1
    n = min(rep.iterations, ro.iterations)
    np.testing.assert_allclose(rep.objective[:n], ro.objective[:n], rtol=1e-9)
    np.testing.assert_allclose(rep.l_change[:n - 1], ro.l_change[:n - 1], rtol=1e-4, atol=1e-12)
    assert _rel(L, Lo) < 1e-8
    assert _rel(L, L0) < 1e-3


def test_f64_engine_matches_oracle_config1(gpu):
    """BASELINE config 1 with the reference's default tolerances: the oracle
    stops on the primal residual (< 1e-7) at iteration 88; the fp64 engine
    reproduces the stop and the traces."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    L, rep = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=400))
    Lo, ro = O.icnnm_solve(X * mask, mask, _oracle_basis(B), O.SolverConfig(max_iters=400))
    assert ro.termination == "converged" and rep.termination == "converged"
    assert abs(rep.iterations - ro.iterations) <= 1
    n = min(rep.iterations, ro.iterations)
    np.testing.assert_allclose(rep.objective[:n], ro.objective[:n], rtol=1e-8)
    np.testing.assert_allclose(rep.primal_residual[:n - 1], ro.primal_residual[:n - 1], rtol=1e-3)
    assert _rel(L, Lo) < 1e-7
    # the same call with an explicit fp32 engine cannot resolve these tolerances
    _, r32 = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=120, engine="f16x3"))
    assert r32.termination == "max_iters"


def test_auto_engine_fp32_when_resolvable(gpu):
    """Engine "auto" keeps the tcgen05 engine when the tolerances are disabled
    or resolvable in fp32 (tol_primal >= 1e-4 with the exact residual)."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    La, ra = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=30, **FIXED))
    Lf, rf = gpu.icnnm_solve(X * mask, mask, B,
                             gpu.SolverConfig(max_iters=30, engine="f16x3", **FIXED))
    np.testing.assert_array_equal(La, Lf)           # same engine, deterministic
    cfg = dict(max_iters=200, tol_primal=1e-3, tol_change=1e-300)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(**cfg))
    Lo, ro = O.icnnm_solve(X * mask, mask, _oracle_basis(B), O.SolverConfig(**cfg))
    assert r1.termination == "converged" and ro.termination == "converged"
    assert abs(r1.iterations - ro.iterations) <= 3
    assert not np.any(np.isnan(r1.primal_residual))


def test_cli_learn_complete_end_to_end(gpu, tmp_path):
    """GPU drop-in of the reference CLI's learn + complete
    (tools/icnnm_cli.cpp:151-166) on the reference's file formats."""
    import json
    import subprocess
    from paper_2604_17001_b200 import io as pio, synth
    from paper_2604_17001_b200._lib import CLI_PATH
    w = synth.WORKLOADS[1]
    X, mask = w.target(), w.mask()
    refs = w.training()
    paths = []
    for i, r in enumerate(refs):
        p = str(tmp_path / f"ref{i}.tnsr")
        pio.write_tnsr(p, r)
        paths.append(p)
    ebas = str(tmp_path / "basis.ebas")
    out = subprocess.run([CLI_PATH, "learn", "--refs", *paths, "--kernel", "5,5,3", "--out", ebas],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    B = pio.read_ebas(ebas)
    Bp = gpu.learn_ensemble_basis(refs, w.kernel)
    np.testing.assert_array_equal(B.K, Bp.K)          # deterministic Gram reduction
    np.testing.assert_array_equal(B.eigenvalues, Bp.eigenvalues)
    pio.write_tnsr(str(tmp_path / "M.tnsr"), X * mask)
    pio.write_tnsr(str(tmp_path / "mask.tnsr"), mask)
    (tmp_path / "cfg.json").write_text(json.dumps({"max_iters": 50, "tol_primal": 1e-300,
                                                   "tol_change": 1e-300}))
    out = subprocess.run([CLI_PATH, "complete", "--input", str(tmp_path / "M.tnsr"), "--mask",
                          str(tmp_path / "mask.tnsr"), "--basis", ebas, "--config",
                          str(tmp_path / "cfg.json"), "--out", str(tmp_path / "L.tnsr"),
                          "--report", str(tmp_path / "rep.json")], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    L = pio.read_tnsr(str(tmp_path / "L.tnsr"))
    rep = json.loads((tmp_path / "rep.json").read_text())
    Lp, rp = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=50, **FIXED))
    assert _rel(L, Lp) < 1e-6
    assert rep["iterations"] == 50 and rep["termination"] == "max_iters"
    np.testing.assert_allclose(rep["objective"], rp.objective, rtol=1e-6)


# --------------------------------------------------------------------------
# Full-size BASELINE configs against committed fp64-oracle goldens
# (tests/golden/*.npz, oracle/gen_golden.py; the basis K is stored with the
# golden so both sides use identical bits): config 2 (300 iterations) and
# config 4's first batch tensor (200 iterations)
# --------------------------------------------------------------------------
GOLDENS = [("cfg2_it300.npz", 2, 0), ("cfg4_it200.npz", 4, 0)]


@pytest.mark.parametrize("fname,cfgno,bidx", GOLDENS)
@pytest.mark.parametrize("engine", ENGINES)
def test_full_size_golden(gpu, engine, fname, cfgno, bidx):
    import os
    from paper_2604_17001_b200 import synth
    path = os.path.join(os.path.dirname(__file__), "golden", fname)
    if not os.path.exists(path):
        pytest.skip(f"{fname} not generated")
    gd = np.load(path)
    w = synth.WORKLOADS[cfgno]
    assert tuple(gd["dims"]) == w.dims and tuple(gd["kernel"]) == w.kernel
    assert int(gd["batch_index"]) == bidx
    X, mask = w.target(b=bidx), w.mask()
    B = gpu.EigenBasis(tuple(int(x) for x in gd["kernel"]), gd["K"], gd["eigenvalues"])
    iters = int(gd["iters"])
    L, rep = gpu.icnnm_solve(X * mask, mask, B,
                             gpu.SolverConfig(max_iters=iters, engine=engine, **FIXED))
    Lo = gd["L"].astype(np.float64)
    assert rep.iterations == iters == w.iters
    assert _rel(L, Lo) <= 1e-4
    miss = mask == 0
    assert _rel(L[miss], Lo[miss]) <= 1e-3
    assert abs(synth.psnr(X, L) - float(gd["psnr"])) <= 0.01
    np.testing.assert_allclose(rep.objective, gd["objective"], rtol=1e-4)


@pytest.mark.parametrize("engine", ENGINES)
def test_config2_recovering_golden(gpu, engine):
    """A full-size problem on which the iteration does real work (the
    BASELINE config-2/4 goldens sit in a nearly stalled regime, recovered
    PSNR within 0.06 dB of zero fill): config 2's dims and kernel on a video
    of low convolution rank (4 sinusoids, no blobs, no noise), 50% i.i.d.
    sampling, init_fill = "mean" (solver.cpp:83-86), 300 iterations.  The
    fp64 oracle recovers 18.26 dB from a zero fill of 8.50 dB
    (oracle/gen_golden.py --config 2 --recover), so rel-L2 and PSNR
    discriminate here."""
    import dataclasses
    import os
    from paper_2604_17001_b200 import synth
    path = os.path.join(os.path.dirname(__file__), "golden", "cfg2_recover_it300.npz")
    if not os.path.exists(path):
        pytest.skip("cfg2_recover_it300.npz not generated")
    gd = np.load(path)
    w = dataclasses.replace(synth.WORKLOADS[2], n_sin=4, n_blob=0, noise=0.0, mask_kind=0,
                            mask_rate=0.5)
    assert tuple(gd["dims"]) == w.dims and tuple(gd["kernel"]) == w.kernel
    assert int(gd["recover"]) == 1 and str(gd["init_fill"]) == "mean"
    X, mask = w.target(), w.mask()
    B = gpu.EigenBasis(w.kernel, gd["K"], gd["eigenvalues"])
    iters = int(gd["iters"])
    L, rep = gpu.icnnm_solve(X * mask, mask, B,
                             gpu.SolverConfig(max_iters=iters, engine=engine, init_fill="mean",
                                              **FIXED))
    Lo = gd["L"].astype(np.float64)
    assert rep.iterations == iters == 300
    assert float(gd["psnr"]) - float(gd["psnr_zero_fill"]) > 9.0      # real recovery
    assert _rel(L, Lo) <= 1e-4
    miss = mask == 0
    assert _rel(L[miss], Lo[miss]) <= 1e-3
    assert abs(synth.psnr(X, L) - float(gd["psnr"])) <= 0.01
    np.testing.assert_allclose(rep.objective, gd["objective"], rtol=1e-4)


@pytest.mark.parametrize("engine", ["f16x3", "tf32x3"])
def test_config3_full_size_golden(gpu, engine):
    """BASELINE config 3 at full size (256x256x48, kernel 13x13x7, k = 1183;
    frames 40-47 missing) against the literal fp64 oracle for 10 iterations
    (out-of-core blocked loop, oracle/icnnm_oracle_blocked.py: Y and Z are
    29.8 GB each): overall rel-L2, the predicted frames 40-47, PSNR and the
    objective trace (solver.cpp:107-139 at the largest contraction)."""
    import os
    from paper_2604_17001_b200 import synth
    path = os.path.join(os.path.dirname(__file__), "golden", "cfg3_it10.npz")
    if not os.path.exists(path):
        pytest.skip("cfg3_it10.npz not generated")
    gd = np.load(path)
    w = synth.WORKLOADS[3]
    assert tuple(gd["dims"]) == w.dims and tuple(gd["kernel"]) == w.kernel
    X, mask = w.target(), w.mask()
    assert mask[:, :, 40:].sum() == 0 and mask[:, :, :40].min() == 1
    B = gpu.EigenBasis(w.kernel, gd["K"], gd["eigenvalues"])
    iters = int(gd["iters"])
    L, rep = gpu.icnnm_solve(X * mask, mask, B,
                             gpu.SolverConfig(max_iters=iters, engine=engine, **FIXED))
    Lo = gd["L"].astype(np.float64)
    assert rep.iterations == iters == 10
    assert _rel(L, Lo) <= 1e-4
    assert _rel(L[:, :, 40:], Lo[:, :, 40:]) <= 1e-3      # the predicted frames
    assert abs(synth.psnr(X, L) - float(gd["psnr"])) <= 0.01
    np.testing.assert_allclose(rep.objective, gd["objective"], rtol=1e-4)


CFG4_GOLDEN_BATCH = (0, 21, 42, 63)


@pytest.mark.parametrize("engine", ["f16x3", "tf32x3"])
def test_config4_batch_goldens(gpu, engine):
    """BASELINE config 4 through the library batch call: tensors {0, 21, 42,
    63} of the 64-tensor batch (each with its own theta0 = 1e-2 max|pm| k,
    solver.cpp:88-91) against their fp64-oracle goldens, split over two
    workers on one device (the per-device blocks of icnnm_cuda_solve_batch)."""
    import os
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[4]
    gds = []
    for b in CFG4_GOLDEN_BATCH:
        path = os.path.join(os.path.dirname(__file__), "golden",
                            "cfg4_it200.npz" if b == 0 else f"cfg4_b{b}_it200.npz")
        if not os.path.exists(path):
            pytest.skip(f"{path} not generated")
        gds.append(np.load(path))
    mask = w.mask()
    Xs = [w.target(b=b) for b in CFG4_GOLDEN_BATCH]
    gd0 = gds[0]
    B = gpu.EigenBasis(tuple(int(x) for x in gd0["kernel"]), gd0["K"], gd0["eigenvalues"])
    for gd in gds[1:]:
        np.testing.assert_array_equal(gd["K"], gd0["K"])
    cfg = gpu.SolverConfig(max_iters=w.iters, engine=engine, **FIXED)
    Ls, reps = gpu.icnnm_solve_batch([X * mask for X in Xs], mask, B, cfg, devices=[0, 0])
    miss = mask == 0
    psnrs = set()
    for b, X, L, rep, gd in zip(CFG4_GOLDEN_BATCH, Xs, Ls, reps, gds):
        Lo = gd["L"].astype(np.float64)
        assert int(gd["batch_index"]) == b
        assert rep.iterations == w.iters
        assert _rel(L, Lo) <= 1e-4, b
        assert _rel(L[miss], Lo[miss]) <= 1e-3, b
        assert abs(synth.psnr(X, L) - float(gd["psnr"])) <= 0.01, b
        np.testing.assert_allclose(rep.objective, gd["objective"], rtol=1e-4)
        psnrs.add(round(float(gd["psnr"]), 3))
    assert len(psnrs) == len(CFG4_GOLDEN_BATCH)  # four distinct problems


def test_solve_batch_equals_single_calls(gpu):
    """icnnm_cuda_solve_batch == one icnnm_cuda_solve per tensor (own theta0,
    own report), for 1, 2 and 3 worker blocks; errors name the problem."""
    from paper_2604_17001_b200 import synth
    w = synth.scaled(synth.WORKLOADS[4], (24, 20, 16), iters=40, n_train=2)
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    mask = w.mask()
    Ms = [w.target(b=b) * mask * (1.0 + 0.5 * b) for b in range(5)]
    cfg = gpu.SolverConfig(max_iters=w.iters, **FIXED)
    single = [gpu.icnnm_solve(M, mask, B, cfg) for M in Ms]
    for devs in ([0], [0, 0], [0, 0, 0]):
        Ls, reps = gpu.icnnm_solve_batch(Ms, mask, B, cfg, devices=devs)
        assert len(Ls) == len(reps) == 5
        for (L1, r1), L, r in zip(single, Ls, reps):
            assert r.iterations == r1.iterations == w.iters
            assert _rel(L, L1) <= 1e-6
            np.testing.assert_allclose(r.objective, r1.objective, rtol=1e-6)
    assert gpu.icnnm_solve_batch([], mask, B, cfg) == ([], [])
    bad = [m.copy() for m in Ms]
    bad[3].flat[7] = np.nan
    with pytest.raises(gpu.InvalidArgument, match="problem 3"):
        gpu.icnnm_solve_batch(bad, mask, B, cfg, devices=[0, 0])
    with pytest.raises(gpu.InvalidArgument, match="out of range"):
        gpu.icnnm_solve_batch(Ms, mask, B, cfg, devices=[0, 99])
    with pytest.raises(gpu.InvalidArgument, match="not orthogonal"):
        gpu.icnnm_solve_batch(Ms, mask, gpu.EigenBasis(B.kernel_shape, 2 * B.K, B.eigenvalues),
                              cfg)


@pytest.mark.parametrize("engine", ["f16x3", "tf32x3"])
@pytest.mark.parametrize("cfgno,dims,iters", [(4, (32, 32, 16), 40), (2, (24, 24, 16), 30),
                                              (1, (32, 32, 8), 30)])
def test_solve_bit_reproducible(gpu, engine, cfgno, dims, iters):
    """Two solves of the same problem are bit-identical (the reference is
    deterministic): the tcgen05 engines reduce the adjoint's
    output bricks, the column norms and the report sums in a fixed order
    (no floating-point atomics).  Covers the resident-B split mode (config-4
    and config-1 recipes) and the streamed-B mode (config-2 recipe)."""
    from paper_2604_17001_b200 import synth
    w = synth.scaled(synth.WORKLOADS[cfgno], dims, iters=iters, n_train=2)
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    cfg = gpu.SolverConfig(max_iters=iters, engine=engine, **FIXED)
    L1, r1 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    L2, r2 = gpu.icnnm_solve(X * mask, mask, B, cfg)
    np.testing.assert_array_equal(L1, L2)
    np.testing.assert_array_equal(np.asarray(r1.objective), np.asarray(r2.objective))
    cfg_x = gpu.SolverConfig(max_iters=iters, engine=engine, exact_residual=True, **FIXED)
    L3, r3 = gpu.icnnm_solve(X * mask, mask, B, cfg_x)
    L4, r4 = gpu.icnnm_solve(X * mask, mask, B, cfg_x)
    np.testing.assert_array_equal(L3, L4)
    np.testing.assert_array_equal(np.asarray(r3.primal_residual), np.asarray(r4.primal_residual))
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B),
                          O.SolverConfig(max_iters=iters, **FIXED))
    assert _rel(L1, Lo) <= 1e-4


def test_rejected_upload_leaves_no_problem(gpu):
    """A rejected upload must not leave the previous problem's scalars next to
    the overwritten staging buffers: the handle then has no problem."""
    from paper_2604_17001_b200 import synth
    w = synth.scaled(synth.WORKLOADS[1], (16, 16, 8), iters=10, n_train=1)
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    X, mask = w.target(), w.mask()
    S = gpu.Solver(w.dims, B)
    try:
        S.upload(X * mask, mask)
        S.run(gpu.SolverConfig(max_iters=5, **FIXED))
        bad = X * mask
        bad[0, 0, 0] = np.inf
        with pytest.raises(gpu.InvalidArgument, match="non-finite"):
            S.upload(bad, mask)
        with pytest.raises(gpu.InvalidArgument, match="no problem uploaded"):
            S.run(gpu.SolverConfig(max_iters=5, **FIXED))
        S.upload(X * mask, mask)
        S.run(gpu.SolverConfig(max_iters=5, **FIXED))
        with pytest.raises(gpu.InvalidArgument):
            S.download(out=np.empty((16, 16, 8), dtype=np.float32))
        with pytest.raises(gpu.InvalidArgument):
            S.download(out=np.empty((16, 16, 7)))
        with pytest.raises(gpu.InvalidArgument):
            S.download(out=np.empty((16, 16, 16))[:, :, ::2])
        out = np.empty((16, 16, 8))
        assert S.download(out=out) is out
    finally:
        S.close()


def test_config3_full_size_engines_agree(gpu):
    """BASELINE config 3 at full size (256x256x48, k = 1183: six N-tiles, three
    tile groups).  The fp64 oracle cannot hold its m x k state in host RAM, so
    full-size parity is the F16x3 tensor-core engine against the exact-fp32
    FFMA engine (itself oracle-checked on the scaled recipe,
    test_recipe_parity) over the first 10 iterations."""
    from paper_2604_17001_b200 import synth
    w = synth.WORKLOADS[3]
    X, mask = w.target(), w.mask()
    B = gpu.learn_ensemble_basis(w.training(), w.kernel)
    out = {}
    for engine in ("f16x3", "ffma"):
        out[engine], rep = gpu.icnnm_solve(
            X * mask, mask, B, gpu.SolverConfig(max_iters=10, engine=engine, **FIXED))
        assert rep.iterations == 10
    assert _rel(out["f16x3"], out["ffma"]) <= 1e-5
    miss = mask == 0
    assert _rel(out["f16x3"][miss], out["ffma"][miss]) <= 1e-4


# --------------------------------------------------------------------------
# tcgen05 engine edge cases: N-tile boundaries (k around 128/256, partial last
# tile), partial bricks, T < 8, order 1/2, kernel box = whole tensor
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dims,ks", [((12, 11, 10), (4, 4, 8)),     # k=128: exactly one tile
                                     ((12, 11, 10), (1, 11, 9)),    # k=99
                                     ((14, 9, 17), (3, 3, 15)),     # k=135: 128 + 7
                                     ((10, 9, 20), (2, 8, 16)),     # k=256: two full tiles
                                     ((9, 9, 7), (9, 9, 4)),        # kernel spans H and W
                                     ((5, 3, 3), (5, 3, 3)),        # kernel = whole tensor
                                     ((40, 3), (7, 3)),             # order 2, T < 8
                                     ((50,), (33,))])               # order 1, k=33
@pytest.mark.parametrize("engine", ENGINES)
def test_operator_edge_cases(gpu, dims, ks, engine):
    rng = np.random.default_rng(7)
    k = int(np.prod(ks))
    Li = rng.integers(-8, 9, size=dims).astype(np.float64)
    np.testing.assert_array_equal(gpu.BasisConvolver(dims, ks, np.eye(k), engine=engine).apply(Li),
                                  O.conv_matrix(Li, ks))
    W = rng.integers(-4, 5, size=(Li.size, k)).astype(np.float64)
    np.testing.assert_array_equal(gpu.conv_adjoint(W, ks, dims, engine=engine),
                                  O.conv_adjoint(W, ks, dims))
    L = rng.uniform(-1, 1, size=dims)
    K = _rand_orth(k, 11)
    got = gpu.BasisConvolver(dims, ks, K, engine=engine).apply(L)
    assert _rel(got, O.BasisConvolver(dims, ks, K).apply(L)) < 1e-5


@pytest.mark.parametrize("dims,ks,iters", [((14, 9, 17), (3, 3, 15), 40), ((10, 9, 20), (2, 8, 16), 30),
                                           ((40, 3), (7, 3), 60), ((50,), (33,), 80)])
@pytest.mark.parametrize("engine", ENGINES)
def test_solve_edge_cases(gpu, dims, ks, iters, engine):
    rng = np.random.default_rng(3)
    base = np.cos(np.linspace(0, 6, int(np.prod(dims)))).reshape(dims)
    X = base + 0.05 * rng.standard_normal(dims)
    mask = gpu.synth.reference_bernoulli_mask(dims, 0.6, 4)
    B = gpu.learn_ensemble_basis([base + 0.05 * rng.standard_normal(dims)], ks)
    Lg, _ = gpu.icnnm_solve(X * mask, mask, B, gpu.SolverConfig(max_iters=iters, engine=engine, **FIXED))
    Lo, _ = O.icnnm_solve(X * mask, mask, _oracle_basis(B), O.SolverConfig(max_iters=iters, **FIXED))
    assert _rel(Lg, Lo) <= 1e-4


# --------------------------------------------------------------------------
# opt-in 2-CTA cluster modes of the F16x3 engine (read from the environment
# once per process, so each runs in a subprocess): CTA pairs (cta_group::2,
# ICNNM_TC_CS=2) and B multicast (ICNNM_TC_MCB=1)
# --------------------------------------------------------------------------
_CLUSTER_CHECK = r"""
import sys, os, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2604_17001_b200._lib as _L
# the A/B knobs are read only by the experiments build (make EXPERIMENTS=1)
_L.LIB_PATH = os.path.join(sys.argv[1], "build", "ab", "libicnnm_b200_ab.so")
import paper_2604_17001_b200 as P
from oracle import icnnm_oracle as O
out = []
for dims, ks in [((16, 16, 32), (9, 9, 5)), ((7, 5, 9), (3, 2, 4)), ((12, 11, 10), (4, 4, 8))]:
    k = int(np.prod(ks))
    L = np.random.default_rng(1).integers(-8, 9, size=dims).astype(np.float64)
    f = P.BasisConvolver(dims, ks, np.eye(k), engine="f16x3").apply(L)
    assert np.array_equal(f, O.conv_matrix(L, ks)), ("fwd", dims)
    W = np.random.default_rng(4).integers(-4, 5, size=(L.size, k)).astype(np.float64)
    a = P.conv_adjoint(W, ks, dims, engine="f16x3")
    assert np.array_equal(a, O.conv_adjoint(W, ks, dims)), ("adj", dims)
from paper_2604_17001_b200 import synth
w = synth.scaled(synth.WORKLOADS[2], (16, 16, 32), iters=30)
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
cfg = P.SolverConfig(max_iters=30, tol_primal=1e-300, tol_change=1e-300)
Lg, _ = P.icnnm_solve(X * mask, mask, B, cfg)
Lo, _ = O.icnnm_solve(X * mask, mask, O.EigenBasis(B.kernel_shape, B.K, B.eigenvalues),
                      O.SolverConfig(max_iters=30, tol_primal=1e-300, tol_change=1e-300))
rel = float(np.linalg.norm(Lg - Lo) / np.linalg.norm(Lo))
assert rel <= 1e-4, rel
print("ok", rel)
"""


@pytest.mark.parametrize("env", [{"ICNNM_TC_CS": "2"}, {"ICNNM_TC_MCB": "1"}])
def test_cluster_modes_exact_and_solve_parity(gpu, env):
    _ab_lib()
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CLUSTER_CHECK, root], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# --------------------------------------------------------------------------
# The NCCL transport of the sharded solve on one GPU: world == 1 with a NCCL
# id routes the halo shifts through self send/recv and the norm vector through
# ncclAllReduce (captured in the solve graph), the same calls a multi-process
# run makes.  In a subprocess with a timeout so a transport hang cannot stall
# the suite.
# --------------------------------------------------------------------------
_NCCL_ONE_RANK = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2604_17001_b200 as P
from oracle import icnnm_oracle as O
from paper_2604_17001_b200 import synth
engine = sys.argv[2]
X = synth.synth_video(48, 16, 16, 8, 2, 21)
mask = synth.synth_mask(48, 16, 16, synth.MASK_IID, 0.3, 22)
mask[20:30, 3:9, 4:12] = 0.0
B = P.learn_ensemble_basis([synth.synth_video(48, 16, 16, 8, 2, 23)], (5, 3, 3))
F = dict(tol_primal=1e-300, tol_change=1e-300)
cfg = P.SolverConfig(max_iters=40, engine=engine, **F)
L1, r1 = P.icnnm_solve(X * mask, mask, B, cfg)
Lo, _ = O.icnnm_solve(X * mask, mask, O.EigenBasis(B.kernel_shape, B.K, B.eigenvalues),
                      O.SolverConfig(max_iters=40, **F))
for G in (1, 3):
    row0, rows, rep = P.sharded_solve(X * mask, mask, B, cfg, local_slabs=G, world=1, rank=0,
                                      nccl_id=P.dist_unique_id())
    assert row0 == 0 and rows.shape == X.shape
    rel = float(np.linalg.norm(rows - L1) / np.linalg.norm(L1))
    relo = float(np.linalg.norm(rows - Lo) / np.linalg.norm(Lo))
    assert rel <= 1e-5 and relo <= 1e-4, (G, rel, relo)
    np.testing.assert_allclose(rep.objective, r1.objective, rtol=1e-5)
print("ok")
"""


@pytest.mark.parametrize("engine", ["f16x3", "ffma"])
def test_sharded_nccl_one_rank_transport(gpu, engine):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _NCCL_ONE_RANK, root, engine],
                       env={**os.environ, "NCCL_DEBUG": "WARN"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# --------------------------------------------------------------------------
# Launch-structure options must not change results: PDL edges (ICNNM_PDL) and
# the head/body graph split (ICNNM_GRAPH_SPLIT), both read once per process.
# 64x64x32 with kernel 9x9x5 and 100 iterations is long enough to split.
# --------------------------------------------------------------------------
_LAUNCH_MODES = r"""
import sys, os, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2604_17001_b200._lib as _L
# the A/B knobs are read only by the experiments build (make EXPERIMENTS=1)
_L.LIB_PATH = os.path.join(sys.argv[1], "build", "ab", "libicnnm_b200_ab.so")
import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import synth
w = synth.scaled(synth.WORKLOADS[2], (64, 64, 32), iters=100, n_train=2)
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
for eng in ("f16x3", "ffma"):
    L, r = P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=100, engine=eng,
                                                           tol_primal=1e-300, tol_change=1e-300))
    assert r.iterations == 100
    np.save(sys.argv[2] + "_" + eng + ".npy", L)
    np.save(sys.argv[2] + "_" + eng + "_obj.npy", np.asarray(r.objective))
print("ok")
"""


def test_launch_modes_do_not_change_results(gpu, tmp_path):
    _ab_lib()
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env in [("base", {}), ("nopdl", {"ICNNM_PDL": "0"}),
                     ("nosplit", {"ICNNM_GRAPH_SPLIT": "0"})]:
        r = subprocess.run([sys.executable, "-c", _LAUNCH_MODES, root, str(tmp_path / tag)],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    for eng in ("f16x3", "ffma"):
        ref = np.load(tmp_path / f"base_{eng}.npy")
        obj = np.load(tmp_path / f"base_{eng}_obj.npy")
        for tag in ("nopdl", "nosplit"):
            assert _rel(np.load(tmp_path / f"{tag}_{eng}.npy"), ref) < 1e-6, (tag, eng)
            np.testing.assert_allclose(np.load(tmp_path / f"{tag}_{eng}_obj.npy"), obj, rtol=1e-6)
