"""CPU tests of the C-ABI library: loads, exports every declared symbol, and
its host-only logic (config validation, shard plan, generators, RNG streams,
eigensolver) behaves.  No GPU compute is called here."""
import os
import re

import numpy as np
import pytest

import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import _lib, synth


def _declared_functions():
    src = open(_lib.HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(icnnm_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = P.lib()
    names = _declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} not bound in _lib.SIGNATURES"
    assert lib.icnnm_version().decode().startswith("icnnm_b200")


def test_generator_library_is_separate():
    """The input generator (include/icnnm_synth.h) lives in synthgen's own
    host-only library: the product library does not carry it, so the oracle
    and bench.py's reference arm never load libicnnm_b200.so."""
    import synthgen
    hdr = os.path.join(os.path.dirname(_lib.HEADER_PATH), "icnnm_synth.h")
    src = re.sub(r"/\*.*?\*/", "", open(hdr).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(icnnm_[a-z0-9_]+)\s*\(", src)))
    assert len(names) == 8
    g = synthgen.lib()
    for n in names:
        assert hasattr(g, n), n
        assert not hasattr(P.lib(), n), f"{n} still exported by the product library"


def test_reference_arm_imports_do_not_map_the_product_library():
    """bench.py --impl reference generates its inputs through synthgen and
    computes with the oracle: neither may map libicnnm_b200.so."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import synthgen, bench; "
            "from oracle import icnnm_oracle; w = synthgen.WORKLOADS[1]; w.target(); w.mask(); "
            "m = open('/proc/self/maps').read(); "
            "assert 'libicnnm_b200' not in m, 'product library mapped'; "
            "assert 'libicnnm_synth' in m" % os.path.dirname(os.path.dirname(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, timeout=300)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_default_config_matches_reference():
    """SolverConfig defaults (solver.hpp:29-43)."""
    import ctypes as C
    c = _lib.SolverConfigC()
    P.lib().icnnm_default_config(C.byref(c))
    assert c.lambda_ == 1000.0 and c.has_theta0 == 0 and c.theta_growth == 1.05
    assert c.theta_max == 1e10 and c.max_iters == 1000 and c.tol_primal == 1e-7
    assert c.tol_change == 1e-8 and c.rank_tol == 1e-8 and c.init_fill == 0
    py = P.SolverConfig()
    assert (py.lambda_, py.theta_growth, py.theta_max, py.max_iters, py.tol_primal,
            py.tol_change, py.init_fill) == (1000.0, 1.05, 1e10, 1000, 1e-7, 1e-8, "zero")


@pytest.mark.parametrize("kw", [dict(lambda_=-1), dict(lambda_=0), dict(theta_growth=0.5),
                                dict(theta0=1e20), dict(theta0=-1.0), dict(theta_max=0),
                                dict(max_iters=0), dict(tol_primal=0), dict(tol_change=-1),
                                dict(rank_tol=0), dict(init_fill="bogus"),
                                dict(engine="nope")])
def test_config_validation_errors(kw):
    """SolverConfig::validate (solver.cpp:26-40) -> std::invalid_argument."""
    with pytest.raises(P.InvalidArgument):
        P.SolverConfig(**kw).validate()


def test_config_validation_ok():
    P.SolverConfig().validate()
    P.SolverConfig(theta0=5.0, init_fill="mean", engine="tf32x3").validate()


def test_product_path_fails_loudly_without_gpu():
    if P.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(P.IcnnmError):
        P.icnnm_solve(np.ones((4, 4)), np.ones((4, 4)),
                      P.EigenBasis((2, 2), np.eye(4), np.ones(4)))


@pytest.mark.parametrize("H,G,kh", [(1024, 8, 9), (1024, 2, 9), (100, 7, 5), (48, 4, 5),
                                    (13, 13, 1), (9, 3, 4)])
def test_shard_plan_partitions_rows(H, G, kh):
    rows = []
    for g in range(G):
        s, c = P.shard_plan(H, G, kh, g)
        rows.append((s, c))
        assert c >= kh - 1 and c >= 1
    assert rows[0][0] == 0
    for (s0, c0), (s1, _) in zip(rows, rows[1:]):
        assert s1 == s0 + c0
    assert rows[-1][0] + rows[-1][1] == H
    assert max(c for _, c in rows) - min(c for _, c in rows) <= 1


@pytest.mark.parametrize("H,G,world", [(1024, 8, 8), (1024, 2, 4), (100, 3, 2), (48, 1, 4)])
def test_sharded_rows_partition_H(H, G, world):
    """icnnm_sharded_rows: each rank's rows are its local_slabs consecutive
    slabs of the G*world-slab plan; the ranks tile [0, H) in order."""
    nxt = 0
    for r in range(world):
        r0, n = P.sharded_rows((H, 16, 8), (9, 3, 3), local_slabs=G, world=world, rank=r)
        assert r0 == nxt and n >= 1
        s0, _ = P.shard_plan(H, G * world, 9, r * G)
        assert s0 == r0
        nxt = r0 + n
    assert nxt == H


def test_shard_plan_rejects_thin_slabs():
    with pytest.raises(P.InvalidArgument):
        P.shard_plan(16, 8, 9, 0)      # 2 rows < 8-row halo
    with pytest.raises(P.InvalidArgument):
        P.shard_plan(16, 0, 3, 0)


def test_synth_deterministic_and_scaled():
    a = synth.synth_video(16, 12, 8, 8, 1, 5)
    b = synth.synth_video(16, 12, 8, 8, 1, 5)
    c = synth.synth_video(16, 12, 8, 8, 1, 6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() == 0.0 and a.max() == 1.0
    n = synth.synth_video(16, 12, 8, 8, 1, 5, noise_sigma=0.01)
    assert 0.005 < np.std(n - a) < 0.015


def test_baseline_masks():
    w1, w2, w3, w4 = (synth.WORKLOADS[i] for i in (1, 2, 3, 4))
    m1 = w1.mask()
    assert set(np.unique(m1)) <= {0.0, 1.0} and 0.45 < m1.mean() < 0.55
    m2 = w2.mask()
    assert m2.sum() == round(0.2 * m2.size)            # exact count (mask.cpp:51)
    m3 = synth.synth_mask(8, 8, 48, synth.MASK_T_PREFIX, 40, 0)
    assert np.all(m3[..., :40] == 1) and np.all(m3[..., 40:] == 0)
    m4 = synth.synth_mask(8, 8, 32, synth.MASK_T_FRAMES, 0, 0)
    assert np.all(m4[..., ::2] == 1) and np.all(m4[..., 1::2] == 0)
    m5 = synth.synth_mask(256, 256, 16, synth.MASK_IID_BOXES, 0.3, 9, n_boxes=20)
    assert m5.mean() < 0.3
    assert w3.dims == (256, 256, 48) and w4.batch == 64


# --- libstdc++ mt19937_64 reproduction (pins the reference-test inputs) -----
class _MT64:
    """Pure-python std::mt19937_64 (the published MT19937-64 recurrence)."""
    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for j in range(312):
                x = (self.mt[j] & 0xFFFFFFFF80000000) | (self.mt[(j + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[j] = self.mt[(j + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def test_mt19937_64_known_value():
    g = _MT64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042   # [rand.predef] requirement


def test_rng_uniform_matches_generate_canonical():
    """uniform_real_distribution<double>(a,b) = generate_canonical * (b-a) + a,
    one 64-bit draw per value (libstdc++)."""
    r = synth.Rng(7)
    got = r.uniform(-1.0, 1.0, 50)
    g = _MT64(7)
    exp = []
    for _ in range(50):
        u = g() / 18446744073709551616.0
        if u >= 1.0:
            u = np.nextafter(1.0, 0.0)
        exp.append(u * 2.0 - 1.0)
    np.testing.assert_array_equal(got, np.array(exp))


def test_reference_bernoulli_mask_exact_count():
    for m, rate, seed in [(32, 0.75, 5), (25, 0.6, 3), (1000, 0.2, 1)]:
        mk = synth.reference_bernoulli_mask((m,), rate, seed)
        assert mk.sum() == round(rate * m)
    assert np.array_equal(synth.reference_bernoulli_mask((32,), 0.75, 5),
                          synth.reference_bernoulli_mask((32,), 0.75, 5))


def test_host_symeig_matches_lapack():
    rng = np.random.default_rng(0)
    for n in (1, 2, 5, 40, 200):
        A = rng.standard_normal((n, n))
        G = A + A.T
        ev, V = P.symeig(G)
        assert np.all(np.diff(ev) <= 0)
        np.testing.assert_allclose(ev, np.linalg.eigvalsh(G)[::-1], atol=1e-10 * max(1, abs(ev).max()))
        assert np.max(np.abs(V.T @ V - np.eye(n))) < 1e-12
        assert np.max(np.abs(G @ V - V * ev)) < 1e-10 * max(1, abs(ev).max())


def test_host_symeig_degenerate_and_psd():
    G = np.diag([3.0, 3.0, 1.0, 0.0])
    ev, V = P.symeig(G)
    np.testing.assert_allclose(ev, [3, 3, 1, 0], atol=1e-14)
    A = np.random.default_rng(1).standard_normal((30, 5))
    ev, V = P.symeig(A @ A.T)       # rank 5 PSD
    assert np.all(ev[5:] < 1e-10 * ev[0])
