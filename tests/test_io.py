"""Reference file formats (tensor_io.cpp:86-128) and config/report JSON
(report_io.cpp:39-68) of the GPU CLI drop-in; CPU only."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import io as pio
from paper_2604_17001_b200._lib import CLI_PATH


def _ref_tnsr_bytes(t):
    """write_tnsr (tensor_io.cpp:86-93) restated with struct."""
    b = b"TNSR" + struct.pack("<I", t.ndim) + b"".join(struct.pack("<I", d) for d in t.shape)
    return b + np.ascontiguousarray(t, dtype="<f8").tobytes()


def test_tnsr_bytes_and_roundtrip(tmp_path):
    t = np.random.default_rng(0).standard_normal((3, 4, 5))
    p = str(tmp_path / "a.tnsr")
    pio.write_tnsr(p, t)
    assert open(p, "rb").read() == _ref_tnsr_bytes(t)
    np.testing.assert_array_equal(pio.read_tnsr(p), t)


def test_ebas_layout_is_column_major(tmp_path):
    k = 6
    K = np.linalg.qr(np.random.default_rng(1).standard_normal((k, k)))[0]
    ev = np.sort(np.random.default_rng(2).uniform(0, 1, k))[::-1].copy()
    b = P.EigenBasis((2, 3), K, ev)
    p = str(tmp_path / "b.ebas")
    pio.write_ebas(p, b)
    raw = open(p, "rb").read()
    hdr = b"EBAS" + struct.pack("<III", 2, 2, 3)
    assert raw[:16] == hdr
    vals = np.frombuffer(raw[16:], dtype="<f8")
    np.testing.assert_array_equal(vals[:k], ev)
    np.testing.assert_array_equal(vals[k:].reshape(k, k).T, K)     # Eigen column-major
    r = pio.read_ebas(p)
    assert r.kernel_shape == (2, 3)
    np.testing.assert_array_equal(r.K, K)


def test_bad_files(tmp_path):
    p = tmp_path / "x.tnsr"
    p.write_bytes(b"NOPE" + b"\0" * 12)
    with pytest.raises(P.IcnnmError, match="bad magic"):
        pio.read_tnsr(str(p))
    p.write_bytes(b"TNSR" + struct.pack("<I", 0))
    with pytest.raises(P.IcnnmError, match="implausible tensor order"):
        pio.read_tnsr(str(p))
    p.write_bytes(b"TNSR" + struct.pack("<II", 1, 4) + b"\0" * 8)
    with pytest.raises(P.IcnnmError, match="truncated payload"):
        pio.read_tnsr(str(p))
    with pytest.raises(P.IcnnmError, match="cannot open"):
        pio.read_tnsr(str(tmp_path / "missing.tnsr"))


def test_config_json():
    c = pio.config_from_json("{}")
    assert c.lambda_ == 1000.0 and c.has_theta0 == 0 and c.max_iters == 1000
    c = pio.config_from_json('{"lambda": 50, "theta0": 2.5, "max_iters": 7, '
                             '"init_fill": "mean", "tol_primal": 1e-3, "engine": "ffma"}')
    assert (c.lambda_, c.has_theta0, c.theta0, c.max_iters, c.init_fill, c.engine) == \
        (50.0, 1, 2.5, 7, 1, 0)
    c = pio.config_from_json('{"theta0": null}')
    assert c.has_theta0 == 0
    for bad in ['{"lambda": -1}', '{"init_fill": "bogus"}', '{"theta0": 1e20}', '[1]',
                '{"max_iters": 0}']:
        with pytest.raises(P.InvalidArgument):
            pio.config_from_json(bad)


def test_report_json_roundtrip():
    import ctypes as C
    from paper_2604_17001_b200._lib import SolveReportC
    obj = np.array([3.0, 2.0, 1.5])
    res = np.array([0.1, np.nan, 0.01])
    r = SolveReportC()
    r.iterations = 3
    r.objective = obj.ctypes.data_as(C.POINTER(C.c_double))
    r.primal_residual = res.ctypes.data_as(C.POINTER(C.c_double))
    r.termination = 1
    r.wall_time_seconds = 0.5
    n = P.lib().icnnm_report_to_json(C.byref(r), None, 0)
    buf = C.create_string_buffer(n + 1)
    P.lib().icnnm_report_to_json(C.byref(r), buf, n + 1)
    d = json.loads(buf.value.decode())
    assert d["iterations"] == 3 and d["termination"] == "converged"
    assert d["objective"] == [3.0, 2.0, 1.5] and d["primal_residual"] == [0.1, None, 0.01]


def test_cli_errors_are_json(tmp_path):
    out = subprocess.run([CLI_PATH, "complete", "--input", str(tmp_path / "none.tnsr"),
                          "--mask", "m", "--basis", "b", "--out", "o"],
                         capture_output=True, text=True)
    assert out.returncode == 1
    assert "cannot open file" in json.loads(out.stderr)["error"]
    out = subprocess.run([CLI_PATH, "learn", "--kernel", "3,3"], capture_output=True, text=True)
    assert out.returncode == 1 and "required" in json.loads(out.stderr)["error"]
