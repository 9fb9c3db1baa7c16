"""Pin the device's math restatements to this host's libm / numpy (CPU).

The kernels' softplus (dynamics.py:59's np.logaddexp) is restated from
glibc 2.39 expf/log1pf in csrc/ss_math.cuh.  oracle/libm_pin compiles that
header as host C++ and compares it with libm bit-for-bit; here we run a
sampled sweep (the exhaustive sweep, `make -C oracle pin-full`, is recorded in
DESIGN.md) and check that numpy's float32 logaddexp(0, z) is exactly
z + log1pf(expf(-z)) on this machine.
"""
import ctypes
import ctypes.util
import subprocess
from pathlib import Path

import numpy as np
import pytest

ORACLE = Path(__file__).resolve().parents[1] / "oracle"


@pytest.fixture(scope="module")
def pin_binary():
    subprocess.run(["make", "-s", "-C", str(ORACLE), "libm_pin", "abi_layout"], check=True)
    return ORACLE / "libm_pin"


def test_restated_expf_log1pf_softplus_bitexact(pin_binary):
    res = subprocess.run([str(pin_binary), "4099"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "expf   0 /" in res.stdout and "log1pf 0 /" in res.stdout and "softplus 0 /" in res.stdout


def test_numpy_logaddexp_is_glibc_composition():
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.expf.restype = ctypes.c_float
    libm.expf.argtypes = [ctypes.c_float]
    libm.log1pf.restype = ctypes.c_float
    libm.log1pf.argtypes = [ctypes.c_float]
    rng = np.random.default_rng(0)
    # z = (d_min - d) / k over contact depths: 0 .. d_min / 1e-3
    z = np.concatenate([rng.uniform(0, 100, 20000), rng.uniform(0, 2, 20000),
                        rng.exponential(5.0, 10000)]).astype(np.float32)
    got = np.logaddexp(np.float32(0.0), z)
    want = np.array([np.float32(zz) + np.float32(libm.log1pf(libm.expf(-zz))) if zz != 0 else np.float32(np.log(2))
                     for zz in z], dtype=np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
