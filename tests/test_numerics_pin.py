"""The kernels' exact numerics (csrc/ss_math.cuh, compiled for the host as
oracle/libsspin.so) pinned against numpy on this machine (CPU):

* float32 sin / cos  == np.sin / np.cos (geometry.py:24,32,82);
* softplus            == np.logaddexp(0, z)  (dynamics.py:59);
* Philox draw / advance / uniform == numpy's Generator(Philox) stream,
  including partially consumed buffers (batching.py:174-198).
"""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2207_03530_b200.batching import state_to_words

ORACLE = Path(__file__).resolve().parents[1] / "oracle"


@pytest.fixture(scope="module")
def pin():
    subprocess.run(["make", "-s", "-C", str(ORACLE), "libsspin.so"], check=True)
    lib = ctypes.CDLL(str(ORACLE / "libsspin.so"))
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.pin_np_sincosf.argtypes = [vp, vp, i64, ctypes.c_int]
    lib.pin_softplus.argtypes = [vp, vp, i64]
    lib.pin_philox_draw.argtypes = [vp, vp, vp, i64]
    lib.pin_philox_advance.argtypes = [vp, ctypes.c_uint64, vp]
    lib.pin_uniform_f32.argtypes = [vp, ctypes.c_double, ctypes.c_double, vp, i64]
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_sincos_matches_numpy(pin):
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.uniform(-np.pi, np.pi, 2_000_000), rng.uniform(-50, 50, 500_000),
        rng.uniform(-8e4, 8e4, 100_000), [0.0, -0.0, np.pi, -np.pi, np.pi / 2, 1e-30, -1e-30],
    ]).astype(np.float32)
    for want_cos, fn in ((1, np.cos), (0, np.sin)):
        out = np.empty_like(x)
        pin.pin_np_sincosf(_p(x), _p(out), x.size, want_cos)
        np.testing.assert_array_equal(out.view(np.uint32), fn(x).view(np.uint32))


def test_softplus_matches_numpy_logaddexp(pin):
    rng = np.random.default_rng(1)
    z = np.concatenate([rng.uniform(0, 120, 1_000_000), rng.exponential(3.0, 500_000), [0.0, 1e-30, 88.0, 104.0]])
    z = z.astype(np.float32)
    out = np.empty_like(z)
    pin.pin_softplus(_p(z), _p(out), z.size)
    np.testing.assert_array_equal(out.view(np.uint32), np.logaddexp(np.float32(0), z).view(np.uint32))


@pytest.mark.parametrize("consumed", [0, 1, 2, 3, 4, 5, 11])
def test_philox_stream_matches_numpy(pin, consumed):
    bg = np.random.Philox(1234 + consumed)
    bg.random_raw(consumed)
    state = bg.state
    words = state_to_words(state)
    idx = np.array([0, 1, 2, 3, 4, 5, 6, 7, 100, 1001, 65537, 4_000_003], dtype=np.uint64)
    got = np.empty(idx.size, dtype=np.uint64)
    pin.pin_philox_draw(_p(words), _p(idx), _p(got), idx.size)
    ref = np.random.Philox()
    ref.state = state
    raw = ref.random_raw(int(idx.max()) + 1)
    np.testing.assert_array_equal(got, raw[idx.astype(np.int64)])
    for n in (0, 1, 3, 4, 5, 17, 1000):
        adv = np.empty(12, dtype=np.uint64)
        pin.pin_philox_advance(_p(words), n, _p(adv))
        r2 = np.random.Philox()
        r2.state = state
        r2.random_raw(n)
        np.testing.assert_array_equal(adv[:11], state_to_words(r2.state)[:11])


def test_uniform_matches_generator(pin):
    g = np.random.Generator(np.random.Philox(5))
    st0 = g.bit_generator.state
    want = g.uniform(-0.9, 0.9, 4096).astype(np.float32)
    r = np.random.Philox()
    r.state = st0
    u = r.random_raw(4096)
    got = np.empty(4096, dtype=np.float32)
    pin.pin_uniform_f32(_p(u), -0.9, 0.9 - (-0.9), _p(got), 4096)
    np.testing.assert_array_equal(got, want)
