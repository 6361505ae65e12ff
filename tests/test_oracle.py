"""Pin the CPU oracle (no GPU).

The reference has no kernel arithmetic, so the C oracle
is pinned by known-answer tests and by independent float64 numpy
restatements at small sizes.
"""

import numpy as np
import pytest

from oracle import kernels_ffi as K
from paper_2407_11488_b200.problems import Convolution, Dedispersion, Gemm, Hotspot


def test_conv_delta_filter_is_identity():
    p = Convolution(width=64, height=48)
    img = p.image()
    padded = np.zeros((p.rows, p.pitch), np.float32)
    padded[: p.in_h, : p.in_w] = img
    f = np.zeros((15, 15), np.float32)
    f[0, 0] = 1.0
    out = np.empty(64 * 48, np.float32)
    K.lib().oracle_convolution(K._p(out), K._p(padded), p.pitch, 64, 48, K._p(f.ravel().copy()), 15, 15)
    np.testing.assert_array_equal(out.reshape(48, 64), img[:48, :64])


def test_conv_matches_float64():
    p = Convolution(width=96, height=40)
    got = K.convolution(p).astype(np.float64)
    want = K.convolution_f64(p)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-6


def test_hotspot_ambient_fixed_point():
    p = Hotspot(width=40, height=30, iterations=7)
    amb = np.full((30, 40), p.k["amb"], np.float32)
    zero = np.zeros((30, 40), np.float32)
    out = np.empty(1200, np.float32)
    scratch = np.empty_like(out)
    k = p.k
    K.lib().oracle_hotspot(K._p(out), K._p(amb), K._p(zero), 40, 30, 7, k["sdc"], k["rx1"], k["ry1"],
                           k["rz1"], k["amb"], K._p(scratch))
    np.testing.assert_array_equal(out, amb.ravel())


def test_hotspot_matches_float64():
    p = Hotspot(width=64, height=48, iterations=20)
    got = K.hotspot(p).astype(np.float64)
    want = K.hotspot_f64(p)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-5


@pytest.mark.parametrize("shape", [(64, 48), (520, 264), (1024, 1024)])
def test_hotspot_tuned_form_within_tolerance(shape):
    """The tuned kernels' folded-coefficient arithmetic vs the Rodinia form
    and float64: well inside the north_star rtol 1e-5 (elementwise)."""
    w, h = shape
    p = Hotspot(width=w, height=h, iterations=20)
    fast = K.hotspot_tuned(p).astype(np.float64)
    rod = K.hotspot(p).astype(np.float64)
    f64 = K.hotspot_f64(p)
    assert np.max(np.abs(fast - rod) / np.abs(rod)) < 2e-6
    assert np.max(np.abs(fast - f64)) / np.max(np.abs(f64)) < 2e-6
    assert not np.array_equal(fast, rod)  # really the other operation order


def test_hotspot_tuned_coefficients_expand_rodinia():
    p = Hotspot(width=8, height=8)
    k, c = p.k, p.tuned_coefficients(p.k)
    assert c["ax"] == pytest.approx(k["sdc"] * k["rx1"], rel=1e-7)
    assert c["at"] + 2 * c["ax"] + 2 * c["ay"] + k["sdc"] * k["rz1"] == pytest.approx(1.0, rel=1e-6)
    assert c["ac"] == pytest.approx(k["sdc"] * k["rz1"] * k["amb"], rel=1e-7)


def test_hotspot_tuned_ambient_fixed_point():
    """Zero power at ambient temperature stays (to fp32 rounding) at ambient."""
    p = Hotspot(width=40, height=30, iterations=7)
    amb = np.full((30, 40), p.k["amb"], np.float32)
    zero = np.zeros((30, 40), np.float32)
    out = np.empty(1200, np.float32)
    scratch = np.empty_like(out)
    c = p.tuned_coefficients(p.k)
    K.lib().oracle_hotspot_tuned(K._p(out), K._p(amb), K._p(zero), 40, 30, 7, c["at"], c["ay"], c["ax"],
                                 c["ap"], c["ac"], K._p(scratch))
    assert np.max(np.abs(out - p.k["amb"])) < 1e-4


def test_hotspot_is_stable_at_full_size_constants():
    """Pinned cell size keeps the explicit scheme stable."""
    p = Hotspot(width=256, height=256, iterations=20)
    out = K.hotspot(p)
    assert np.all(np.isfinite(out))
    assert 300.0 < out.min() and out.max() < 340.0
    assert p.k["sdc"] * (2 * p.k["rx1"] + 2 * p.k["ry1"]) < 1.0


def test_dedisp_zero_shift_is_channel_sum():
    p = Dedispersion(channels=16, samples=200, dms=4, dm_step=0.0)
    got = K.dedispersion(p).reshape(4, 200)
    data = p.data()
    want = np.zeros(200, np.float32)
    for ch in range(16):
        want = want + data[ch, :200]
    for d in range(4):
        np.testing.assert_array_equal(got[d], want)


def test_dedisp_matches_float64():
    p = Dedispersion(channels=32, samples=300, dms=24, dm_step=2.0)
    got = K.dedispersion(p).astype(np.float64)
    want = K.dedispersion_f64(p)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-5
    assert p.max_shift > 0


def test_gemm_identity():
    g = Gemm(m=32, n=16, k=32)
    a = np.eye(32, dtype=np.float32)  # a(m,k) = A[k*M+m] -> identity
    b = g.b()
    c = np.empty(32 * 16, np.float32)
    K.lib().oracle_gemm(K._p(c), K._p(a.copy()), K._p(b), 32, 16, 32)
    # c(m,n) = b(m,n) -> C[n*M+m] = B[m*N+n]
    np.testing.assert_array_equal(c.reshape(16, 32), b.T)


def test_gemm_matches_float64():
    g = Gemm(m=64, n=48, k=80)
    got = K.gemm(g).astype(np.float64)
    want = K.gemm_f64(g)
    assert np.max(np.abs(got - want)) <= 80 * 2.0 ** -24 * 80 * 4


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_is_thread_count_invariant(threads):
    p = Hotspot(width=64, height=64, iterations=5)
    K.set_threads(threads)
    try:
        a = K.hotspot(p)
    finally:
        K.set_threads(0)
    np.testing.assert_array_equal(a, K.hotspot(p))
