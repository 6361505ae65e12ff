"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

* small problems, many configurations per space (stratified, including
  the extreme block shapes): kernel output BIT-EXACT vs the C oracle's
  restatement of the tuned arithmetic (``K.tuned``: the answer itself,
  except hotspot's folded-coefficient form, itself within 1e-6 of the
  Rodinia answer -- tests/test_oracle.py);
* full BASELINE sizes: the on-device answer kernel bit-exact vs the
  oracle, then a sweep of configurations verified on-device against it
  (tolerance stated in the test: rtol 1e-5 norm-wise; 0 expected except
  for hotspot's folded form);
* failure mapping: NVRTC error -> compile_failed, oversize launch ->
  invalid, never an exception.
"""

import numpy as np
import pytest

from oracle import kernels_ffi as K
from paper_2407_11488_b200.cuda_backend import CudaTarget
from paper_2407_11488_b200.measure import MeasurementProtocol, Status
from paper_2407_11488_b200.problems import Convolution, Dedispersion, Gemm, Hotspot
from paper_2407_11488_b200.sweep import stratified_sample

pytestmark = pytest.mark.gpu

PROTO = MeasurementProtocol(warmup_runs=1, benchmark_runs=2)

SMALL = {
    "convolution": (lambda: Convolution(width=272, height=200), "tile_size_y", 40),
    "hotspot": (lambda: Hotspot(width=300, height=260, iterations=20), "temporal_tiling_factor", 60),
    "dedispersion": (lambda: Dedispersion(channels=48, samples=700, dms=96, dm_step=1.0), "tile_size_y", 40),
    "gemm": (lambda: Gemm(m=256, n=128, k=96), "VWM", 40),
}

EDGE = {
    "convolution": [(16, 1, 1, 1, 0, 0, 0), (256, 4, 4, 4, 1, 0, 0), (16, 16, 4, 4, 1, 1, 1),
                    (240, 1, 3, 2, 0, 1, 1)],
    "hotspot": [(1, 32, 1, 1, 1, 1, 0), (1024, 1, 1, 1, 1, 1, 0), (32, 32, 1, 1, 10, 5, 1),
                (4, 8, 10, 10, 3, 1, 1)],
    "dedispersion": [(1, 32, 1, 1, 0, 0), (32, 32, 4, 8, 1, 1), (4, 256, 3, 4, 0, 1)],
    "gemm": [(16, 16, 16, 8, 8, 8, 8, 1, 1, 0, 0, 0, 0), (128, 128, 32, 16, 16, 16, 16, 8, 8, 1, 1, 1, 1),
             (64, 128, 16, 8, 16, 8, 16, 8, 4, 1, 0, 1, 0)],
}


@pytest.fixture(scope="module")
def device():
    from paper_2407_11488_b200 import runtime as rt

    d = rt.Device(0)
    yield d
    d.close()


@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_problem_bit_exact(name, device):
    make, param, n = SMALL[name]
    prob = make()
    want = K.answer(prob)
    tuned = K.tuned(prob)
    tgt = CudaTarget(prob, device=device, answer=want)
    try:
        ref = tgt.answer()
        np.testing.assert_array_equal(ref, want)
        configs = EDGE[name] + stratified_sample(prob.space, n, seed=11, param=param)
        assert all(prob.space.is_valid(c) for c in configs)
        ok = 0
        for c in configs:
            obs = tgt.execute(c, PROTO)
            assert obs.status in (Status.OK, Status.INVALID), (c, obs)
            if not obs.ok:
                continue
            st, out = tgt.run_output(c)
            assert st is Status.OK, (c, out)
            diff = int(np.sum(out != tuned))
            assert diff == 0, f"{name} {c}: {diff} elements differ"
            ok += 1
        assert ok >= 0.9 * len(configs)
    finally:
        tgt.close()


FULL = {"convolution": (Convolution, "tile_size_y", 12), "hotspot": (Hotspot, "temporal_tiling_factor", 20),
        "dedispersion": (Dedispersion, "tile_size_y", 4), "gemm": (Gemm, "VWM", 6)}


@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size_answer_and_sweep(name, device):
    cls, param, n = FULL[name]
    prob = cls()
    tgt = CudaTarget(prob, device=device)  # answer = naive reference kernel on device
    try:
        np.testing.assert_array_equal(tgt.answer(), K.answer(prob))
        for c in stratified_sample(prob.space, n, seed=5, param=param):
            obs = tgt.execute(c, PROTO)
            assert obs.status in (Status.OK, Status.INVALID), (c, obs)
            if obs.ok:
                rel = tgt.extras[",".join(map(str, c))]["verify_rel_err"]
                assert rel <= 1e-5, (c, rel)  # tolerance: 1e-5 norm-wise
                if name != "hotspot":  # hotspot: folded form, ~1e-6 (tests/test_oracle.py)
                    assert rel == 0.0, (c, rel)
    finally:
        tgt.close()


def _stream_configs(prob, n_per_t=4, mode="stream"):
    """Stream-mode configurations: every T, odd and even TSX, both sh_power
    values, one and two rows per iteration."""
    names = prob.space.param_names
    out = []
    for c in stratified_sample(prob.space, 2000, seed=23, param="temporal_tiling_factor"):
        d = dict(zip(names, c))
        if prob.kernel_mode(d)[0] == mode:
            key = (d["temporal_tiling_factor"], d["tile_size_x"] % 2, d["sh_power"],
                   d["loop_unroll_factor_t"] > 1)
            if sum(1 for o in out if o[0] == key) < 1:
                out.append((key, c))
    return [c for _, c in out]


def test_hotspot_stream_mode_bit_exact(device):
    """Warp-streaming hotspot (TMA bulk rows, shuffles, register level rings):
    every T (incl. the remainder launch of 20 % T), odd/even TSX, power in
    smem or through L1, grid edges -- bit-exact vs the C oracle."""
    prob = Hotspot(width=520, height=264, iterations=20)
    want = K.tuned(prob)
    tgt = CudaTarget(prob, device=device, answer=K.answer(prob))
    try:
        configs = _stream_configs(prob)
        assert len(configs) >= 30
        for c in configs:
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
            st, out = tgt.run_output(c)
            assert st is Status.OK, (c, out)
            diff = int(np.sum(out != want))
            assert diff == 0, f"stream {c}: {diff} elements differ"
    finally:
        tgt.close()


def test_hotspot_stream_smem_mode_bit_exact(device):
    """Warp-streaming hotspot with the level rings in shared memory (the
    register-heavy TT x TSX configurations): every T, odd/even TSX, both
    sh_power values -- bit-exact vs the C oracle."""
    prob = Hotspot(width=520, height=264, iterations=20)
    want = K.tuned(prob)
    tgt = CudaTarget(prob, device=device, answer=K.answer(prob))
    try:
        configs = _stream_configs(prob, mode="stream_smem")
        assert len(configs) >= 12
        for c in configs:
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
            st, out = tgt.run_output(c)
            assert st is Status.OK, (c, out)
            diff = int(np.sum(out != want))
            assert diff == 0, f"stream_smem {c}: {diff} elements differ"
    finally:
        tgt.close()


def test_failure_mapping(device):
    from paper_2407_11488_b200 import runtime as rt

    bad = rt.compile_source('extern "C" __global__ void k() { nope; }', ["--gpu-architecture=sm_100a"])
    assert not bad.ok
    prob = Hotspot(width=64, height=64, iterations=2)
    tgt = CudaTarget(prob, device=device, answer=K.answer(prob))
    try:
        tgt.source = "#error deliberately broken\n" + tgt.source
        obs = tgt.execute((32, 1, 1, 1, 1, 1, 0), PROTO)
        assert obs.status is Status.COMPILE_FAILED and "deliberately broken" in obs.detail
    finally:
        tgt.close()


def test_hotspot_large_smem_configs_run(device):
    """Configurations needing >48 KiB dynamic smem opt in and verify."""
    prob = Hotspot(width=512, height=512, iterations=20)
    want = K.answer(prob)
    tgt = CudaTarget(prob, device=device, answer=want)
    try:
        big = [c for c in prob.space.enumerate_configs()
               if prob.smem_bytes(dict(zip(prob.space.param_names, c))) > 60 * 1024][:5]
        assert big
        for c in big:
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
    finally:
        tgt.close()


def test_gemm_tc_tf32_within_k_scaled_tolerance(device):
    """tcgen05/TMEM/TMA tf32 GEMM vs the fp32 oracle: |dC| <= K * 2^-11 (|a|,|b| <= 1)."""
    from paper_2407_11488_b200.problems import GemmTC

    # the persistent grid capped at 3 CTAs / clusters: every CTA walks several
    # whole and half tiles through both TMEM accumulators
    for max_units in (None, 3):
        prob = GemmTC(m=512, n=512, k=384, max_units=max_units)
        want = K.answer(prob)
        tgt = CudaTarget(prob, device=device, answer=want)
        try:
            for c in prob.space.enumerate_configs():
                obs = tgt.execute(c, PROTO)
                assert obs.ok, (max_units, c, obs)
                st, out = tgt.run_output(c)
                err = float(np.max(np.abs(out.astype(np.float64) - want)))
                assert err <= prob.K * 2.0 ** -11, (max_units, c, err)
                assert err > 0  # it really is tf32, not a silent fp32 path
        finally:
            tgt.close()
    big = GemmTC()
    tgt = CudaTarget(big, device=device)
    try:
        for c in [(256, 4, 1), (256, 6, 2)]:  # single CTA; 2-SM UMMA pair (cta_group::2)
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
            assert tgt.extras[",".join(map(str, c))]["verify"]["max_abs_err"] <= big.abs_tol
    finally:
        tgt.close()


@pytest.mark.parametrize("shape", [(96, 1500, 512, 0.07), (100, 1500, 300, 0.06)],
                         ids=["chunked", "ragged"])
def test_dedispersion_window_mode_bit_exact(device, shape):
    """Register-window dedispersion (warp-uniform shifts, TMA-staged rows,
    pattern dispatch, FADD2): every eligible configuration of the space,
    bit-exact vs the C oracle on problems whose 8-DM groups span up to 3
    samples -- one with whole 32-channel chunks and 256-DM blocks, one with
    a channel tail chunk, a partial DM block and a ragged sample tail."""
    ch, ns, nd, step = shape
    prob = Dedispersion(channels=ch, samples=ns, dms=nd, dm_step=step, ch_bw_mhz=1.0)
    want = K.answer(prob)
    names = prob.space.param_names
    configs = [c for c in prob.space.enumerate_configs()
               if prob.window_span(dict(zip(names, c))) is not None]
    assert len(configs) >= 20
    assert max(prob.window_span(dict(zip(names, c))) for c in configs) == 3
    tgt = CudaTarget(prob, device=device, answer=want)
    try:
        for c in configs:
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
            st, out = tgt.run_output(c)
            assert st is Status.OK, (c, out)
            diff = int(np.sum(out != want))
            assert diff == 0, f"window {c}: {diff} elements differ"
    finally:
        tgt.close()


@pytest.mark.parametrize("staged", ["all", "0"], ids=["staged", "plain"])
def test_dedispersion_generic_modes_bit_exact(device, monkeypatch, staged):
    """Generic dedispersion, both kernels: the TMA-staged one (5..2-deep
    ring sized to the block's DM spread; TSG_DD_STG=all forces it wherever
    it fits) and the plain load-per-add one (TSG_DD_STG=0).  Partial last warp (1x40 threads), channel tail chunk,
    partial DM block, ragged sample tail, strided and contiguous tiles."""
    monkeypatch.setenv(Dedispersion.STAGED_ENV, staged)
    prob = Dedispersion(channels=200, samples=3001, dms=300, dm_step=0.05, ch_bw_mhz=1.0)
    want = K.answer(prob)
    names = prob.space.param_names
    configs = [(1, 40, 1, 1, 0, 0), (2, 48, 3, 4, 1, 1), (16, 64, 4, 3, 1, 0), (4, 256, 2, 8, 0, 1),
               (8, 128, 3, 7, 1, 1), (32, 32, 4, 2, 0, 1), (1, 256, 4, 8, 0, 0)]
    configs += stratified_sample(prob.space, 24, seed=5, param="block_size_x")
    tgt = CudaTarget(prob, device=device, answer=want)
    try:
        n_staged = 0
        for c in configs:
            cfg = dict(zip(names, c))
            if prob.window_span(cfg) is not None:
                continue
            n_staged += bool(prob.staged_stages(cfg))
            obs = tgt.execute(c, PROTO)
            assert obs.ok, (c, obs)
            st, out = tgt.run_output(c)
            assert st is Status.OK, (c, out)
            diff = int(np.sum(out != want))
            assert diff == 0, f"generic {c} staged={staged}: {diff} elements differ"
        assert n_staged == (0 if staged == "0" else len([c for c in configs
                                                           if prob.window_span(dict(zip(names, c))) is None]))
    finally:
        tgt.close()
