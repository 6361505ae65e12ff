"""Pipelined protocol (CudaTarget.execute_many over tsg_submit_timed /
tsg_collect): same statuses and verified outputs as the one-by-one
``execute``, failures in the middle of the pipeline (compile failure,
verification failure, rejected launch) map exactly as they do there, and
a consumer that stops early leaves no slot in flight."""

import numpy as np
import pytest

from oracle import kernels_ffi as K
from paper_2407_11488_b200.cuda_backend import CudaTarget
from paper_2407_11488_b200.measure import MeasurementProtocol, Status, cuda_backend
from paper_2407_11488_b200.problems import Convolution, Hotspot
from paper_2407_11488_b200.strategies import brute_force
from paper_2407_11488_b200.sweep import stratified_sample

pytestmark = pytest.mark.gpu

PROTO = MeasurementProtocol(warmup_runs=1, benchmark_runs=3)


@pytest.fixture(scope="module")
def device():
    from paper_2407_11488_b200 import runtime as rt

    d = rt.Device(0)
    yield d
    d.close()


def test_pipelined_matches_sequential(device):
    prob = Hotspot(width=300, height=260, iterations=20)
    want = K.answer(prob)
    configs = stratified_sample(prob.space, 24, seed=4, param="temporal_tiling_factor")
    configs += [(1024, 1, 1, 1, 1, 1, 0), (32, 32, 1, 1, 10, 5, 1)]
    tgt = CudaTarget(prob, device=device, answer=want)
    try:
        seq = {c: tgt.execute(c, PROTO) for c in configs}
        for depth in (1, 2, 3, 4):
            tgt.pipeline_depth = depth
            pip = list(tgt.execute_many(configs, PROTO))
            assert [c for c, _ in pip] == configs
            assert [o.status for _, o in pip] == [seq[c].status for c in configs]
        for c, o in pip:
            assert o.status is seq[c].status, (c, o, seq[c])
            if o.ok:
                assert len(o.times_ms) == 3 and o.time_ms > 0
                assert tgt.extras[",".join(map(str, c))]["verify"]["n_bad"] == 0
                # same kernel, same protocol: times agree to within noise
                assert 0.5 < o.time_ms / seq[c].time_ms < 2.0, (c, o.time_ms, seq[c].time_ms)
        assert sum(o.ok for _, o in pip) >= 0.9 * len(configs)
        # device timeline (tsg_slot_timeline): submissions run in order,
        # back to back, each containing its 1 + 3 runs
        tl = [tgt.extras[",".join(map(str, c))] for c, o in pip if o.ok]
        for a, b in zip(tl, tl[1:]):
            assert a["t_dev_start_ms"] < a["t_dev_end_ms"] <= b["t_dev_start_ms"] + 1e-3
        for (c, o), x in zip([co for co in pip if co[1].ok], tl):
            assert x["t_dev_end_ms"] - x["t_dev_start_ms"] >= 0.99 * sum(o.times_ms)
        # and the outputs really are the verified ones
        st, out = tgt.run_output(configs[0])
        assert st is Status.OK and np.array_equal(out, K.tuned(prob))
    finally:
        tgt.close()


def test_pipeline_failures_in_the_middle(device):
    prob = Convolution(width=272, height=200)
    want = K.answer(prob)
    configs = stratified_sample(prob.space, 12, seed=2, param="block_size_x")
    tgt = CudaTarget(prob, device=device, answer=want)
    orig = tgt.source_for
    try:
        broken = {configs[3], configs[7]}
        names = prob.space.param_names
        tgt.source_for = lambda cfg: ("#error broken on purpose\n" + orig(cfg)
                                      if tuple(cfg[n] for n in names) in broken else orig(cfg))
        res = list(tgt.execute_many(configs, PROTO))
        assert [c for c, _ in res] == configs
        for c, o in res:
            if c in broken:
                assert o.status is Status.COMPILE_FAILED and "broken on purpose" in o.detail
            else:
                assert o.status in (Status.OK, Status.INVALID), (c, o)
        # early stop: the generator is closed with a slot in flight
        gen = tgt.execute_many(configs[:6], PROTO)
        first = [next(gen) for _ in range(2)]
        gen.close()
        assert len(first) == 2
        again = list(tgt.execute_many(configs[:4], PROTO))
        assert len(again) == 4
    finally:
        tgt.close()
    # wrong answer buffer: every configuration fails verification, in order
    tgt = CudaTarget(prob, device=device, answer=want + 1.0)
    try:
        res = list(tgt.execute_many(configs[:5], PROTO))
        for c, o in res:
            if o.status is not Status.INVALID:
                assert o.status is Status.RUNTIME_FAILED and "verification failed" in o.detail, (c, o)
    finally:
        tgt.close()


def test_brute_force_pipelined_trace(device):
    """brute_force over an explicit list through the cuda backend: the
    trace is the list order, every configuration measured once."""
    prob = Convolution(width=272, height=200)
    tgt = CudaTarget(prob, device=device, answer=K.answer(prob))
    try:
        configs = stratified_sample(prob.space, 16, seed=9, param="tile_size_y")
        result, cache = brute_force(prob.space, cuda_backend(tgt), PROTO, configs=configs)
        assert [c for c, _ in result.trace] == configs
        assert len(cache.records) == len(set(configs))
        ok = [o for _, o in result.trace if o.ok]
        assert ok and all(o.metric_value is not None for o in ok)
        assert result.best_observation.time_ms == min(o.time_ms for o in ok)
    finally:
        tgt.close()
