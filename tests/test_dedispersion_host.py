"""Host-side logic of the window dedispersion kernel (no GPU).

* eligibility / SPAN / BLKSPAN from the exact fp32 shift table;
* the generated inline-PTX jump-table dispatch: one case per increment
  pattern of popcount <= SPAN, in the kernel's dense (span-major) order,
  compiling with NVRTC for sm_100a.
"""

import re

import numpy as np
import pytest

from paper_2407_11488_b200 import runtime as rt
from paper_2407_11488_b200.problems import Dedispersion, dd_asm_dispatch, dm_shifts


def test_window_eligibility_and_spans():
    p = Dedispersion()
    names = p.space.param_names
    elig = [c for c in p.space.enumerate_configs() if p.window_span(dict(zip(names, c))) is not None]
    assert len(elig) == 32 and all(c[0] == 32 and c[1] == 32 for c in elig)
    sh = dm_shifts(p.delay, p.NDM, p.dm_first, p.dm_step).astype(np.int64)
    assert np.diff(sh, axis=0).max() == 1  # adjacent DMs shift by 0 or 1 sample
    g = sh.reshape(-1, 8, p.NCH)
    assert p.window_span(dict(zip(names, (32, 32, 4, 8, 1, 0)))) == int((g[:, -1] - g[:, 0]).max()) == 3
    blk = p.block_span(dict(zip(names, (32, 32, 4, 8, 1, 0))))
    assert blk == int((sh[255::256] - sh[0::256]).max())
    # smem: 3 stages x 32 rows + barriers + delay table + pattern table, under the opt-in cap
    assert p.smem_bytes(dict(zip(names, (32, 32, 4, 8, 1, 0)))) < 227 * 1024


@pytest.mark.parametrize("tsx,tsy,span", [(2, 1, 0), (2, 4, 1), (4, 6, 2), (4, 8, 3), (2, 8, 3)])
def test_asm_dispatch_cases(tsx, tsy, span):
    code = dd_asm_dispatch(tsx, tsy, span)
    pats = [q for q in range(1 << (tsy - 1)) if bin(q).count("1") <= span]
    # the single-channel block (section a) and the two-channel block
    # (sections a, b: one dispatch per channel, in order)
    one, two = code.split("dd_asm_dispatch2")
    blocks = ((one, "a"), (two, "ab"))  # one and two channels per block
    for text, secs in blocks:
        for sec in secs:
            labels = re.findall(rf"L{sec}(\d+)_%=:", text)
            assert [int(x) for x in labels] == list(range(len(pats)))
        # adds per case = TSY x TSX/2 packed accumulators, per channel
        assert text.count("add.rn.f32x2") == len(secs) * len(pats) * tsy * (tsx // 2)


def test_asm_dispatch_source_compiles_for_sm100a():
    p = Dedispersion()
    names = p.space.param_names
    cfg = dict(zip(names, (32, 32, 4, 8, 1, 0)))
    src = p.source_for(cfg)
    assert "#define DD_HAVE_ASM" in src
    res = rt.compile_source(src, p.options(cfg))
    assert res.ok, res.error
    assert "#define DD_HAVE_ASM" not in p.source_for(dict(zip(names, (32, 32, 2, 4, 1, 0))))
    odd = dict(zip(names, (32, 32, 3, 8, 1, 0)))
    assert "#define DD_HAVE_ASM" not in p.source_for(odd)  # odd TSX keeps the C++ switch


def test_staged_generic_selection_and_smem():
    """Host side of the staged generic kernel (kernels/dedispersion.cu DD_STG):
    window and staged modes are exclusive, the selection rule is the measured
    one, the ring depth is the deepest (<= 5) that fits 200 KiB, and the
    smem size matches the kernel's layout (stages of CC rows of ROWLEN floats,
    2 x NSTAGE mbarriers, the delay table)."""
    import collections

    p = Dedispersion()
    names = p.space.param_names
    seen = collections.Counter()
    for c in p.space.enumerate_configs():
        cfg = dict(zip(names, c))
        d = p.config_defines(cfg)
        assert not ("DD_WIN" in d and "DD_STG" in d)
        ns = p.staged_stages(cfg)
        if "DD_WIN" in d:
            seen["window"] += 1
            continue
        rule = cfg["block_size_x"] >= 4 and cfg["block_size_x"] * cfg["tile_size_x"] >= 12 \
            and cfg["tile_size_x"] * cfg["tile_size_y"] >= 8
        assert bool(ns) == rule, c
        if not ns:
            assert p.smem_bytes(cfg) == 0
            seen["plain"] += 1
            continue
        seen["staged"] += 1
        assert d["DD_STG"] == 1 and d["DD_NSTAGE"] == ns and 2 <= ns <= 5
        rowlen = (cfg["block_size_x"] * cfg["tile_size_x"] + p.block_span(cfg) + 4 + 3) & ~3
        want = 4 * ns * 32 * rowlen + 16 * ns + 4 * p.NCH
        assert p.smem_bytes(cfg) == want <= 200 * 1024
        if ns < 5:  # one stage deeper would not fit
            assert 4 * (ns + 1) * 32 * rowlen + 16 * (ns + 1) + 4 * p.NCH > 200 * 1024
        # staged rows stay inside the padded input row (no read past the pitch)
        assert p.NSAMP - 1 + p.max_shift + rowlen + 3 <= p.pitch
    assert seen["staged"] > 2000 and seen["plain"] > 5000 and seen["window"] > 0


def test_staged_mode_env_overrides(monkeypatch):
    p = Dedispersion()
    cfg = dict(zip(p.space.param_names, (2, 48, 3, 4, 1, 1)))  # narrow: plain by the rule
    assert p.staged_stages(cfg) == 0
    monkeypatch.setenv(Dedispersion.STAGED_ENV, "all")
    assert p.staged_stages(cfg) > 0 and "DD_STG" in p.config_defines(cfg)
    monkeypatch.setenv(Dedispersion.STAGED_ENV, "0")
    wide = dict(zip(p.space.param_names, (16, 64, 4, 3, 1, 0)))
    assert p.staged_stages(wide) == 0 and "DD_STG" not in p.config_defines(wide)
