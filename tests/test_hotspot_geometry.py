"""Host-side geometry of the warp-streaming hotspot kernel (no GPU).

Mirrors the invariants kernels/hotspot.cu relies on (HS_STREAM): bulk
copies and stores need 16-byte aligned window origins and widths, the
useful columns must lie inside the cells that stay valid for TT levels,
strips and segments must tile the grid, and smem must fit.
"""

import numpy as np

from paper_2407_11488_b200.problems import Hotspot
from paper_2407_11488_b200.sweep import stratified_sample


def test_stream_geometry_invariants():
    prob = Hotspot()
    names = prob.space.param_names
    n_stream = 0
    for c in stratified_sample(prob.space, 3000, seed=3, param="temporal_tiling_factor"):
        d = dict(zip(names, c))
        g = prob.stream_geometry(d)
        mode = prob.kernel_mode(d)[0]
        assert (g is not None) == mode.startswith("stream")
        if g is None:
            continue
        n_stream += 1
        t = d["temporal_tiling_factor"]
        assert g["sw"] == 32 * d["tile_size_x"]
        assert g["ta"] % 4 == 0 and g["uw"] % 4 == 0 and g["uw"] >= 4
        assert g["ta"] >= t and g["ta"] + g["uw"] <= g["sw"] - t  # useful cells valid after t levels
        assert g["nstrips"] * g["uw"] >= prob.W and (g["nstrips"] - 1) * g["uw"] < prob.W
        for sh, sh0, ns in ((g["segh"], g["segh0"], g["nsegs"]), (g["seghe"], g["segh0e"], g["nsegse"])):
            assert ns * sh >= prob.H
            last = prob.H - sh0 - (ns - 2) * sh if ns > 1 else prob.H
            assert 0 < sh0 <= sh and 0 < last <= sh  # segments tile the rows
        assert g["blocks"] * g["wpb"] >= g["nxi"] * g["nsegs"] + g["nxe"] * g["nsegse"]
        if g["nxi"]:  # border strips: shorter segments (all-selects code)
            assert g["nsegse"] >= g["nsegs"]
        _check_tiles(prob, g, t)
        assert (g["sw"] * 4) % 16 == 0  # bulk-copy row size
        assert g["smem"] <= Hotspot.STREAM_SMEM_MAX
        assert prob.smem_bytes(d) == g["smem"]
        lau = prob.launches(d, None, {k: _Fake() for k in ("temp", "tmp", "out", "power")})
        assert lau[0].grid == (g["blocks"], 1, 1)
    assert n_stream > 1000


def test_stream_mode_needs_aligned_width():
    d = dict(block_size_x=32, block_size_y=4, tile_size_x=4, tile_size_y=4, temporal_tiling_factor=6,
             loop_unroll_factor_t=6, sh_power=1)
    assert Hotspot(width=4096, height=64).kernel_mode(d)[0] == "stream"
    assert Hotspot(width=4094, height=64).kernel_mode(d)[0] != "stream"
    # too many registers for a 1024-thread block -> block-tile modes
    big = dict(d, block_size_x=1024, block_size_y=1, tile_size_x=4)
    assert Hotspot().kernel_mode(big)[0] != "stream"


class _Fake:
    ptr = 0


def _check_tiles(prob, g, t):
    """Emulate the kernel's warp -> (strip, segment) mapping (hs_stream_body,
    XL/XR): every output cell is produced by exactly one warp, border strips
    are exactly those whose window touches a grid edge."""
    sw, ta, uw, ns = g["sw"], g["ta"], g["uw"], g["nstrips"]
    xl = min(ta // uw + 1, ns)
    xr_raw = 0 if prob.W - 1 - sw + ta < 0 else (prob.W - 1 - sw + ta) // uw + 1
    xr = min(max(xr_raw, xl), ns)
    nxe, nxi = xl + ns - xr, xr - xl
    assert (nxe, nxi) == (g["nxe"], g["nxi"])
    rows = np.zeros((ns,), dtype=np.int64)
    for gi in range(g["blocks"] * g["wpb"]):
        if gi < nxe * g["nsegse"]:
            e = gi % nxe
            strip, seg = (e if e < xl else xr + e - xl), gi // nxe
            sh, nsg, sh0 = g["seghe"], g["nsegse"], g["segh0e"]
        else:
            h = gi - nxe * g["nsegse"]
            if nxi == 0 or h >= nxi * g["nsegs"]:
                continue
            strip, seg = xl + h % nxi, h // nxi
            sh, nsg, sh0 = g["segh"], g["nsegs"], g["segh0"]
        gx0 = strip * uw - ta
        assert (gx0 <= 0 or gx0 + sw > prob.W - 1) == (strip < xl or strip >= xr)
        y0 = 0 if seg == 0 else sh0 + (seg - 1) * sh
        y1 = prob.H if seg == nsg - 1 else min(y0 + (sh0 if seg == 0 else sh), prob.H)
        assert 0 <= y0 < y1 <= prob.H
        rows[strip] += y1 - y0
    assert (rows == prob.H).all()


def test_stream_segments_tile_the_rows():
    """Every segment count the launcher can ask for yields segments that tile
    [0, H) exactly as the kernel computes them (first/last shortened)."""
    for h in (Hotspot(), Hotspot(width=520, height=264), Hotspot(width=64, height=7)):
        for n in range(1, min(h.H, 600) + 1):
            segh, segh0, nsegs = h._segments(n)
            prev = 0
            for seg in range(nsegs):
                y0 = 0 if seg == 0 else segh0 + (seg - 1) * segh
                y1 = h.H if seg == nsegs - 1 else min(y0 + (segh0 if seg == 0 else segh), h.H)
                assert y0 == prev and y1 > y0 and y1 - y0 <= segh, (h.H, n, seg)
                prev = y1
            assert prev == h.H


def test_stream_compile_keys_ignore_launch_geometry():
    """Stream-mode cubins depend on the thread count, not on the block shape
    or TSY (launch geometry): configurations that differ only there share one
    compilation.  Over the whole 105,412-point space that is 5,762 distinct
    NVRTC compilations (5,881 with the round-2 ring depths).""" 
    import collections

    from paper_2407_11488_b200.problems import make_problem

    p = make_problem("hotspot")
    names = p.space.param_names
    a = dict(zip(names, (32, 2, 4, 1, 8, 2, 1)))
    b = dict(zip(names, (64, 1, 4, 3, 8, 4, 1)))  # same 64 threads, other shape/TSY/unroll>1
    assert p.options(a) == p.options(b)
    assert p.source_for(a) == p.source_for(b)
    keys = collections.Counter()
    for c in p.space.enumerate_configs():
        cfg = dict(zip(names, c))
        keys[tuple(p.options(cfg))] += 1
    assert len(keys) == 5881
