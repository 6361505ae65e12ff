"""The paper's four tunable benchmark problems on B200.

Each :class:`Problem` fixes, for one bundled space
(`paper_2407_11488_b200/spaces/*.spec`, identical to ref
`ts/spaces/*.spec`):

* the synthetic inputs (seeded, fp32) and their HBM layout,
* the NVRTC source and the ``-D`` macros a configuration maps to,
* the launch sequence of ONE benchmark run (hotspot: ceil(20/T)
  launches with ping-pong buffers; the others: one launch),
* the naive reference kernel that produces the on-device answer,
* the algorithmic work (FLOP, compulsory bytes) used for roofline
  accounting, and the verification tolerance.

The reference holds none of this: tunescape only has the spaces
(`SURVEY.md` §0.5); kernel definitions follow the paper's BAT / CLBlast
kernels (`PAPER.md:141`) as restated in SURVEY.md §8(a) row a19.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .paramspace import SearchSpaceSpec, bundled_space

KDIR = Path(__file__).resolve().parent / "kernels"


def _src(name: str) -> str:
    return (KDIR / name).read_text()


@dataclass
class BufferSpec:
    name: str
    nbytes: int
    init: np.ndarray | None = None  # host data uploaded at setup (None = scratch)


class Problem:
    """Base class; subclasses define one benchmark kernel family."""

    space_name: str = ""
    source_file: str = ""
    kernel_name: str = ""
    reference_kernel: str = ""
    rtol: float = 1e-5
    atol: float = 0.0
    abs_tol: float | None = None  # when set: pass iff max|out-ref| <= abs_tol
    extra_options: tuple = ()

    def __init__(self):
        self.space: SearchSpaceSpec = bundled_space(self.space_name)
        self._host = None

    # -- inputs --------------------------------------------------------------
    def host_buffers(self) -> list:
        raise NotImplementedError

    def buffers(self) -> list:
        if self._host is None:
            self._host = self.host_buffers()
        return self._host

    def constants(self) -> dict:
        """``__constant__`` symbol -> host array (Kernel Tuner cmem_args)."""
        return {}

    @property
    def output_name(self) -> str:
        return "out"

    @property
    def output_count(self) -> int:
        raise NotImplementedError

    # -- compilation -----------------------------------------------------------
    def source(self) -> str:
        return _src(self.source_file)

    def source_for(self, cfg: dict | None, base: str | None = None) -> str:
        """Source compiled for ``cfg``: the kernel file, plus any per-config
        generated code (default: none)."""
        return base if base is not None else self.source()

    def problem_defines(self) -> dict:
        return {}

    def config_defines(self, cfg: dict) -> dict:
        return {k.upper(): int(v) for k, v in cfg.items()}

    def options(self, cfg: dict | None) -> list:
        # -lineinfo costs ~25% NVRTC time per configuration: only for profiling
        # builds (TSG_LINEINFO=1, set by tools/run_config.py for ncu)
        opts = ["--gpu-architecture=sm_100a", "-std=c++17"] + list(self.extra_options)
        if os.environ.get("TSG_LINEINFO"):
            opts.append("-lineinfo")
        d = dict(self.problem_defines())
        if cfg is not None:
            d.update(self.config_defines(cfg))
        # experiments only: TSG_EXTRA_DEFINES="NAME=V,NAME2=V2"
        for kv in filter(None, os.environ.get("TSG_EXTRA_DEFINES", "").split(",")):
            k, _, v = kv.partition("=")
            d[k] = v or 1
        opts += [f"-D{k}={v}" for k, v in sorted(d.items())]
        return opts

    # -- execution ---------------------------------------------------------------
    def smem_bytes(self, cfg: dict) -> int:
        return 0

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        raise NotImplementedError

    def reference_launches(self, kernel, bufs: dict) -> list:
        raise NotImplementedError

    # -- work accounting -----------------------------------------------------------
    def flops(self, cfg: dict | None = None) -> float:
        return 0.0

    def compulsory_bytes(self, cfg: dict | None = None) -> float:
        return 0.0

    def describe(self) -> dict:
        return {}


def _u64(buf) -> C.c_uint64:
    return C.c_uint64(buf.ptr)


# =============================================================================
# Convolution


class Convolution(Problem):
    """out[y][x] = sum_{i,j<15} in[y+i][x+j] * f[i][j].

    HBM layout: input fp32 [(H+FH-1)+8 rows][IN_PITCH], IN_PITCH =
    round_up(W+FW-1, 4) so every row starts 16-byte aligned (float4 /
    TMA-friendly); 8 zero rows of slack let register-tiled threads read
    past the last row without guards.  Output fp32 [H][W] dense.
    Inputs: U[0,1) image (seed 1), U[0,1) filter (seed 2).
    """

    space_name = "convolution"
    source_file = "convolution.cu"
    kernel_name = "convolution_kernel"
    reference_kernel = "convolution_reference"
    rtol = 1e-5

    def __init__(self, width: int = 4096, height: int = 4096, fw: int = 15, fh: int = 15,
                 seed_image: int = 1, seed_filter: int = 2):
        super().__init__()
        self.W, self.H, self.FW, self.FH = width, height, fw, fh
        self.in_w, self.in_h = width + fw - 1, height + fh - 1
        self.pitch = ((self.in_w + 3) // 4) * 4
        self.rows = self.in_h + 8
        self.seed_image, self.seed_filter = seed_image, seed_filter

    def image(self) -> np.ndarray:
        return np.random.default_rng(self.seed_image).random((self.in_h, self.in_w), dtype=np.float32)

    def filter(self) -> np.ndarray:
        return np.random.default_rng(self.seed_filter).random((self.FH, self.FW), dtype=np.float32)

    def host_buffers(self) -> list:
        padded = np.zeros((self.rows, self.pitch), dtype=np.float32)
        padded[: self.in_h, : self.in_w] = self.image()
        return [BufferSpec("in", padded.nbytes, padded), BufferSpec("out", self.W * self.H * 4)]

    def constants(self) -> dict:
        return {"d_filter": self.filter().ravel()}

    @property
    def output_count(self) -> int:
        return self.W * self.H

    def problem_defines(self) -> dict:
        return dict(IMG_W=self.W, IMG_H=self.H, FW=self.FW, FH=self.FH, IN_PITCH=self.pitch)

    def config_defines(self, cfg: dict) -> dict:
        return dict(BSX=cfg["block_size_x"], BSY=cfg["block_size_y"], TSX=cfg["tile_size_x"],
                    TSY=cfg["tile_size_y"], READ_ONLY=cfg["read_only"],
                    USE_PADDING=cfg["use_padding"], USE_SHMEM=cfg["use_shmem"])

    def smem_bytes(self, cfg: dict) -> int:
        if not cfg["use_shmem"]:
            return 0
        tw = cfg["block_size_x"] * cfg["tile_size_x"]
        th = cfg["block_size_y"] * cfg["tile_size_y"]
        w4 = ((tw + self.FW - 1 + 3) // 4) * 4
        pitch = w4 + (1 if cfg["use_padding"] else 0)
        return (th + self.FH - 1) * pitch * 4

    def grid(self, cfg: dict) -> tuple:
        tw = cfg["block_size_x"] * cfg["tile_size_x"]
        th = cfg["block_size_y"] * cfg["tile_size_y"]
        return (math.ceil(self.W / tw), math.ceil(self.H / th), 1)

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        from .runtime import Launch

        return [Launch(kernel, self.grid(cfg), (cfg["block_size_x"], cfg["block_size_y"], 1),
                       [_u64(bufs["out"]), _u64(bufs["in"])], smem=self.smem_bytes(cfg))]

    def reference_launches(self, kernel, bufs: dict) -> list:
        from .runtime import Launch

        return [Launch(kernel, (math.ceil(self.W / 32), math.ceil(self.H / 8), 1), (256, 1, 1),
                       [_u64(bufs["out"]), _u64(bufs["in"])])]

    def flops(self, cfg=None) -> float:
        return 2.0 * self.W * self.H * self.FW * self.FH

    def compulsory_bytes(self, cfg=None) -> float:
        return 4.0 * (self.in_w * self.in_h + self.W * self.H + self.FW * self.FH)

    def describe(self) -> dict:
        return {"image": f"{self.W}x{self.H}", "filter": f"{self.FW}x{self.FH}", "dtype": "fp32"}


# =============================================================================
# Hotspot


def rodinia_constants(rows: int, cols: int, cell_m: float = 0.016 / 512) -> dict:
    """Rodinia hotspot physical constants -> the kernel's fp32 coefficients.

    Rodinia derives the per-cell geometry from a 0.016 m chip split into
    rows x cols cells; at 4096^2 that makes the explicit scheme unstable
    (sdc*r ~ 2.2 > 1/4).  We keep Rodinia's formulas but pin the CELL size
    to Rodinia's 512^2 default (0.016/512 m), i.e. a proportionally larger
    chip, so the 20-step run stays physical.  Unpinned by the reference
    (SURVEY 8a a19); DESIGN.md records the choice.
    """
    max_pd, precision, spec_heat_si, k_si, factor_chip = 3.0e6, 0.001, 1.75e6, 100.0, 0.5
    t_chip, amb = 0.0005, 80.0
    gh = gw = cell_m
    cap = factor_chip * spec_heat_si * t_chip * gw * gh
    rx = gw / (2.0 * k_si * t_chip * gh)
    ry = gh / (2.0 * k_si * t_chip * gw)
    rz = t_chip / (k_si * gh * gw)
    max_slope = max_pd / (factor_chip * t_chip * spec_heat_si)
    step = precision / max_slope
    f32 = lambda v: float(np.float32(v))  # noqa: E731
    return dict(sdc=f32(step / cap), rx1=f32(1.0 / rx), ry1=f32(1.0 / ry), rz1=f32(1.0 / rz),
                amb=f32(amb))


class Hotspot(Problem):
    """Rodinia hotspot, ``iterations`` explicit steps on a GH x GW grid.

    One benchmark run = ceil(iterations / T) launches (T =
    temporal_tiling_factor), the last advancing the remainder; buffers
    ping-pong between ``tmp`` and ``out`` so the pristine input ``temp``
    is never overwritten (every run does identical work) and the final
    state always lands in ``out``.
    Inputs: temp = 323.15 + U[0,10) (seed 3), power =
    U[0,1)*1e-3 (seed 4), fp32 [GH][GW].
    """

    space_name = "hotspot"
    source_file = "hotspot.cu"
    kernel_name = "hotspot_kernel"
    reference_kernel = "hotspot_reference"
    rtol = 1e-5  # north_star tolerance vs the Rodinia-form answer (elementwise |d| <= 1e-5 |ref|)
    extra_options = ("--fmad=false",)
    # algorithmic FLOP per cell update: the Rodinia form's 4 FADD + 5 FMA
    # (the reference kernel's HS_STEP; the tuned kernels need 5 operations)
    FLOP_PER_CELL = 15

    def __init__(self, width: int = 4096, height: int = 4096, iterations: int = 20,
                 seed_temp: int = 3, seed_power: int = 4):
        super().__init__()
        self.W, self.H, self.iterations = width, height, iterations
        self.seed_temp, self.seed_power = seed_temp, seed_power
        self.k = rodinia_constants(height, width)

    def temperature(self) -> np.ndarray:
        rng = np.random.default_rng(self.seed_temp)
        return (np.float32(323.15) + rng.random((self.H, self.W), dtype=np.float32) * np.float32(10.0))

    def power(self) -> np.ndarray:
        rng = np.random.default_rng(self.seed_power)
        return rng.random((self.H, self.W), dtype=np.float32) * np.float32(1e-3)

    def host_buffers(self) -> list:
        n = self.W * self.H * 4
        return [BufferSpec("temp", n, self.temperature()), BufferSpec("power", n, self.power()),
                BufferSpec("tmp", n), BufferSpec("out", n)]

    @property
    def output_count(self) -> int:
        return self.W * self.H

    def problem_defines(self) -> dict:
        return dict(GW=self.W, GH=self.H)

    def config_defines(self, cfg: dict) -> dict:
        """Compile-time macros of one configuration.

        Stream kernels (kinds 1, 2) see only what changes their code: the
        thread count (not the block shape), TSX, TT, rows per iteration
        (loop_unroll_factor_t 1 vs > 1; kind 2 always streams one row),
        sh_power, the ring depth and the remainder level count.  TSY only
        sets the launch geometry.  Configurations equal in these share one
        cubin through the compile cache: the 105,412-point space needs 5,762
        compilations (tests/test_hotspot_geometry.py), while every
        configuration is still launched and timed with its own geometry.
        """
        geo = self.stream_geometry(cfg) or {}
        kind = geo.get("kind", 0)
        rem = self.iterations % cfg["temporal_tiling_factor"]
        if kind:
            unroll = 1 if kind == 2 else min(cfg["loop_unroll_factor_t"], 2)
            return dict(HS_THREADS=cfg["block_size_x"] * cfg["block_size_y"], TSX=cfg["tile_size_x"],
                        TT=cfg["temporal_tiling_factor"], UNROLL=unroll, SH_POWER=cfg["sh_power"],
                        HS_STREAM=kind, HS_REM=rem, HS_NR=geo["nr"],
                        HS_PD=geo["pd"] if cfg["sh_power"] else 0)  # no power ring: PD unused
        return dict(BSX=cfg["block_size_x"], BSY=cfg["block_size_y"], TSX=cfg["tile_size_x"],
                    TSY=cfg["tile_size_y"], TT=cfg["temporal_tiling_factor"],
                    UNROLL=cfg["loop_unroll_factor_t"], SH_POWER=cfg["sh_power"],
                    HS_STREAM=0, HS_REM=rem, HS_NR=8)

    # -- stream mode (kernels/hotspot.cu, HS_STREAM) --------------------------
    # cp.async input ring depth (rows) and power prefetch distance, measured
    # on B200 (tools/gpu/hs_exp.sh, profiles/round2/hs_ring/):
    # * register rings: 8 input rows (3 row pairs in flight), power rows 6
    #   ahead (4 at T >= 9, 4 for one row per iteration): with the power
    #   ring decoupled from the input ring (16 + 7 mirror rows instead of
    #   32) 8 rows beat 16 by 3-14% on the T = 5-10 front (best 0.1587 ->
    #   0.1448 ms);
    # * shared-memory rings (kind 2): 4 rows -- the smaller input (and
    #   power) ring raises occupancy; 1.16x geomean over 16 rows on a
    #   24-configuration sample.
    # TSG_HS_NR / TSG_HS_PD force one value for experiments
    STREAM_NR_ENV = os.environ.get("TSG_HS_NR")

    def stream_nr(self, t: int, kind: int = 1, unroll: int = 2) -> int:
        if self.STREAM_NR_ENV:
            return int(self.STREAM_NR_ENV)
        return 4 if kind == 2 else 8

    STREAM_PD_ENV = os.environ.get("TSG_HS_PD")

    def stream_pd(self, t: int, kind: int, unroll: int, nr: int) -> int:
        """Power-row prefetch distance (rows ahead of level 1's first use)."""
        if self.STREAM_PD_ENV:
            pd = int(self.STREAM_PD_ENV)
        else:
            # the power ring holds pow2(TT + PD + 2) rows: keep it at 16
            # for every TT <= 10 (PD 6 -> 4 at TT 9, 10)
            pd = min(nr - 2, 6 if unroll > 1 else 4, 14 - t)
        rpi = 1 if kind == 2 or unroll == 1 else 2
        pd = max(rpi, min(pd, nr - 2))
        return pd - (pd % 2) if rpi == 2 else pd

    STREAM_SMEM_MAX = 200 * 1024
    STREAM_REG_BASE = 48     # addresses, masks, coefficients, temporaries

    def stream_geometry(self, cfg: dict, blocks_per_sm: int | None = None,
                        n_sm: int = 148) -> dict | None:
        """Warp-streaming geometry, or None when the config does not fit it.

        Mirrors the SW/TA/UW/WARP_FLOATS macros of kernels/hotspot.cu:
        register estimate 3*TT*TSX (level rings) + 4*TSX + 2*TT (hoisted
        shuffles) must fit the __launch_bounds__ budget, per-block smem the
        200 KiB cap.  Row segments: TSY whole waves of warp tiles, one wave
        = (resident blocks per SM x warps per block x SMs) tiles; the
        resident count comes from the driver's occupancy query at launch
        (``blocks_per_sm``), else from the register estimate.
        """
        bx, by = cfg["block_size_x"], cfg["block_size_y"]
        tsx, tsy = cfg["tile_size_x"], cfg["tile_size_y"]
        t, shp = cfg["temporal_tiling_factor"], cfg["sh_power"]
        nthreads = bx * by
        if self.W % 4 or nthreads % 32:
            return None
        budget = min(255, 65536 // nthreads)
        # fitted to ptxas counts of the static-depth kernel (tools/hs_regs.py):
        # ~3.5 registers per (level x column), odd TSX pays a scalar tail
        regs = math.ceil(3.5 * t * tsx) + self.STREAM_REG_BASE + (12 * t if tsx % 2 else 0)
        kind = 1  # level rings in registers
        if regs > budget:
            # level rings in shared memory (HS_STREAM=2): ~5 rows of TSX live
            kind = 2
            # with >= 128 registers per thread it beats the block-tile modes
            # even where ptxas spills (measured: 5.6 -> 1.3 ms at TSX=T=10)
            if self._smem_ring_regs(t, tsx) > budget and budget < 128:
                return None
        sw = 32 * tsx
        ta = (t + 3) & ~3
        uw = ((sw - ta - t) // 4) * 4
        if uw < 4:
            return None
        nr = self.stream_nr(t, kind, cfg["loop_unroll_factor_t"])
        pd = self.stream_pd(t, kind, cfg["loop_unroll_factor_t"], nr)
        need = t + pd + 2  # power ring rows (kernels/hotspot.cu PR)
        pr = (8 if need <= 8 else 16 if need <= 16 else 32 if need <= 32 else 64) if shp else 0
        wpb = nthreads // 32
        warp_floats = sw * (nr + pr + (t - 1 if shp else 0) + (3 * t if kind == 2 else 0))  # + power mirror rows
        smem = 4 * wpb * warp_floats
        if smem > self.STREAM_SMEM_MAX:
            return None
        nstrips = -(-self.W // uw)
        if blocks_per_sm is None:  # estimate (CPU-side planning / tests)
            used = min(regs, budget) if kind == 1 else self._smem_ring_regs(t, tsx)
            per_warp = -(-used * 32 // 256) * 256
            by_regs = 65536 // per_warp // wpb
            by_smem = (228 * 1024) // (smem + 1024) if smem else 32
            blocks_per_sm = max(1, min(by_regs, by_smem, 32, 64 // wpb))
        # border strips (kernels/hotspot.cu XL/XR): a prefix and a suffix
        # whose windows touch the grid edge; they run the all-selects code
        xl = min(ta // uw + 1, nstrips)
        xr_raw = 0 if self.W - 1 - sw + ta < 0 else (self.W - 1 - sw + ta) // uw + 1
        xr = min(max(xr_raw, xl), nstrips)
        nxe, nxi = xl + nstrips - xr, xr - xl
        warps = tsy * blocks_per_sm * wpb * n_sm  # TSY whole waves of warp tiles
        cap = self.H // max(8, 2 * t)
        f = self.STREAM_XEDGE_F or (1.5 if t <= 8 else 1.3)
        if nxi:
            ni = max(1, min(int(warps // (nxi + nxe * f)), cap))
            ne = max(1, min(math.ceil(ni * f), cap))
        else:
            ni, ne = 1, max(1, min(warps // nxe, cap))
        segh, segh0, ni = self._segments(ni)
        seghe, segh0e, ne = self._segments(ne)
        tiles = nxi * ni + nxe * ne
        return dict(sw=sw, ta=ta, uw=uw, segh=segh, segh0=segh0, nsegs=ni, seghe=seghe, segh0e=segh0e,
                    nsegse=ne, nxe=nxe, nxi=nxi, wpb=wpb, smem=smem, nstrips=nstrips,
                    blocks=-(-tiles // wpb), blocks_per_sm=blocks_per_sm, kind=kind, nr=nr, pd=pd)

    def _smem_ring_regs(self, t: int, tsx: int) -> int:
        """Register estimate of the smem-ring stream kernel (ptxas hoists
        level loads across the unrolled level loop; conservative fit)."""
        return 2 * t * tsx + 4 * tsx + self.STREAM_REG_BASE + 8

    # top/bottom segment height relative to the others (measured optimum on B200;
    # TSG_HS_EDGE_SEG overrides it for experiments)
    STREAM_EDGE_SEG = float(os.environ.get("TSG_HS_EDGE_SEG", "0.25"))
    # border strips run the all-selects code (~1.6x the interior's
    # instructions per row, SASS loop bodies): they get this many times the
    # interior strips' segment count -- 1.5 for T <= 8 (the faster
    # four-iteration interior loop), 1.3 above (measured,
    # profiles/round2/hs_ring/hs_exp_xe2.jsonl); TSG_HS_XEDGE_F overrides
    STREAM_XEDGE_F = float(os.environ.get("TSG_HS_XEDGE_F", "0"))
    # programmatic dependent launch between the launches of one run
    # (TSG_HS_PDL=0 disables it for experiments)
    STREAM_PDL = os.environ.get("TSG_HS_PDL", "1") != "0"
    # experiments: cap the warps per SM the segment geometry assumes
    STREAM_WARPS_CAP = int(os.environ.get("TSG_HS_WARPS_CAP", "0"))

    def _segments(self, nsegs: int) -> tuple:
        """(segh, segh0, nsegs): interior and first segment heights, segment count.

        The first and last segments are ~STREAM_EDGE_SEG of the others:
        their warps pay the N/S boundary selects, and in a single wave the
        slowest warp sets the launch time.  Rows: segh0 + (nsegs-2)*segh +
        last = H with 0 < last <= segh.
        """
        if nsegs == 1:
            return self.H, self.H, 1
        f = self.STREAM_EDGE_SEG
        segh = max(1, int(self.H // (nsegs - 2 + 2 * f)))
        while self.H - (nsegs - 2) * segh > 2 * segh:  # edge segments must not exceed segh
            segh += 1
        rest = self.H - (nsegs - 2) * segh  # split over the first and last segment
        segh0 = rest // 2
        if segh0 < 1 or rest - segh0 < 1:  # too many segments for H: no edge shortening
            segh = -(-self.H // nsegs)
            return segh, segh, -(-self.H // segh)
        return segh, segh0, nsegs

    def kernel_mode(self, cfg: dict) -> tuple:
        """(mode, floats per buffer, guard floats, buffers) -- mirrors kernels/hotspot.cu macros."""
        geo = self.stream_geometry(cfg)
        if geo is not None:
            return ("stream" if geo["kind"] == 1 else "stream_smem"), 0, 0, 0
        bx, by = cfg["block_size_x"], cfg["block_size_y"]
        t, shp = cfg["temporal_tiling_factor"], cfg["sh_power"]
        ew = bx * cfg["tile_size_x"] + 2 * t
        eh = by * cfg["tile_size_y"] + 2 * t
        ry = -(-eh // by)
        budget = min(255, 65536 // (bx * by))
        cxp = -(-ew // (2 * bx))
        pairs_max = min(16, (budget - 40) // (4 + 2 * shp))
        sp = 2 * cxp * bx
        skew = 0 if 2 * bx >= 32 else (2 * bx - (ry * sp) % (4 * bx)) % (4 * bx)
        ss = ry * sp + skew
        guard = sp + 34
        reg_bytes = 4 * (2 * by * ss + 3 * guard)
        if cxp * ry <= pairs_max and reg_bytes <= 200 * 1024:
            return "register", by * ss, guard, 2  # power lives in registers
        skew_s = 0 if bx >= 32 else (bx - (ry * ew) % (2 * bx)) % (2 * bx)
        return "shared", by * (ry * ew + skew_s), ew + 1, 2 + shp

    def smem_bytes(self, cfg: dict) -> int:
        # window buffers (the space's own smem model is (2 + sh_power) x
        # window, ts/spaces/hotspot.spec:25; we pad/skew them and add three
        # guard bands -- register mode keeps power in registers)
        geo = self.stream_geometry(cfg)
        if geo is not None:
            return geo["smem"]
        _, buf, guard, nbuf = self.kernel_mode(cfg)
        return 4 * (nbuf * buf + 3 * guard)

    def step_plan(self, t: int) -> list:
        n = math.ceil(self.iterations / t)
        return [t] * (n - 1) + [self.iterations - t * (n - 1)]

    @staticmethod
    def tuned_coefficients(k: dict) -> dict:
        """The tuned kernels' folded coefficients (kernels/hotspot.cu header).

        T' = ax*(E+W) + ay*(N+S) + at*T + c,  c = ap*P + ac -- the Rodinia
        update T + sdc*(P + ry1*(N+S-2T) + rx1*(E+W-2T) + rz1*(amb-T))
        expanded; derived in float64 from the fp32 Rodinia coefficients,
        then rounded once to fp32.
        """
        sdc, rx1, ry1, rz1, amb = (float(k[n]) for n in ("sdc", "rx1", "ry1", "rz1", "amb"))
        f32 = lambda v: float(np.float32(v))  # noqa: E731
        return dict(at=f32(1.0 - sdc * (2.0 * rx1 + 2.0 * ry1 + rz1)), ay=f32(sdc * ry1),
                    ax=f32(sdc * rx1), ap=f32(sdc), ac=f32(sdc * rz1 * amb))

    def _coeff_args(self):
        c = self.tuned_coefficients(self.k)
        return [C.c_float(c[n]) for n in ("at", "ay", "ax", "ap", "ac")]

    def _rodinia_args(self):
        k = self.k
        return [C.c_float(k[n]) for n in ("sdc", "rx1", "ry1", "rz1", "amb")]

    def _chain(self, kernel, bufs, n_launch, make):
        """Buffers for a ping-pong chain ending in bufs['out']."""
        seq = []
        src = bufs["temp"]
        for i in range(n_launch):
            dst = bufs["out"] if (n_launch - 1 - i) % 2 == 0 else bufs["tmp"]
            seq.append(make(i, src, dst))
            src = dst
        return seq

    def launch_shape(self, cfg: dict, kernel) -> tuple:
        """(grid, block, smem, extra args) of one launch of this configuration.

        Stream mode sizes its row segments from the kernel's occupancy
        (driver query through ``kernel.occupancy``) so the grid is whole
        waves; block-tile modes use the paper's ceil(problem / tile) grid.
        """
        block = (cfg["block_size_x"], cfg["block_size_y"], 1)
        geo = self.stream_geometry(cfg)
        if geo is not None:
            occ = getattr(kernel, "occupancy", None)
            if occ is not None:
                bps = occ(cfg["block_size_x"] * cfg["block_size_y"], geo["smem"])
                if self.STREAM_WARPS_CAP:  # experiments: fewer, taller segments
                    bps = min(bps, max(1, self.STREAM_WARPS_CAP // geo["wpb"]))
                geo = self.stream_geometry(cfg, blocks_per_sm=max(1, bps), n_sm=kernel.sm_count)
            return (geo["blocks"], 1, 1), block, geo["smem"], [
                C.c_int(geo[k]) for k in ("segh", "nsegs", "segh0", "seghe", "nsegse", "segh0e")]
        ow = cfg["block_size_x"] * cfg["tile_size_x"]
        oh = cfg["block_size_y"] * cfg["tile_size_y"]
        return (math.ceil(self.W / ow), math.ceil(self.H / oh), 1), block, self.smem_bytes(cfg), []

    def launch(self, cfg: dict, kernel, dst: int, src: int, power: int, nsteps: int, shape=None,
               pdl: bool = False):
        """One launch advancing ``src`` by ``nsteps`` into ``dst`` (raw device addresses).

        Stream mode: the remainder launch (nsteps = iterations % T) runs the
        module's ``hotspot_rem_kernel`` (static level count HS_REM).
        """
        from .runtime import Launch

        grid, block, smem, extra = shape or self.launch_shape(cfg, kernel)
        if extra and nsteps != cfg["temporal_tiling_factor"]:
            assert nsteps == self.iterations % cfg["temporal_tiling_factor"], nsteps
            kernel = self._rem_kernel(kernel, smem)
        return Launch(kernel, grid, block, [C.c_uint64(int(dst)), C.c_uint64(int(src)), C.c_uint64(int(power)),
                                            C.c_int(nsteps)] + self._coeff_args() + extra, smem=smem,
                      pdl=bool(extra) and pdl and self.STREAM_PDL)

    @staticmethod
    def _rem_kernel(kernel, smem: int):
        if kernel is None:  # host-side planning (tests): no module
            return None
        rem = getattr(kernel, "_hs_rem", None)
        if rem is None:
            rem = kernel.module.function("hotspot_rem_kernel")
            if smem > 48 * 1024:
                rem.set_max_dynamic_smem(smem)
            if smem > 0:
                rem.set_smem_carveout(100)
            kernel._hs_rem = rem
        return rem

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        plan = self.step_plan(cfg["temporal_tiling_factor"])
        shape = self.launch_shape(cfg, kernel)
        # launches 2..n of a run: programmatic dependent launch (stream
        # kernels wait on griddepcontrol before reading the previous output)
        return self._chain(kernel, bufs, len(plan), lambda i, s, d: self.launch(
            cfg, kernel, d.ptr, s.ptr, bufs["power"].ptr, plan[i], shape, pdl=i > 0))

    def reference_launches(self, kernel, bufs: dict) -> list:
        from .runtime import Launch

        grid = (math.ceil(self.W / 32), math.ceil(self.H / 8), 1)
        return self._chain(kernel, bufs, self.iterations, lambda i, s, d: Launch(
            kernel, grid, (256, 1, 1), [_u64(d), _u64(s), _u64(bufs["power"])]
            + self._rodinia_args()))

    def flops(self, cfg=None) -> float:
        return float(self.FLOP_PER_CELL) * self.W * self.H * self.iterations

    def compulsory_bytes(self, cfg=None) -> float:
        t = cfg["temporal_tiling_factor"] if cfg else 1
        return 12.0 * self.W * self.H * len(self.step_plan(t))

    def describe(self) -> dict:
        return {"grid": f"{self.W}x{self.H}", "iterations": self.iterations, "dtype": "fp32"}


# =============================================================================
# Dedispersion


K_DM = 4148.808  # s MHz^2 pc^-1 cm^3


def dd_asm_dispatch(tsx: int, tsy: int, span: int) -> str:
    """Inline-PTX jump-table dispatch of the window dedispersion kernel.

    One case per increment pattern P with popcount <= ``span``, in the same
    dense order as the kernel's ``dd_rank`` (span-major, then value).  A
    case loads the popc(P)+1 window samples of every owned sample pair from
    the staged row (shared memory) and adds them to the TSY x TSX/2 packed
    accumulators (``add.rn.f32x2``, per lane identical to the C++ cases);
    ``brx.idx`` makes ptxas emit an indexed jump (BRX) instead of the
    compare tree a C++ switch is lowered to.
    """
    assert tsx % 2 == 0
    xp = tsx // 2
    pats = sorted((p for p in range(1 << (tsy - 1)) if bin(p).count("1") <= span),
                  key=lambda p: (bin(p).count("1"), p))
    nacc = tsy * xp

    def section(tag: str, idx_op: int, addr_op: int) -> list:
        body = [f"ts{tag}_%=: .branchtargets " + ", ".join(f"L{tag}{i}_%=" for i in range(len(pats))) + ";",
                f"brx.idx.uni %{idx_op}, ts{tag}_%=;"]
        for i, p in enumerate(pats):
            body.append(f"L{tag}{i}_%=:")
            ps = bin(p).count("1")
            for q in range(xp):
                for k in range(ps + 1):
                    body.append(f" ld.shared.f32 lo, [%{addr_op}+{4 * (64 * q + k)}];")
                    body.append(f" ld.shared.f32 hi, [%{addr_op}+{4 * (64 * q + 32 + k)}];")
                    body.append(f" mov.b64 w{q}_{k}, {{lo, hi}};")
            for j in range(tsy):
                g = bin(p & ((1 << j) - 1)).count("1")
                for q in range(xp):
                    a = j * xp + q
                    body.append(f" add.rn.f32x2 %{a}, %{a}, w{q}_{g};")
            if i != len(pats) - 1:
                body.append(f" bra.uni D{tag}_%=;")
        body.append(f"D{tag}_%=:")
        return body

    head = ["{", ".reg .f32 lo, hi;"] + [f".reg .b64 w{q}_{k};" for q in range(xp) for k in range(span + 1)]
    outs = ", ".join(f'"+l"(acc[{j}][{q}])' for j in range(tsy) for q in range(xp))
    one = "\\n".join(head + section("a", nacc, nacc + 1) + ["}"])  # C string escapes: one PTX statement per line
    # two channels (in order) per asm block: the loop trip and the
    # convergence region are paid once per pair (four per block: slower)
    two = "\\n".join(head + section("a", nacc, nacc + 1) + section("b", nacc + 2, nacc + 3) + ["}"])
    return (
        "#define DD_HAVE_ASM 1\n"
        "__device__ __forceinline__ void dd_asm_dispatch(unsigned long long (&acc)[TSY][XP], int idx, unsigned saddr) {\n"
        # volatile keeps it ordered after the (volatile) mbarrier wait; no
        # "memory" clobber, so the compiler may overlap the next channel's
        # decode with the adds
        f'  asm volatile("{one}" : {outs} : "r"(idx), "r"(saddr));\n'
        "}\n"
        "__device__ __forceinline__ void dd_asm_dispatch2(unsigned long long (&acc)[TSY][XP], int idx0, unsigned saddr0,"
        " int idx1, unsigned saddr1) {\n"
        f'  asm volatile("{two}" : {outs} : "r"(idx0), "r"(saddr0), "r"(idx1), "r"(saddr1));\n'
        "}\n")


def dm_delay_table(nch: int, f_min_mhz: float, ch_bw_mhz: float, t_samp_s: float) -> np.ndarray:
    """Per-channel delay in samples per unit DM (fp32), channel 0 = lowest.

    delay[ch] = K_DM * (f_ch^-2 - f_max^-2) / t_samp, f_ch = f_min + ch*bw.
    Constants are unpinned by the reference; DESIGN.md fixes
    an L-band LOFAR/Apertif-like setup.
    """
    f = f_min_mhz + ch_bw_mhz * np.arange(nch, dtype=np.float64)
    fmax = f[-1]
    return (K_DM * (f ** -2 - fmax ** -2) / t_samp_s).astype(np.float32)


def dm_shifts(delay: np.ndarray, ndm: int, dm_first: float, dm_step: float) -> np.ndarray:
    """int32 [ndm][nch] shifts with the kernel's exact fp32 rounding."""
    d = np.arange(ndm, dtype=np.float32)
    dmv = (np.float32(dm_first) + d * np.float32(dm_step)).astype(np.float32)
    prod = (dmv[:, None] * delay[None, :]).astype(np.float32)
    return np.trunc(prod).astype(np.int32)


class Dedispersion(Problem):
    """out[dm][s] = sum_ch in[ch][s + shift(dm, ch)].

    HBM layout: input fp32 [NCH][IN_PITCH] with IN_PITCH = round_up(NSAMP
    + max_shift + 128, 32) (zero tail: grid overshoot reads stay in the
    row), output fp32 [NDM][NSAMP].  Inputs U[0,1) (seed 5).
    """

    space_name = "dedispersion"
    source_file = "dedispersion.cu"
    kernel_name = "dedispersion_kernel"
    reference_kernel = "dedispersion_reference"
    rtol = 1e-5

    def __init__(self, channels: int = 1536, samples: int = 25000, dms: int = 2048,
                 f_min_mhz: float = 1425.0, ch_bw_mhz: float = 0.1953125,
                 t_samp_s: float = 40.96e-6, dm_first: float = 0.0, dm_step: float = 0.02,
                 seed: int = 5):
        super().__init__()
        self.NCH, self.NSAMP, self.NDM = channels, samples, dms
        self.dm_first, self.dm_step = float(np.float32(dm_first)), float(np.float32(dm_step))
        self.delay = dm_delay_table(channels, f_min_mhz, ch_bw_mhz, t_samp_s)
        self.max_shift = int(dm_shifts(self.delay, dms, self.dm_first, self.dm_step).max())
        self.in_w = samples + self.max_shift
        # slack: grid-overshoot reads of the generic kernel (128) and the
        # staged row segments of the window / staged generic kernels: a block
        # row starts at (first sample + its first DM's shift) & ~3 and spans
        # <= 128 samples + the block's DM spread (<= max_shift) + 8
        self.pitch = ((samples + self.max_shift + max(640, self.max_shift + 160) + 31) // 32) * 32
        self.seed = seed

    def data(self) -> np.ndarray:
        return np.random.default_rng(self.seed).random((self.NCH, self.in_w), dtype=np.float32)

    def host_buffers(self) -> list:
        padded = np.zeros((self.NCH, self.pitch), dtype=np.float32)
        padded[:, : self.in_w] = self.data()
        return [BufferSpec("in", padded.nbytes, padded), BufferSpec("out", self.NDM * self.NSAMP * 4)]

    def constants(self) -> dict:
        return {"d_delay": self.delay}

    @property
    def output_count(self) -> int:
        return self.NDM * self.NSAMP

    def problem_defines(self) -> dict:
        return dict(NCH=self.NCH, NSAMP=self.NSAMP, NDM=self.NDM, IN_PITCH=self.pitch)

    def config_defines(self, cfg: dict) -> dict:
        d = dict(BSX=cfg["block_size_x"], BSY=cfg["block_size_y"], TSX=cfg["tile_size_x"],
                 TSY=cfg["tile_size_y"], STX=cfg["tile_stride_x"], STY=cfg["tile_stride_y"])
        span = self.window_span(cfg)
        if span is not None:
            d.update(DD_WIN=1, SPAN=span, BLKSPAN=self.block_span(cfg))
        else:
            ns = self.staged_stages(cfg)
            if ns:
                d.update(DD_STG=1, DD_NSTAGE=ns, BLKSPAN=self.block_span(cfg))
        return d

    DD_ASM_MARKER = "// @DD_ASM_DISPATCH@"

    def source_for(self, cfg: dict | None, base: str | None = None) -> str:
        """Window-mode configurations where it pays get a generated
        jump-table dispatch (``dd_asm_dispatch``, kernels/dedispersion.cu)."""
        src = base if base is not None else self.source()
        if cfg is None:
            return src
        span = self.window_span(cfg)
        if span is None or not self.use_asm_dispatch(cfg["tile_size_x"], cfg["tile_size_y"], span):
            return src
        return src.replace(self.DD_ASM_MARKER, dd_asm_dispatch(cfg["tile_size_x"], cfg["tile_size_y"], span))

    @staticmethod
    def use_asm_dispatch(tsx: int, tsy: int, span: int) -> bool:
        """Jump table only where it pays (measured on B200): a deep compare
        tree (>= 32 live patterns) AND >= 16 packed adds per case -- with
        less work per case the indirect branch's bubble costs more than the
        few compares it replaces (e.g. (2,8): 6.3 -> 8.1 ms, (4,8): 4.88 ->
        4.70 ms)."""
        npat = sum(1 for p in range(1 << (tsy - 1)) if bin(p).count("1") <= span)
        return tsx % 2 == 0 and npat >= 32 and tsy * (tsx // 2) >= 16

    DD_STAGES = 5  # kernels/dedispersion.cu NSTAGE
    DD_CC = 32     # channels per stage

    def block_span(self, cfg: dict) -> int:
        """Max shift spread over one block's BSY*TSY DMs (window kernel BLKSPAN)."""
        nd = cfg["block_size_y"] * cfg["tile_size_y"]
        key = ("blk", nd, self.NCH, self.NDM, self.dm_first, self.dm_step)
        if key not in Dedispersion._spans:
            sh = dm_shifts(self.delay, self.NDM, self.dm_first, self.dm_step).astype(np.int64)
            first = np.arange(0, self.NDM, nd)
            last = np.minimum(first + nd - 1, self.NDM - 1)
            Dedispersion._spans[key] = int((sh[last] - sh[first]).max())
        return Dedispersion._spans[key]

    def smem_bytes(self, cfg: dict) -> int:
        span = self.window_span(cfg)
        if span is None:
            ns = self.staged_stages(cfg)
            return self._staged_smem(cfg, ns) if ns else 0
        rowlen = (32 * cfg["tile_size_x"] + self.block_span(cfg) + span + 4 + 3) & ~3
        npat = 1 << (cfg["tile_size_y"] - 1)
        return 4 * self.DD_STAGES * self.DD_CC * rowlen + 16 * self.DD_STAGES + 4 * self.NCH + npat

    # staged generic mode (kernels/dedispersion.cu DD_STG) for non-window
    # configurations with enough work per staged row: >= 4 threads and >= 12
    # samples per block row, >= 8 outputs per thread.  Measured on B200
    # (46-configuration A/B, profiles/round1/dd_staged_ab.md): those run
    # 1.0-2.0x faster staged; narrower blocks (1-2 threads in x, few
    # samples per block) re-stage nearly the same DM-spread rows per handful
    # of outputs and run up to 4x slower, so they keep the plain kernel.
    # TSG_DD_STG=0 forces the plain kernel everywhere, =all staged wherever
    # it fits (A/B measurements).
    STAGED_ENV = "TSG_DD_STG"
    STAGED_SMEM_MAX = 200 * 1024

    def _staged_smem(self, cfg: dict, ns: int) -> int:
        rowlen = (cfg["block_size_x"] * cfg["tile_size_x"] + self.block_span(cfg) + 4 + 3) & ~3
        return 4 * ns * self.DD_CC * rowlen + 16 * ns + 4 * self.NCH

    def staged_stages(self, cfg: dict) -> int:
        """Ring depth of the staged generic kernel (largest <= 5 that fits), 0 = plain kernel."""
        mode = os.environ.get(self.STAGED_ENV, "1")
        if mode == "0":
            return 0
        if mode != "all" and not (cfg["block_size_x"] >= 4 and cfg["block_size_x"] * cfg["tile_size_x"] >= 12
                                  and cfg["tile_size_x"] * cfg["tile_size_y"] >= 8):
            return 0
        for ns in range(self.DD_STAGES, 1, -1):
            if self._staged_smem(cfg, ns) <= self.STAGED_SMEM_MAX:
                return ns
        return 0

    _spans: dict = {}

    def _group_span(self, tsy: int) -> tuple:
        """(max increment between adjacent DMs, max shift span of a TSY-DM group)."""
        key = (tsy, self.NCH, self.NDM, self.dm_first, self.dm_step)
        if key not in Dedispersion._spans:
            sh = dm_shifts(self.delay, self.NDM, self.dm_first, self.dm_step).astype(np.int64)
            n = -(-self.NDM // tsy) * tsy
            idx = np.minimum(np.arange(n), self.NDM - 1)  # overshoot rows use the last DM (kernel clamp)
            g = sh[idx].reshape(-1, tsy, self.NCH)
            inc = int(np.diff(g, axis=1).max()) if tsy > 1 else 0
            Dedispersion._spans[key] = (inc, int((g[:, -1, :] - g[:, 0, :]).max()))
        return Dedispersion._spans[key]

    def window_span(self, cfg: dict) -> int | None:
        """SPAN of the register-window kernel (kernels/dedispersion.cu DD_WIN), or None.

        Eligible: block_size_x == 32 (a warp's lanes share their DMs, so the
        shifts are warp-uniform), strided samples (or one per lane),
        contiguous DMs (or one per lane), adjacent DMs shifting by <= 1
        sample, and a window of <= 4 samples.
        """
        if cfg["block_size_x"] != 32:
            return None
        if cfg["tile_size_x"] > 1 and cfg["tile_stride_x"] != 1:
            return None
        if cfg["tile_size_y"] > 1 and cfg["tile_stride_y"] != 0:
            return None
        inc, span = self._group_span(cfg["tile_size_y"])
        if inc > 1 or span > 3:
            return None
        return span

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        from .runtime import Launch

        # x = DM tiles (fastest varying: L2 reuse of the input), y = sample tiles
        grid = (math.ceil(self.NDM / (cfg["block_size_y"] * cfg["tile_size_y"])),
                math.ceil(self.NSAMP / (cfg["block_size_x"] * cfg["tile_size_x"])), 1)
        return [Launch(kernel, grid, (cfg["block_size_x"], cfg["block_size_y"], 1),
                       [_u64(bufs["out"]), _u64(bufs["in"]), C.c_float(self.dm_first),
                        C.c_float(self.dm_step)], smem=self.smem_bytes(cfg))]

    def reference_launches(self, kernel, bufs: dict) -> list:
        from .runtime import Launch

        return [Launch(kernel, (math.ceil(self.NSAMP / 256), self.NDM, 1), (256, 1, 1),
                       [_u64(bufs["out"]), _u64(bufs["in"]), C.c_float(self.dm_first),
                        C.c_float(self.dm_step)])]

    def adds(self) -> float:
        return float(self.NDM) * self.NSAMP * self.NCH

    def flops(self, cfg=None) -> float:
        return self.adds()

    def compulsory_bytes(self, cfg=None) -> float:
        return 4.0 * (self.NCH * self.in_w + self.NDM * self.NSAMP)

    def paper_bytes(self) -> float:
        """Bytes the kernel *loads* (one fp32 per add): the paper's GB/s basis."""
        return 4.0 * self.adds()

    def describe(self) -> dict:
        return {"channels": self.NCH, "samples": self.NSAMP, "dms": self.NDM,
                "max_shift": self.max_shift, "dtype": "fp32"}


# =============================================================================
# GEMM (CLBlast xgemm space)


class Gemm(Problem):
    """c(m,n) = sum_k a(m,k) b(k,n), BLAS column-major with A transposed:
    a(m,k) = A[k*M+m], b(k,n) = B[k*N+n], c(m,n) = C[n*M+m]
    (SURVEY 8a a19 leaves layout unpinned; this is CLBlast's xgemm view).
    Inputs U[-1,1) (seeds 6, 7).
    """

    space_name = "gemm"
    source_file = "gemm.cu"
    kernel_name = "gemm_kernel"
    reference_kernel = "gemm_reference"

    def config_defines(self, cfg: dict) -> dict:
        """All 13 tunables as macros, except that the load re-shape of an
        operand that is NOT staged in shared memory (MDIMA when SA = 0, NDIMB
        when SB = 0) never reaches the code: those configurations share one
        cubin through the compile cache (116,928 configurations -> 61,672
        compilations); each is still launched and timed on its own."""
        d = {k.upper(): int(v) for k, v in cfg.items()}
        if not d["SA"]:
            d["MDIMA"] = d["MDIMC"]
        if not d["SB"]:
            d["NDIMB"] = d["NDIMC"]
        return d

    def __init__(self, m: int = 4096, n: int = 4096, k: int = 4096, seed_a: int = 6,
                 seed_b: int = 7):
        super().__init__()
        self.M, self.N, self.K = m, n, k
        self.seed_a, self.seed_b = seed_a, seed_b
        # identical fmaf chains everywhere -> bit-exact; keep a K-scaled
        # bound for callers that compare against other orders
        self.rtol = 1e-5

    def a(self) -> np.ndarray:
        r = np.random.default_rng(self.seed_a)
        return (r.random((self.K, self.M), dtype=np.float32) * np.float32(2) - np.float32(1))

    def b(self) -> np.ndarray:
        r = np.random.default_rng(self.seed_b)
        return (r.random((self.K, self.N), dtype=np.float32) * np.float32(2) - np.float32(1))

    def host_buffers(self) -> list:
        return [BufferSpec("A", self.K * self.M * 4, self.a()),
                BufferSpec("B", self.K * self.N * 4, self.b()),
                BufferSpec("out", self.M * self.N * 4)]

    @property
    def output_count(self) -> int:
        return self.M * self.N

    def problem_defines(self) -> dict:
        return dict(GM=self.M, GN=self.N, GK=self.K, GEMM_NS=self.GEMM_NS)

    def smem_bytes(self, cfg: dict) -> int:
        # GEMM_NS-deep cp.async ring of staged k-tiles (kernels/gemm.cu)
        return 4 * self.GEMM_NS * cfg["KWG"] * (cfg["MWG"] * cfg["SA"] + cfg["NWG"] * cfg["SB"])

    GEMM_NS = int(os.environ.get("TSG_GEMM_NS", "3"))

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        from .runtime import Launch

        grid = (self.M // cfg["MWG"], self.N // cfg["NWG"], 1)
        return [Launch(kernel, grid, (cfg["MDIMC"] * cfg["NDIMC"], 1, 1),
                       [_u64(bufs["out"]), _u64(bufs["A"]), _u64(bufs["B"])], smem=self.smem_bytes(cfg))]

    def reference_launches(self, kernel, bufs: dict) -> list:
        from .runtime import Launch

        return [Launch(kernel, (math.ceil(self.M / 64), math.ceil(self.N / 4), 1), (256, 1, 1),
                       [_u64(bufs["out"]), _u64(bufs["A"]), _u64(bufs["B"])])]

    def flops(self, cfg=None) -> float:
        return 2.0 * self.M * self.N * self.K

    def compulsory_bytes(self, cfg=None) -> float:
        return 4.0 * (self.M * self.K + self.K * self.N + self.M * self.N)

    def describe(self) -> dict:
        return {"m": self.M, "n": self.N, "k": self.K, "dtype": "fp32"}


class GemmTC(Gemm):
    """The tf32 tcgen05/TMEM/TMA variant of :class:`Gemm` (same layout).

    Not part of the reference's GEMM space (north_star: "optional ...
    variant"), so it carries its own small space: the N extent of the
    UMMA tile (BN_T) and the smem pipeline depth (STAGES), restricted to
    B200's 227 KB of shared memory per CTA.  Verified against the fp32
    naive kernel with a K-scaled tf32 tolerance: max|dC| <= K * 2^-11 *
    max|a|*max|b| relative to max|C| (= 2/max|C| here, ~0.02).
    """

    space_name = "gemm_tc"
    source_file = "gemm_tc.cu"
    kernel_name = "gemm_tc_kernel"
    reference_kernel = "gemm_reference"

    def __init__(self, m: int = 4096, n: int = 4096, k: int = 4096, seed_a: int = 6, seed_b: int = 7,
                 max_units: int | None = None):
        from .paramspace import space_from_tune_params

        self.space = space_from_tune_params(
            "gemm_tc", {"BN_T": [128, 256], "STAGES": [2, 3, 4, 5, 6], "CLUSTER": [1, 2]},
            ["STAGES * (16384 + BN_T * 128 / CLUSTER) + 1280 <= 232448"],
            metric="(2 * 4096^3) / (time_ms * 1e6)")
        self._host = None
        self.M, self.N, self.K = m, n, k
        self.seed_a, self.seed_b = seed_a, seed_b
        self.max_units = max_units  # cap on the persistent grid (tests: several items per CTA)
        # K-scaled tf32 bound: |dC| <= c*K*eps*max|a|*max|b|, eps = 2^-11, c = 1
        self.abs_tol = self.K * 2.0 ** -11
        self.rtol = 1.0  # the norm-wise check is replaced by abs_tol

    def source(self) -> str:
        # the fp32 naive answer kernel comes from gemm.cu (tuned part compiled out)
        return _src("gemm_tc.cu") + "\n#undef REFERENCE_ONLY\n#define REFERENCE_ONLY 1\n" + _src("gemm.cu")

    def config_defines(self, cfg: dict) -> dict:
        return {"BN_T": cfg["BN_T"], "STAGES": cfg["STAGES"], "CLUSTER": cfg.get("CLUSTER", 1)}

    def host_buffers(self) -> list:
        a, b = self.a(), self.b()
        # CLBlast layout (for the fp32 answer kernel) + K-major copies (TMA/UMMA operands)
        return [BufferSpec("A", a.nbytes, a), BufferSpec("B", b.nbytes, b),
                BufferSpec("Ak", a.nbytes, np.ascontiguousarray(a.T)),
                BufferSpec("Bk", b.nbytes, np.ascontiguousarray(b.T)),
                BufferSpec("out", self.M * self.N * 4)]

    def smem_bytes(self, cfg: dict) -> int:
        # >= 116 KiB: one CTA per SM (a second CTA's 2 x BN_T TMEM columns
        # would wait for the first to finish anyway)
        return max(cfg["STAGES"] * (16384 + cfg["BN_T"] * 128 // cfg.get("CLUSTER", 1)) + 1024 + 256, 116 * 1024)

    def launches(self, cfg: dict, kernel, bufs: dict) -> list:
        from .runtime import Launch

        dev = bufs["Ak"].dev
        # K-major operands: dim0 = K (contiguous), dim1 = M / N; boxes of 32 K x (128 | BN_T)
        cluster = cfg.get("CLUSTER", 1)
        # 2-SM pair (cta_group::2): each CTA holds its own 128 A rows and half of the B tile
        ta = dev.tma_2d_f32(bufs["Ak"], self.K, self.M, self.K * 4, 32, 128, 128)
        tb = dev.tma_2d_f32(bufs["Bk"], self.K, self.N, self.K * 4, 32, cfg["BN_T"] // cluster, 128)
        tiles_m = self.M // 128
        tiles = tiles_m * (self.N // cfg["BN_T"])
        # persistent: one CTA (cluster == 1) or one 2-CTA cluster per SM
        # (pair); work units = whole tiles (pairs of M tiles for clusters)
        # while they fill whole waves of the persistent grid, then halves
        n_sm = int(dev.info.get("sm_count", 148))
        units = tiles // cluster
        n_units = min(n_sm // cluster, units, self.max_units or units)
        n_full = (units // n_units) * n_units
        items = n_full + 2 * (units - n_full)
        return [Launch(kernel, (n_units * cluster, 1, 1), (192, 1, 1),
                       [_u64(bufs["out"]), ta, tb, C.c_int(tiles_m), C.c_int(n_full), C.c_int(items)],
                       smem=self.smem_bytes(cfg), cluster=(cluster, 1, 1))]


PROBLEMS = {"convolution": Convolution, "hotspot": Hotspot, "dedispersion": Dedispersion,
            "gemm": Gemm, "gemm_tc": GemmTC}


def make_problem(name: str, **kw) -> Problem:
    try:
        cls = PROBLEMS[name]
    except KeyError:
        raise KeyError(f"unknown problem {name!r}; known: {sorted(PROBLEMS)}") from None
    return cls(**kw)
