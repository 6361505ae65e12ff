"""Domain-decomposed hotspot across the GPUs of one node (north_star N9).

The 16384^2 grid is split into P row slabs, one per rank.  Rank p stores
its H/P owned rows plus a halo of h = T rows on each side that has a
neighbour (none above rank 0, none below rank P-1).  The tuned kernel
(kernels/hotspot.cu) advances any block of consecutive rows as an
isolated grid: its clamped edge produces wrong values that travel at
most nsteps <= T rows inward.  That is what makes the schedule below
exact.

Per launch of k <= T steps (``run``):

1. *edge bands* -- the 3h stored rows at each internal slab edge (the
   halo plus 2h owned rows) are advanced into small band buffers.  Rows
   [h, 2h) of a band are exact: they are the h owned rows the neighbour
   needs next.
2. *interior* -- the owned rows alone are advanced as one grid into
   ``dst``.  All but the h rows next to an internal edge are exact.
3. *exchange* (not after the last launch) -- each band's exact rows go
   to the neighbour, whose receive lands in ``dst``'s halo rows.  NCCL
   point-to-point over NVLink via ``torch.distributed.batch_isend_irecv``.
   This is the only data-path collective of the build.  It runs on its
   own stream, so it overlaps step 2.
4. *patch* -- the exact band rows are copied over ``dst``'s h damaged
   owned rows at each internal edge.

Extra work per launch: 2 x 3h band rows against H/P owned rows, i.e. 3%
at 16384^2 on 8 GPUs with T = 8.

Ordering contract (CUDA path).  Kernels and copies run on libtsgpu's
context stream S.  torch.distributed's NCCL work runs on torch's current
stream C (and its internal NCCL stream, which ProcessGroupNCCL orders
after C at issue time; ``req.wait()`` orders C after it).  The two
streams are ordered explicitly through the C ABI:

* ``edges_done``: C waits for S once the edge bands are enqueued
  (``tsg_stream_signal``), so the sends read finished band rows;
* ``comm_done``: S waits for C before the next launch
  (``tsg_stream_wait``), so the next launch reads the received halos,
  and the band buffers are not overwritten while a send still reads them.

Nothing else crosses streams: the interior launch writes only owned rows,
the receives write only halo rows, the bands only band buffers.  Without
the two waits the next launch could read halo rows before they land.
``tests/test_dd_hotspot.py`` shows exactly that on one GPU, with a delayed
producer on another stream standing in for the receive.

The schedule is independent of the step function.  The same ``run``
drives (a) GPUs with the tuned kernel and NCCL (``CudaOps``) and (b) CPU
ranks under gloo with the C oracle as the step function (the tests).  The
gloo tests prove the decomposition bit-exact against the single-domain
run.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class Slab:
    rank: int
    world: int
    rows: int        # owned rows
    row0: int        # global index of the first owned row
    halo_top: int    # halo rows stored above (0 on rank 0)
    halo_bot: int    # halo rows stored below (0 on the last rank)

    @property
    def height(self) -> int:
        return self.halo_top + self.rows + self.halo_bot

    @property
    def first_stored_row(self) -> int:
        return self.row0 - self.halo_top

    @property
    def halo(self) -> int:
        return self.halo_top or self.halo_bot


def make_slab(rank: int, world: int, gh: int, halo: int) -> Slab:
    if gh % world:
        raise ValueError(f"grid height {gh} not divisible by {world} ranks")
    rows = gh // world
    if world > 1 and 2 * halo > rows:
        raise ValueError(f"slab of {rows} rows too thin for a {halo}-row halo (need >= {2 * halo})")
    return Slab(rank, world, rows, rank * rows, halo if rank > 0 else 0,
                halo if rank < world - 1 else 0)


def band_rows(slab: Slab) -> int:
    return 3 * slab.halo


def run(slab: Slab, temp, power, scratch_a, scratch_b, iterations: int, t: int, ops,
        band_top=None, band_bot=None):
    """Advance ``iterations`` steps in launches of <= t; returns the buffer holding the result.

    ``temp``/``power``/``scratch_*``: [height][W] row-indexable buffers (the
    initial slab INCLUDING valid halos).  ``band_*``: [3h][W] buffers, needed
    on the sides with a neighbour.  ``ops`` supplies the step function,
    copies, the exchange and the two ordering hooks (see the module doc).
    """
    n_launch = math.ceil(iterations / t)
    plan = [t] * (n_launch - 1) + [iterations - t * (n_launch - 1)]
    h, H, ht, rows = slab.halo, slab.height, slab.halo_top, slab.rows
    top, bot = slab.halo_top > 0, slab.halo_bot > 0
    src = temp
    for i, k in enumerate(plan):
        dst = scratch_a if i % 2 == 0 else scratch_b
        last = i == n_launch - 1
        if top:
            ops.advance(src[0:3 * h], band_top, power[0:3 * h], k)
        if bot:
            ops.advance(src[H - 3 * h:H], band_bot, power[H - 3 * h:H], k)
        if not last and (top or bot):
            ops.edges_done()
        ops.advance(src[ht:ht + rows], dst[ht:ht + rows], power[ht:ht + rows], k)
        if not last and (top or bot):
            sends, recvs = [], []
            if top:
                sends.append((band_top[h:2 * h], slab.rank - 1))
                recvs.append((dst[0:h], slab.rank - 1))
            if bot:
                sends.append((band_bot[h:2 * h], slab.rank + 1))
                recvs.append((dst[H - h:H], slab.rank + 1))
            ops.exchange(sends, recvs)
        if top:
            ops.copy(dst[ht:ht + h], band_top[h:2 * h])
        if bot:
            ops.copy(dst[ht + rows - h:ht + rows], band_bot[h:2 * h])
        if not last and (top or bot):
            ops.comm_done()
        src = dst
    return src


def slab_rows(slab: Slab, full):
    """The stored rows (owned + halos) of a full-grid array for this slab."""
    lo = slab.first_stored_row
    return full[lo: lo + slab.height]


def owned(slab: Slab, buf):
    return buf[slab.halo_top: slab.halo_top + slab.rows]


class TorchExchange:
    """Halo exchange through torch.distributed point-to-point (NCCL or gloo)."""

    def __init__(self, dist, group=None):
        self.dist, self.group = dist, group

    def exchange(self, sends, recvs) -> None:
        d = self.dist
        ops = [d.P2POp(d.isend, buf, peer, self.group) for buf, peer in sends]
        ops += [d.P2POp(d.irecv, buf, peer, self.group) for buf, peer in recvs]
        for req in d.batch_isend_irecv(ops):
            req.wait()


# ---------------------------------------------------------------------------
# CUDA driver: tuned kernel per row block + NCCL halo exchange (torchrun)


class CudaOps(TorchExchange):
    """Step function = the tuned kernel on libtsgpu's stream; exchange on torch's.

    One compiled module per row-block height (the kernel takes the grid
    height as a compile-time constant): the owned rows and, with
    neighbours, the 3h-row bands.
    """

    def __init__(self, dev, compiler, cfg: dict, width: int, iterations: int, heights, dist=None):
        super().__init__(dist)
        from .problems import Hotspot

        self.dev, self.cfg = dev, cfg
        self.variants = {}
        self.modules = []
        for hgt in sorted(set(heights)):
            prob = Hotspot(width=width, height=hgt, iterations=iterations)
            res = compiler.compile(prob.source(), prob.options(cfg))
            if not res.ok:
                raise RuntimeError(res.error)
            rc, mod = dev.load(res.image)
            if rc != 0:
                raise RuntimeError(mod)
            self.modules.append(mod)
            kern = mod.function(prob.kernel_name)
            smem = prob.smem_bytes(cfg)
            if smem > 48 * 1024:
                kern.set_max_dynamic_smem(smem)
            if smem > 0:
                kern.set_smem_carveout(100)
            self.variants[hgt] = (prob, kern, prob.launch_shape(cfg, kern))

    def advance(self, src, dst, power, nsteps: int) -> None:
        prob, kern, shape = self.variants[src.shape[0]]
        self.dev.launch_async([prob.launch(self.cfg, kern, dst.data_ptr(), src.data_ptr(), power.data_ptr(),
                                           nsteps, shape)])

    def copy(self, dst, src) -> None:
        self.dev.copy_async(dst.data_ptr(), src.data_ptr(), src.numel() * src.element_size())

    def _torch_stream(self) -> int:
        import torch

        return torch.cuda.current_stream().cuda_stream

    def edges_done(self) -> None:
        self.dev.signal_stream(self._torch_stream())

    def comm_done(self) -> None:
        self.dev.wait_stream(self._torch_stream())

    def close(self) -> None:
        for m in self.modules:
            m.unload()


class DDRunner:
    """One rank of the decomposed 16384^2 run on its GPU (env: RANK/WORLD_SIZE/LOCAL_RANK).

    Buffers are torch tensors on this rank's GPU (so NCCL can send/recv
    row ranges directly); kernels run through libtsgpu on the same
    primary context.  ``run_once`` enqueues one full run (all launches and
    exchanges) bracketed by device markers; ``verify`` checks the owned rows
    against the single-domain run of the same configuration (bit-exact) and
    the naive Rodinia-form chain (tolerance).
    """

    def __init__(self, config: tuple, width: int = 16384, height: int = 16384, iterations: int = 20,
                 dist=None):
        import os

        import numpy as np
        import torch

        from . import runtime as rt
        from .cuda_backend import Compiler
        from .problems import Hotspot

        self.rank, self.world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(self.local)
        self.dist = dist
        self.prob = Hotspot(width=width, height=height, iterations=iterations)
        self.config = tuple(config)
        self.cfg = dict(zip(self.prob.space.param_names, config))
        self.t = self.cfg["temporal_tiling_factor"]
        self.W, self.H, self.iterations = width, height, iterations
        self.slab = make_slab(self.rank, self.world, height, self.t)
        self.dev = rt.Device(self.local)
        self.cuda = f"cuda:{self.local}"
        self.host_t = np.ascontiguousarray(slab_rows(self.slab, self.prob.temperature()))
        self.host_p = np.ascontiguousarray(slab_rows(self.slab, self.prob.power()))
        self.temp = torch.from_numpy(self.host_t).to(self.cuda)
        self.power = torch.from_numpy(self.host_p).to(self.cuda)
        self.a, self.b = torch.empty_like(self.temp), torch.empty_like(self.temp)
        self.bands = {}
        heights = [self.slab.rows]
        if self.world > 1:
            heights.append(band_rows(self.slab))
            for side in ("top", "bot"):
                self.bands[side] = torch.empty((band_rows(self.slab), width), dtype=torch.float32,
                                               device=self.cuda)
        self.compiler = Compiler()
        self.ops = CudaOps(self.dev, self.compiler, self.cfg, width, iterations, heights, dist)
        self.out = None
        torch.cuda.synchronize()

    @property
    def launch_count(self) -> int:
        return self.dev.launch_count

    def run_once(self):
        self.out = run(self.slab, self.temp, self.power, self.a, self.b, self.iterations, self.t, self.ops,
                       self.bands.get("top"), self.bands.get("bot"))
        return self.out

    def timed(self, repeats: int, marker0: int = 0, marker1: int = 1) -> list:
        """Device times (ms) of ``repeats`` whole runs, each bracketed by markers."""
        import torch

        times = []
        for _ in range(repeats):
            if self.world > 1:
                self.dist.barrier()
            torch.cuda.synchronize()
            self.dev.sync()
            self.dev.mark(marker0)
            self.run_once()
            self.dev.mark(marker1)
            times.append(self.dev.elapsed_ms(marker0, marker1))
        return times

    def owned_rows(self):
        self.dev.sync()
        return owned(self.slab, self.out)

    def verify(self) -> dict:
        import numpy as np

        from .cuda_backend import CudaTarget

        got = self.owned_rows().cpu().numpy()
        tgt = CudaTarget(self.prob, device=self.dev, compiler=self.compiler)
        try:
            st, full = tgt.run_output(self.config)
            if st.value != "ok":
                raise RuntimeError(f"single-domain run failed: {full}")
            r0, n = self.slab.row0, self.slab.rows
            want = full.reshape(self.H, self.W)[r0:r0 + n]
            ref = tgt.answer().reshape(self.H, self.W)[r0:r0 + n]
        finally:
            tgt.close()
        return {"bit_exact_vs_single_domain": bool(np.array_equal(got, want)),
                "max_rel_err_vs_rodinia_chain": float(np.max(np.abs(got.astype(np.float64) - ref))
                                                      / np.max(np.abs(ref)))}

    def close(self):
        self.ops.close()
        self.compiler.shutdown()


def cuda_run(config: tuple, width: int = 16384, height: int = 16384, iterations: int = 20,
             repeats: int = 3, verify: bool = True) -> dict:
    """One rank of the decomposed run (under torchrun for P > 1): best of
    ``repeats`` device times after one warm-up (max over ranks), and the
    verification of :meth:`DDRunner.verify` (AND / max over ranks)."""
    import os

    import torch
    import torch.distributed as tdist

    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1 and not tdist.is_initialized():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
    r = DDRunner(config, width, height, iterations, tdist if world > 1 else None)
    ms = min(r.timed(repeats + 1)[1:])
    res = {"bit_exact_vs_single_domain": None, "max_rel_err_vs_rodinia_chain": None}
    if verify:
        res = r.verify()
    if world > 1:
        t = torch.tensor([ms, 1.0 if res["bit_exact_vs_single_domain"] else 0.0,
                          res["max_rel_err_vs_rodinia_chain"] or 0.0], device=r.cuda)
        tdist.all_reduce(t[:1], op=tdist.ReduceOp.MAX)
        tdist.all_reduce(t[1:2], op=tdist.ReduceOp.MIN)
        tdist.all_reduce(t[2:3], op=tdist.ReduceOp.MAX)
        ms = float(t[0].item())
        if verify:
            res = {"bit_exact_vs_single_domain": bool(t[1].item()), "max_rel_err_vs_rodinia_chain": float(t[2].item())}
    r.close()
    cells = float(width) * height * iterations
    return {"world": world, "config": r.cfg, "ms": ms, "gcells_per_s": cells / ms / 1e6,
            "gflops": cells * r.prob.FLOP_PER_CELL / ms / 1e6, **res, "halo_rows": r.t,
            "slab_rows": r.slab.rows}
