"""Domain-decomposed hotspot across the GPUs of one node (north_star N9).

The 16384^2 grid is split into P row slabs, one per rank.  Rank p
stores its H/P rows plus a halo of T rows on each side that has a
neighbour (none above rank 0, none below rank P-1), so the slab's own
first/last rows ARE the global boundary rows where one exists.  Every
launch runs the UNMODIFIED tuned kernel (kernels/hotspot.cu, compiled
with GH = slab height) for nsteps <= T steps; its clamped boundary at an
internal slab edge produces wrong values that travel at most nsteps <= T
rows -- i.e. only into the halo -- so the owned rows are exact, and the
halo is refreshed by exchanging T rows with each neighbour between
launches (NCCL send/recv over NVLink via torch.distributed, grouped with
``batch_isend_irecv``; the only data-path collective of the build).

The slab logic is independent of the step function, so the same code
runs (a) on GPUs with the tuned kernel and NCCL and (b) on CPU under
gloo with the C oracle as the step function -- the test that proves the
decomposition bit-exact against the single-domain run (tests/
test_dd_hotspot.py).
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


def make_slab(rank: int, world: int, gh: int, halo: int) -> Slab:
    if gh % world:
        raise ValueError(f"grid height {gh} not divisible by {world} ranks")
    rows = gh // world
    if halo > rows:
        raise ValueError("halo deeper than a slab")
    return Slab(rank, world, rows, rank * rows, halo if rank > 0 else 0,
                halo if rank < world - 1 else 0)


def exchange_halos(slab: Slab, buf, dist, group=None) -> None:
    """Refresh ``buf``'s halo rows from the neighbours (buf: [height][W] tensor)."""
    ops = []
    h = slab.halo_top or slab.halo_bot
    if slab.world == 1 or h == 0:
        return
    top_own = buf[slab.halo_top: slab.halo_top + h]
    bot_own = buf[slab.halo_top + slab.rows - h: slab.halo_top + slab.rows]
    if slab.rank > 0:
        ops.append(dist.P2POp(dist.isend, top_own.contiguous() if not top_own.is_contiguous() else top_own,
                              slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[0: slab.halo_top], slab.rank - 1, group))
    if slab.rank < slab.world - 1:
        ops.append(dist.P2POp(dist.isend, bot_own, slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[slab.halo_top + slab.rows:], slab.rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def run(slab: Slab, temp, power, scratch_a, scratch_b, iterations: int, t: int, step_fn, dist) -> object:
    """Advance ``iterations`` steps in launches of <= t; returns the buffer holding the result.

    ``step_fn(src, dst, nsteps)`` advances the whole slab (tensors
    [height][W]); ``temp`` holds the initial slab INCLUDING valid halos.
    """
    n_launch = math.ceil(iterations / t)
    plan = [t] * (n_launch - 1) + [iterations - t * (n_launch - 1)]
    src = temp
    for i, k in enumerate(plan):
        dst = scratch_a if i % 2 == 0 else scratch_b
        step_fn(src, dst, k)
        if i < n_launch - 1:
            exchange_halos(slab, dst, dist)
        src = dst
    return src


def slab_rows(slab: Slab, full):
    """The stored rows (owned + halos) of a full-grid array for this slab."""
    lo = slab.first_stored_row
    return full[lo: lo + slab.height]


def owned(slab: Slab, buf):
    return buf[slab.halo_top: slab.halo_top + slab.rows]


# ---------------------------------------------------------------------------
# CUDA driver: tuned kernel per slab + NCCL halo exchange (torchrun)


def cuda_run(config: tuple, width: int = 16384, height: int = 16384, iterations: int = 20,
             repeats: int = 3, verify: bool = True) -> dict:
    """One rank of the decomposed run (env: RANK/WORLD_SIZE/LOCAL_RANK).

    Buffers are torch tensors on this rank's GPU (so NCCL can send/recv
    row ranges directly); kernels are launched through libtsgpu on the
    same primary context.  Returns timing (max over ranks) and, with
    ``verify``, whether the owned rows equal the single-GPU result of the
    naive reference chain bit-for-bit.
    """
    import ctypes as C
    import os

    import numpy as np
    import torch
    import torch.distributed as tdist

    from . import runtime as rt
    from .cuda_backend import Compiler
    from .problems import Hotspot

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1 and not tdist.is_initialized():
        tdist.init_process_group("nccl")
    prob = Hotspot(width=width, height=height, iterations=iterations)
    space = prob.space
    cfg = dict(zip(space.param_names, config))
    t = cfg["temporal_tiling_factor"]
    slab = make_slab(rank, world, height, t)
    dev = rt.Device(local)
    full_t = prob.temperature()
    full_p = prob.power()
    dev_t = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, full_t))).to(f"cuda:{local}")
    dev_p = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, full_p))).to(f"cuda:{local}")
    a, b = torch.empty_like(dev_t), torch.empty_like(dev_t)
    slab_prob = Hotspot(width=width, height=slab.height, iterations=iterations)
    comp = Compiler()
    res = comp.compile(slab_prob.source(), slab_prob.options(cfg))
    if not res.ok:
        raise RuntimeError(res.error)
    rc, mod = dev.load(res.image)
    kern = mod.function(slab_prob.kernel_name)
    smem = slab_prob.smem_bytes(cfg)
    if smem > 48 * 1024:
        kern.set_max_dynamic_smem(smem)
    if smem > 0:
        kern.set_smem_carveout(100)
    shape = slab_prob.launch_shape(cfg, kern)  # stream mode: segments sized to this slab
    torch.cuda.synchronize()

    def step(src, dst, nsteps):
        launch = slab_prob.launch(cfg, kern, dst.data_ptr(), src.data_ptr(), dev_p.data_ptr(), nsteps, shape)
        code, err = dev.run([launch])
        if code != rt.OK:
            raise RuntimeError(err)

    class _Dist:
        P2POp = tdist.P2POp if world > 1 else None
        isend = tdist.isend
        irecv = tdist.irecv

        @staticmethod
        def batch_isend_irecv(ops):
            return tdist.batch_isend_irecv(ops)

    times = []
    out = None
    for _ in range(repeats + 1):
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = run(slab, dev_t, dev_p, a, b, iterations, t, step, _Dist)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times = times[1:]  # first repeat is warm-up
    ms = min(times)
    if world > 1:
        tt = torch.tensor([ms], device=f"cuda:{local}")
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        ms = float(tt.item())
    ok = None
    if verify:
        from .cuda_backend import CudaTarget

        ref = CudaTarget(prob, device=dev, compiler=comp)  # full grid, naive reference chain
        want = torch.from_numpy(ref.answer().reshape(height, width)[slab.row0: slab.row0 + slab.rows].copy())
        got = owned(slab, out).cpu()
        ok = bool(torch.equal(got, want))
        ref.close()
        if world > 1:
            flag = torch.tensor([1 if ok else 0], device=f"cuda:{local}")
            tdist.all_reduce(flag, op=tdist.ReduceOp.MIN)
            ok = bool(flag.item())
    mod.unload()
    comp.shutdown()
    cells = float(width) * height * iterations
    return {"world": world, "config": cfg, "ms": ms, "gcells_per_s": cells / ms / 1e6,
            "gflops": cells * prob.FLOP_PER_CELL / ms / 1e6, "bit_exact": ok,
            "halo_rows": t, "slab_rows": slab.rows}
