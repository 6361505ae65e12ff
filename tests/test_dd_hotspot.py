"""Domain-decomposed hotspot: the overlapped slab schedule (dd_hotspot.run).

CPU (gloo): each rank advances its bands and owned rows with the C
oracle (the same clamped-edge semantics and operation order as the tuned
CUDA kernel) and exchanges halos with torch.distributed P2P; the owned
rows must be BIT-EXACT with the single-domain run.

GPU (one device): the same schedule with the tuned kernel on libtsgpu
streams -- several virtual ranks in one process (threads, one libtsgpu
context each) and a delayed copy on a shared torch stream standing in
for NCCL.  It is bit-exact with the stream ordering of the C ABI
(tsg_stream_signal / tsg_stream_wait), and demonstrably wrong without it.
"""

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kernels_ffi as K
from paper_2407_11488_b200.dd_hotspot import TorchExchange, band_rows, make_slab, owned, run, slab_rows
from paper_2407_11488_b200.problems import Hotspot


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps(TorchExchange):
    """Step function = the C oracle of the tuned arithmetic on CPU tensors."""

    def __init__(self, prob, dist_mod):
        super().__init__(dist_mod)
        self.w = prob.W
        self.c = prob.tuned_coefficients(prob.k)

    def advance(self, src, dst, power, nsteps):
        c = self.c
        scratch = np.empty(src.numel(), np.float32)
        K.lib().oracle_hotspot_tuned(K._p(dst.numpy().reshape(-1)), K._p(src.numpy().reshape(-1)),
                                     K._p(power.numpy().reshape(-1)), self.w, src.shape[0], nsteps, c["at"],
                                     c["ay"], c["ax"], c["ap"], c["ac"], K._p(scratch))

    def copy(self, dst, src):
        dst.copy_(src)

    def edges_done(self):
        pass

    def comm_done(self):
        pass


def _worker(rank, world, port, outdir, w, h, iters, t):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = Hotspot(width=w, height=h, iterations=iters)
        slab = make_slab(rank, world, h, t)
        temp = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, prob.temperature())))
        power = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, prob.power())))
        a, b = torch.empty_like(temp), torch.empty_like(temp)
        bt = torch.empty((band_rows(slab), w), dtype=torch.float32)
        bb = torch.empty_like(bt)
        res = run(slab, temp, power, a, b, iters, t, OracleOps(prob, dist), bt, bb)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), owned(slab, res).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,t", [(2, 3), (3, 4), (4, 5), (2, 7)])
def test_dd_matches_single_domain(tmp_path, world, t):
    w, h, iters = 80, 120, 20
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), w, h, iters, t), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    want = K.hotspot_tuned(Hotspot(width=w, height=h, iterations=iters)).reshape(h, w)
    np.testing.assert_array_equal(got, want)


def test_slab_geometry():
    s0, s1, s2 = (make_slab(r, 3, 300, 7) for r in range(3))
    assert (s0.halo_top, s0.halo_bot, s0.height) == (0, 7, 107)
    assert (s1.halo_top, s1.halo_bot, s1.height, s1.first_stored_row) == (7, 7, 114, 93)
    assert (s2.halo_top, s2.halo_bot, s2.row0) == (7, 0, 200)
    assert band_rows(s1) == 21
    with pytest.raises(ValueError):
        make_slab(0, 3, 301, 7)
    with pytest.raises(ValueError):  # the overlapped schedule needs >= 2 halos of owned rows
        make_slab(0, 8, 80, 6)


class _Recorder:
    def __init__(self):
        self.log = []

    def advance(self, src, dst, power, k):
        self.log.append(("advance", src.shape[0], k))

    def copy(self, dst, src):
        self.log.append(("copy", src.shape[0]))

    def edges_done(self):
        self.log.append(("edges_done",))

    def exchange(self, sends, recvs):
        self.log.append(("exchange", [p for _, p in sends], [p for _, p in recvs]))

    def comm_done(self):
        self.log.append(("comm_done",))


def test_schedule_orders_exchange_between_edges_and_next_launch():
    """Middle rank, 20 iterations at T=8: 3 launches (8, 8, 4); per launch
    two bands, then the interior, the exchange (not after the last), the
    patches, and the compute stream waits for the exchange."""
    slab = make_slab(1, 3, 300, 8)
    buf = np.zeros((slab.height, 4), np.float32)
    band = np.zeros((band_rows(slab), 4), np.float32)
    rec = _Recorder()
    run(slab, buf, buf, buf.copy(), buf.copy(), 20, 8, rec, band, band.copy())
    per = [("advance", 24, 8), ("advance", 24, 8), ("edges_done",), ("advance", 100, 8),
           ("exchange", [0, 2], [0, 2]), ("copy", 8), ("copy", 8), ("comm_done",)]
    last = [("advance", 24, 4), ("advance", 24, 4), ("advance", 100, 4), ("copy", 8), ("copy", 8)]
    assert rec.log == per + per + last


# ---------------------------------------------------------------------------
# GPU: virtual ranks on one device


class _VirtualComm:
    """NCCL stand-in for virtual ranks: a shared torch stream; a copy of each
    send into the peer's receive buffer after a deliberate device delay."""

    def __init__(self, world, delay_cycles):
        self.world = world
        self.delay = delay_cycles
        self.stream = torch.cuda.Stream()
        self.barrier = threading.Barrier(world)
        self.mail = {}


def _virtual_rank(rank, comm, cfg, w, h, iters, results, ordered, errors):
    try:
        from paper_2407_11488_b200 import runtime as rt
        from paper_2407_11488_b200.cuda_backend import Compiler
        from paper_2407_11488_b200.dd_hotspot import CudaOps

        class VirtualOps(CudaOps):
            def exchange(self, sends, recvs):
                for buf, peer in sends:
                    comm.mail[(rank, peer)] = buf
                comm.barrier.wait()  # every rank's edges_done is on the stream
                with torch.cuda.stream(comm.stream):
                    torch.cuda._sleep(comm.delay)
                    for buf, peer in recvs:
                        buf.copy_(comm.mail[(peer, rank)])
                comm.barrier.wait()  # every copy is on the stream

            def _torch_stream(self):
                return comm.stream.cuda_stream

            def edges_done(self):
                if ordered:
                    super().edges_done()

            def comm_done(self):
                if ordered:
                    super().comm_done()

        prob = Hotspot(width=w, height=h, iterations=iters)
        t = cfg["temporal_tiling_factor"]
        slab = make_slab(rank, comm.world, h, t)
        dev = rt.Device(0)
        temp = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, prob.temperature()))).cuda()
        power = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, prob.power()))).cuda()
        a, b = torch.empty_like(temp), torch.empty_like(temp)
        bt = torch.empty((band_rows(slab), w), dtype=torch.float32, device="cuda")
        bb = torch.empty_like(bt)
        comp = Compiler(workers=2)
        ops = VirtualOps(dev, comp, cfg, w, iters, [slab.rows, band_rows(slab)])
        torch.cuda.synchronize()
        out = run(slab, temp, power, a, b, iters, t, ops, bt, bb)
        dev.sync()
        torch.cuda.synchronize()
        results[rank] = owned(slab, out).cpu().numpy()
        ops.close()
        comp.shutdown()
        dev.close()
    except Exception as e:  # noqa: BLE001
        errors.append(repr(e))
        comm.barrier.abort()


def _virtual_run(config, world, ordered, w=512, h=384, iters=20, delay=20_000_000):
    prob = Hotspot(width=w, height=h, iterations=iters)
    cfg = dict(zip(prob.space.param_names, config))
    comm = _VirtualComm(world, delay)
    results, errors = [None] * world, []
    th = [threading.Thread(target=_virtual_rank, args=(r, comm, cfg, w, h, iters, results, ordered, errors))
          for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    return np.concatenate(results), K.hotspot_tuned(prob).reshape(h, w)


@pytest.mark.gpu
@pytest.mark.parametrize("config,world", [((32, 2, 4, 1, 8, 2, 1), 4), ((16, 4, 4, 1, 4, 2, 1), 3),
                                          ((32, 16, 3, 2, 6, 6, 1), 2), ((2, 16, 9, 6, 8, 4, 0), 2)])
def test_virtual_ranks_bit_exact(config, world):
    """The overlapped schedule with the tuned kernel (stream, stream_smem and
    block-tile modes) and the C-ABI stream ordering: bit-exact vs the oracle."""
    got, want = _virtual_run(config, world, ordered=True)
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_without_stream_ordering_the_halos_race():
    """Same run with the two ordering calls removed: the next launch reads
    halo rows before the (delayed) receive lands -- the race the C-ABI
    ordering exists for."""
    got, want = _virtual_run((32, 2, 4, 1, 8, 2, 1), 4, ordered=False)
    assert not np.array_equal(got, want)


@pytest.mark.gpu
def test_stream_wait_orders_a_foreign_producer():
    """tsg_stream_wait: a kernel on the libtsgpu stream sees what a delayed
    producer on a torch stream wrote, exactly when the wait is in place."""
    from paper_2407_11488_b200 import runtime as rt

    dev = rt.Device(0)
    try:
        side = torch.cuda.Stream()
        for wait in (True, False):
            src = torch.zeros(1 << 20, device="cuda")
            dst = torch.full_like(src, -1.0)
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                torch.cuda._sleep(50_000_000)
                src.fill_(7.0)
            if wait:
                dev.wait_stream(side.cuda_stream)
            dev.copy_async(dst.data_ptr(), src.data_ptr(), src.numel() * 4)
            dev.sync()
            torch.cuda.synchronize()
            seen = float(dst[0].item())
            assert seen == (7.0 if wait else 0.0), (wait, seen)
    finally:
        dev.close()


@pytest.mark.gpu
@pytest.mark.parametrize("config", [(16, 4, 4, 1, 4, 2, 1), (32, 2, 4, 1, 8, 1, 1), (32, 16, 3, 2, 6, 6, 1)])
def test_cuda_run_single_rank_bit_exact(config):
    """cuda_run on one GPU (one slab) equals the single-domain tuned run."""
    from paper_2407_11488_b200.dd_hotspot import cuda_run

    r = cuda_run(config, width=1024, height=768, iterations=20, repeats=1, verify=True)
    assert r["bit_exact_vs_single_domain"] is True, r
    assert r["max_rel_err_vs_rodinia_chain"] < 1e-5, r
