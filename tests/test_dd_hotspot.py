"""Domain-decomposed hotspot: slab + halo exchange logic, gloo on CPU.

Each rank advances its slab with the C oracle (the same clamped-edge
semantics as the CUDA kernel) and exchanges halos with torch.distributed
P2P; the owned rows must be BIT-EXACT with the single-domain run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kernels_ffi as K
from paper_2407_11488_b200.dd_hotspot import make_slab, owned, run, slab_rows
from paper_2407_11488_b200.problems import Hotspot


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, w, h, iters, t):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = Hotspot(width=w, height=h, iterations=iters)
        slab = make_slab(rank, world, h, t)
        temp = torch.from_numpy(np.ascontiguousarray(slab_rows(slab, prob.temperature())))
        power = np.ascontiguousarray(slab_rows(slab, prob.power()))
        a = torch.empty_like(temp)
        b = torch.empty_like(temp)
        k = prob.k

        def step(src, dst, nsteps):
            scratch = np.empty(src.numel(), np.float32)
            K.lib().oracle_hotspot(K._p(dst.numpy().reshape(-1)), K._p(src.numpy().reshape(-1)),
                                   K._p(power.reshape(-1)), w, slab.height, nsteps, k["sdc"], k["rx1"],
                                   k["ry1"], k["rz1"], k["amb"], K._p(scratch))

        res = run(slab, temp, power, a, b, iters, t, step, dist)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), owned(slab, res).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,t", [(2, 3), (3, 4), (4, 5)])
def test_dd_matches_single_domain(tmp_path, world, t):
    w, h, iters = 80, 120, 20
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), w, h, iters, t), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    want = K.hotspot(Hotspot(width=w, height=h, iterations=iters)).reshape(h, w)
    np.testing.assert_array_equal(got, want)


def test_slab_geometry():
    s0, s1, s2 = (make_slab(r, 3, 300, 7) for r in range(3))
    assert (s0.halo_top, s0.halo_bot, s0.height) == (0, 7, 107)
    assert (s1.halo_top, s1.halo_bot, s1.height, s1.first_stored_row) == (7, 7, 114, 93)
    assert (s2.halo_top, s2.halo_bot, s2.row0) == (7, 0, 200)
    with pytest.raises(ValueError):
        make_slab(0, 3, 301, 7)


@pytest.mark.gpu
@pytest.mark.parametrize("config", [(16, 4, 4, 1, 4, 2, 1), (32, 2, 4, 1, 8, 1, 1), (32, 16, 3, 2, 6, 6, 1)])
def test_cuda_run_single_rank_bit_exact(config):
    """The slab driver with the tuned kernel (stream and block-tile modes) on
    one GPU equals the naive reference chain bit-for-bit."""
    from paper_2407_11488_b200.dd_hotspot import cuda_run

    r = cuda_run(config, width=1024, height=768, iterations=20, repeats=1, verify=True)
    assert r["bit_exact"] is True, r
