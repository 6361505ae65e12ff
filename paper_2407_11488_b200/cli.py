"""Command line: ``python -m paper_2407_11488_b200 tune ...``.

Mirrors the reference's ``tunescape tune`` (ref ``ts/cli.py:58-139``: same
options, same output lines, same cache file) and its exit-code contract
(ref ``ts/cli.py:277-283``: a domain error prints ``error: <Type>: <msg>``
and exits 1; usage errors exit 2 through click).  Additions:

* ``--backend cuda:<kernel>`` -- the in-process B200 backend
  (:class:`cuda_backend.CudaTarget` on ``LOCAL_RANK``'s GPU) for one of the
  four bundled kernels (``convolution``, ``hotspot``, ``dedispersion``,
  ``gemm``; also ``gemm_tc``).  ``sim:`` and ``cmd:`` are the reference's.
* ``--strategy genetic`` (north_star) next to brute / random / local.
* ``--devices N`` -- brute force sharded over N GPUs of this node: the
  command re-launches itself under ``torch.distributed.run`` (one process
  per GPU, 127.0.0.1 rendezvous) and the ranks pull configuration chunks
  from a shared queue (:mod:`multigpu`); rank 0 writes the merged cache,
  identical to the one-GPU cache.
* ``--resume LOG`` -- append every observation to a JSON-lines log as it
  is measured and skip configurations already in it (multi-hour sweeps
  survive a lost box; the reference writes only at the end).
* ``--kt-out PATH`` -- also write the Kernel-Tuner-format cache that the
  reference's ``import_external_cache`` reads.
"""

from __future__ import annotations

import os
import sys

import click

from . import store, strategies
from .errors import ProtocolError, TunescapeError
from .measure import Aggregate, MeasurementProtocol, command_backend, simulated_backend
from .paramspace import NeighborScheme, load_space_spec


def _fmt(x: float) -> str:
    return f"{x:.6g}"


def _cuda_backend(kernel: str, space, verify: bool):
    from . import runtime as rt
    from .cuda_backend import CudaTarget
    from .measure import cuda_backend
    from .problems import PROBLEMS, make_problem

    if kernel not in PROBLEMS:
        raise click.UsageError(f"cuda backend kernel must be one of {sorted(PROBLEMS)}, got {kernel!r}")
    prob = make_problem(kernel)
    if prob.space.fingerprint() != space.fingerprint():
        raise ProtocolError(f"--space does not match the {kernel} kernel's space "
                            f"({space.kernel_name} vs {prob.space.kernel_name})")
    dev = rt.Device(int(os.environ.get("LOCAL_RANK", "0")))
    return cuda_backend(CudaTarget(prob, device=dev, verify=verify))


def _load_backend(spec: str, space, workdir, env_pairs, parameterless, verify):
    kind, _, rest = spec.partition(":")
    if kind == "sim" and rest:
        return simulated_backend(store.read_cache(rest))
    if kind == "cmd" and rest:
        env = {}
        for pair in env_pairs:
            name, _, value = pair.partition("=")
            env[name] = value
        return command_backend(rest, workdir=workdir, env=env, parameterless=parameterless)
    if kind == "cuda" and rest:
        return _cuda_backend(rest, space, verify)
    raise click.UsageError(f"backend must be sim:<cache-file>, cmd:<template> or cuda:<kernel>, got {spec!r}")


def _relaunch(devices: int) -> None:
    """Re-run this command as ``devices`` torch.distributed ranks (never returns)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    argv = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={devices}",
            "--master-addr=127.0.0.1", f"--master-port={port}", "-m", "paper_2407_11488_b200"] + sys.argv[1:]
    os.execv(sys.executable, argv)


@click.group()
def cli():
    """Tune kernels on B200 GPUs and record caches the reference reads."""


@cli.command()
@click.option("--space", "space_path", required=True, help="Space spec file (or a bundled space name).")
@click.option("--backend", "backend_spec", required=True,
              help="sim:<cache-file>, cmd:<command template with {param} slots> or cuda:<kernel>.")
@click.option("--strategy", type=click.Choice(["brute", "random", "local", "genetic"]), default="brute",
              show_default=True)
@click.option("--budget", type=int, default=0, help="Max evaluations (random/local/genetic).")
@click.option("--seed", type=int, default=0, show_default=True)
@click.option("--out", "out_path", required=True, help="Cache file to write.")
@click.option("--device", default=None, help="Device name recorded in the cache.")
@click.option("--scheme", type=click.Choice([s.value for s in NeighborScheme]), default=None)
@click.option("--first-improvement", is_flag=True, help="Local search takes the first improving neighbor.")
@click.option("--warmup", type=int, default=1, show_default=True)
@click.option("--runs", type=int, default=7, show_default=True)
@click.option("--aggregate", type=click.Choice([a.value for a in Aggregate]), default="mean", show_default=True)
@click.option("--timeout-ms", type=float, default=60_000.0, show_default=True)
@click.option("--workdir", default=None, help="Working directory for cmd backends.")
@click.option("--env", "env_pairs", multiple=True, help="NAME=VALUE for cmd backends (repeatable).")
@click.option("--parameterless", is_flag=True, help="Allow a cmd template without placeholders.")
@click.option("--devices", type=int, default=1, show_default=True,
              help="GPUs for a sharded brute-force sweep (cuda backend).")
@click.option("--chunk", type=int, default=16, show_default=True, help="Configurations per queue chunk.")
@click.option("--resume", "resume_path", default=None, help="JSON-lines observation log to append to / resume from.")
@click.option("--kt-out", "kt_out_path", default=None, help="Also write a Kernel-Tuner-format cache here.")
@click.option("--no-verify", is_flag=True, help="cuda backend: skip on-device output verification.")
def tune(space_path, backend_spec, strategy, budget, seed, out_path, device, scheme, first_improvement,
         warmup, runs, aggregate, timeout_ms, workdir, env_pairs, parameterless, devices, chunk,
         resume_path, kt_out_path, no_verify):
    """Search a space for the best configuration and record a cache."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if devices > 1:
        if not backend_spec.startswith("cuda:") or strategy != "brute":
            raise click.UsageError("--devices > 1 needs --backend cuda:<kernel> and --strategy brute")
        if world == 1:
            _relaunch(devices)
    space = load_space_spec(space_path)
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    backend = _load_backend(backend_spec, space, workdir, env_pairs, parameterless, not no_verify)
    protocol = MeasurementProtocol(warmup_runs=warmup, benchmark_runs=runs, aggregate=Aggregate(aggregate),
                                   timeout_ms=timeout_ms)
    metadata = {"strategy": strategy, "seed": str(seed)}
    rank = 0
    try:
        if strategy == "brute" and (world > 1 or resume_path):
            from .multigpu import sharded_sweep, merged_result, torch_dist_plumbing

            import glob

            st, gather, rank, world = torch_dist_plumbing()
            mine = f"{resume_path}.rank{rank}" if resume_path and world > 1 else resume_path
            # every log of an earlier run counts (one file, or one per rank)
            earlier = sorted(set(glob.glob(f"{resume_path}.rank*")) | {resume_path}) if resume_path else []
            trace, _ = sharded_sweep(space, list(space.enumerate_configs()), backend, protocol, chunk, st,
                                     gather, mine, rank, resume_from=earlier)
            result = merged_result(trace)
            cache = strategies.result_to_cache(space, result, strategies.default_device_name(backend, device),
                                               metadata)
        elif strategy == "brute":
            result, cache = strategies.brute_force(space, backend, protocol, device, metadata=metadata)
        else:
            if strategy == "random":
                result = strategies.random_search(space, backend, protocol, budget, seed)
            elif strategy == "local":
                result = strategies.greedy_local_search(space, backend, protocol, budget, seed, scheme=scheme,
                                                        first_improvement=first_improvement)
            else:
                result = strategies.genetic_algorithm(space, backend, protocol, budget, seed)
            metadata["budget"] = str(budget)
            cache = strategies.result_to_cache(space, result,
                                               device_name=strategies.default_device_name(backend, device),
                                               metadata=metadata)
    finally:
        if backend.kind == "cuda":
            backend.target.close()
    if rank == 0:
        store.write_cache(cache, out_path)
        if kt_out_path:
            store.write_kernel_tuner_cache(cache, kt_out_path, space=space)
        click.echo(f"evaluations : {result.evaluations_used}")
        if result.best is not None:
            click.echo(f"best config : {','.join(map(str, result.best))}")
            click.echo(f"best_ms     : {_fmt(result.best_observation.time_ms)}")
        for note in result.notes:
            click.echo(f"note        : {note}")
        click.echo(f"wrote {out_path}")
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main(argv=None):
    """Entry point mapping domain errors to exit code 1 (ref ts/cli.py:277-283)."""
    try:
        cli.main(args=argv, prog_name="paper_2407_11488_b200", standalone_mode=True)
    except TunescapeError as e:
        click.echo(f"error: {type(e).__name__}: {e}", err=True)
        sys.exit(1)
