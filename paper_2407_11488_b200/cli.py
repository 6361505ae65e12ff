"""Command line: ``python -m paper_2407_11488_b200 tune ...``.

``tune`` takes the reference's options and prints the reference's summary
lines (``evaluations :``, ``best config :``, ``best_ms     :``,
``note        :``, ``wrote <path>``), writes the same cache file, and keeps
its exit-code contract: a domain error prints ``error: <Type>: <msg>`` and
exits 1, a usage error exits 2 (click).  B200 additions:

* ``--backend cuda:<kernel>`` -- the in-process B200 backend
  (:class:`cuda_backend.CudaTarget` on ``LOCAL_RANK``'s GPU) for one of the
  bundled kernels (``convolution``, ``hotspot``, ``dedispersion``, ``gemm``,
  ``gemm_tc``); ``sim:`` and ``cmd:`` are the reference's kinds;
* ``--strategy genetic`` next to brute / random / local;
* ``--devices N`` (cuda backend) -- any strategy on N GPUs of this node: the command
  re-launches itself under ``torch.distributed.run`` (one process per GPU,
  127.0.0.1 rendezvous) and every batch the strategy issues is split over
  the ranks (:class:`multigpu.ShardedEvaluator`); rank 0 writes the cache,
  identical to the one-GPU cache;
* ``--resume LOG`` -- every measured observation is appended to
  ``LOG`` (``LOG.rank<N>`` per rank) and a rerun skips whatever any earlier
  log holds; a log recorded for another space or protocol is refused;
* ``--kt-out PATH`` -- also write the Kernel-Tuner-format cache that the
  reference's ``import_external_cache`` reads;
* the reference's analysis commands over any cache (:mod:`landscape`):
  ``analyze stats|topk|centrality|portability``, ``export dist|ffg``,
  ``import --from external``.
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import click

from . import landscape, store, strategies
from .errors import ProtocolError, TunescapeError
from .measure import Aggregate, MeasurementProtocol, command_backend, simulated_backend
from .paramspace import NeighborScheme, load_space_spec

STRATEGY_NAMES = ("brute", "random", "local", "genetic")


# ---------------------------------------------------------------------------
# Backends named on the command line: "<kind>:<argument>"


def _sim(arg, job):
    return simulated_backend(store.read_cache(arg))


def _cmd(arg, job):
    env = dict(pair.partition("=")[::2] for pair in job.env_pairs)
    return command_backend(arg, workdir=job.workdir, env=env, parameterless=job.parameterless)


def _cuda(arg, job):
    from . import runtime as rt
    from .cuda_backend import CudaTarget
    from .measure import cuda_backend
    from .problems import PROBLEMS, make_problem

    if arg not in PROBLEMS:
        raise click.UsageError(f"cuda backend kernel must be one of {sorted(PROBLEMS)}, got {arg!r}")
    problem = make_problem(arg)
    if problem.space.fingerprint() != job.space.fingerprint():
        raise ProtocolError(f"--space does not match the {arg} kernel's space "
                            f"({job.space.kernel_name} vs {problem.space.kernel_name})")
    device = rt.Device(_local_device())
    return cuda_backend(CudaTarget(problem, device=device, verify=job.verify))


def _local_device() -> int:
    """This rank's GPU: LOCAL_RANK, wrapped over the visible GPUs (more ranks
    than GPUs share them -- a functional test of the sharded path on a
    one-GPU host; one rank per GPU is the measuring setup)."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    try:
        import torch

        n = torch.cuda.device_count()
    except Exception:  # noqa: BLE001 -- no torch: one device per rank
        n = 0
    return local % n if n else local


_BACKEND_KINDS = {"sim": _sim, "cmd": _cmd, "cuda": _cuda}


@dataclass
class TuneJob:
    """One ``tune`` invocation, resolved from its options."""

    space: object
    strategy: str
    budget: int
    seed: int
    scheme: str | None
    first_improvement: bool
    protocol: MeasurementProtocol
    workdir: str | None
    env_pairs: tuple
    parameterless: bool
    verify: bool
    chunk: int
    resume: str | None

    def backend(self, spec: str):
        kind, _, arg = spec.partition(":")
        make = _BACKEND_KINDS.get(kind) if arg else None
        if make is None:
            raise click.UsageError(
                f"backend must be sim:<cache-file>, cmd:<template> or cuda:<kernel>, got {spec!r}")
        return make(arg, self)

    def evaluator(self, backend, comm):
        """Local evaluator, or the sharded one (several ranks and/or a resume log)."""
        if comm.world == 1 and not self.resume:
            return strategies.LocalEvaluator(self.space, backend, self.protocol)
        from .multigpu import ShardedEvaluator

        mine = self.resume if comm.world == 1 else (f"{self.resume}.rank{comm.rank}" if self.resume else None)
        earlier = store.rank_logs(self.resume) if self.resume else []
        return ShardedEvaluator(self.space, backend, self.protocol, comm, self.chunk, mine, earlier)

    def run(self, evaluator):
        s, ev = self.space, evaluator
        if self.strategy == "brute":
            return strategies.brute_force(s, None, None, evaluator=ev)[0]
        if self.strategy == "random":
            return strategies.random_search(s, None, None, self.budget, self.seed, evaluator=ev)
        if self.strategy == "local":
            return strategies.greedy_local_search(s, None, None, self.budget, self.seed, scheme=self.scheme,
                                                  first_improvement=self.first_improvement, evaluator=ev)
        return strategies.genetic_algorithm(s, None, None, self.budget, self.seed, evaluator=ev)


def _report(result, out_path: str) -> None:
    lines = [f"evaluations : {result.evaluations_used}"]
    if result.best is not None:
        lines += [f"best config : {','.join(str(v) for v in result.best)}",
                  f"best_ms     : {result.best_observation.time_ms:.6g}"]
    lines += [f"note        : {n}" for n in result.notes]
    lines.append(f"wrote {out_path}")
    for line in lines:
        click.echo(line)


def _relaunch(devices: int) -> None:
    """Re-run this command as ``devices`` torch.distributed ranks (never returns)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                              f"--nproc-per-node={devices}", "--master-addr=127.0.0.1",
                              f"--master-port={port}", "-m", "paper_2407_11488_b200", *sys.argv[1:]])


def _join_ranks(world: int, backend_spec: str):
    """Initialise the process group of a multi-rank run (NCCL for GPU ranks)."""
    import torch.distributed as dist

    if world == 1 or dist.is_initialized():
        return
    # the sharded sweep's only inter-rank traffic is host-side (a TCPStore
    # counter and one gather of the results): gloo, for every backend
    dist.init_process_group("gloo")


# ---------------------------------------------------------------------------
# click wiring: the tune options as a table


_TUNE_OPTIONS = [
    (("--space", "space_path"), dict(required=True, help="Space spec file (or a bundled space name).")),
    (("--backend", "backend_spec"), dict(required=True,
                                         help="sim:<cache-file>, cmd:<template with {param} slots> or cuda:<kernel>.")),
    (("--strategy",), dict(type=click.Choice(STRATEGY_NAMES), default="brute", show_default=True)),
    (("--budget",), dict(type=int, default=0, help="Max evaluations (random/local/genetic).")),
    (("--seed",), dict(type=int, default=0, show_default=True)),
    (("--out", "out_path"), dict(required=True, help="Cache file to write.")),
    (("--device",), dict(default=None, help="Device name recorded in the cache.")),
    (("--scheme",), dict(type=click.Choice([s.value for s in NeighborScheme]), default=None)),
    (("--first-improvement",), dict(is_flag=True, help="Local search takes the first improving neighbor.")),
    (("--warmup",), dict(type=int, default=1, show_default=True)),
    (("--runs",), dict(type=int, default=7, show_default=True)),
    (("--aggregate",), dict(type=click.Choice([a.value for a in Aggregate]), default="mean", show_default=True)),
    (("--timeout-ms",), dict(type=float, default=60_000.0, show_default=True)),
    (("--workdir",), dict(default=None, help="Working directory for cmd backends.")),
    (("--env", "env_pairs"), dict(multiple=True, help="NAME=VALUE for cmd backends (repeatable).")),
    (("--parameterless",), dict(is_flag=True, help="Allow a cmd template without placeholders.")),
    (("--devices",), dict(type=int, default=1, show_default=True,
                          help="Ranks (GPUs of this node) sharing every measurement batch.")),
    (("--chunk",), dict(type=int, default=16, show_default=True, help="Configurations per queue chunk.")),
    (("--resume", "resume_path"), dict(default=None, help="JSON-lines observation log to append to / resume from.")),
    (("--kt-out", "kt_out_path"), dict(default=None, help="Also write a Kernel-Tuner-format cache here.")),
    (("--no-verify",), dict(is_flag=True, help="cuda backend: skip on-device output verification.")),
]


def _with_options(table):
    def apply(fn):
        for decls, kwargs in reversed(table):
            fn = click.option(*decls, **kwargs)(fn)
        return fn
    return apply


@click.group()
def cli():
    """Tune kernels on B200 GPUs and analyse the caches (reference-compatible)."""


@cli.command()
@_with_options(_TUNE_OPTIONS)
def tune(space_path, backend_spec, strategy, budget, seed, out_path, device, scheme, first_improvement,
         warmup, runs, aggregate, timeout_ms, workdir, env_pairs, parameterless, devices, chunk,
         resume_path, kt_out_path, no_verify):
    """Search a space for the best configuration and record a cache."""
    from .multigpu import current_comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if devices > 1 and not backend_spec.startswith("cuda:"):
        raise click.UsageError("--devices > 1 shards measurements over GPUs: it needs --backend cuda:<kernel>")
    if devices > 1 and world == 1:
        _relaunch(devices)
    job = TuneJob(load_space_spec(space_path), strategy, budget, seed, scheme, first_improvement,
                  MeasurementProtocol(warmup_runs=warmup, benchmark_runs=runs, aggregate=Aggregate(aggregate),
                                      timeout_ms=timeout_ms),
                  workdir, tuple(env_pairs), parameterless, not no_verify, chunk, resume_path)
    _join_ranks(world, backend_spec)
    comm = current_comm()
    backend = job.backend(backend_spec)
    ev = job.evaluator(backend, comm)
    try:
        result = job.run(ev)
    finally:
        if hasattr(ev, "close"):
            ev.close()
        if backend.kind == "cuda":
            backend.target.close()
    metadata = {"strategy": strategy, "seed": str(seed)}
    if strategy != "brute":
        metadata["budget"] = str(budget)
    if comm.rank == 0:
        cache = strategies.result_to_cache(job.space, result, ev.device_name(device), metadata)
        store.write_cache(cache, out_path)
        if kt_out_path:
            store.write_kernel_tuner_cache(cache, kt_out_path, space=job.space)
        _report(result, out_path)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


@cli.group()
def analyze():
    """Landscape statistics of caches (impact, difficulty, portability)."""


def _rows(pairs) -> None:
    for name, value in pairs:
        click.echo(f"{name:<7} : {value}")


@analyze.command("stats")
@click.option("--cache", "cache_path", required=True)
def analyze_stats(cache_path):
    """Table 4 row: median, maximum, impact (+ best/worst, best time)."""
    cache = store.read_cache(cache_path)
    st = landscape.perf_stats(cache)
    _rows((("kernel", f"{cache.kernel_name} on {cache.device_name}"),
           ("records", f"{st.n_ok} ok, {st.n_failed} failed"),
           ("median", f"{st.median_perf:.6g}"), ("maximum", f"{st.max_perf:.6g}"),
           ("impact", f"{st.impact:.1f}x"), ("range", f"{st.best_over_worst:.1f}x (best/worst)"),
           ("best_ms", f"{st.min_time_ms:.6g}")))


@analyze.command("topk")
@click.option("--cache", "cache_path", required=True)
@click.option("-k", "k", type=int, default=5, show_default=True)
def analyze_topk(cache_path, k):
    """Tables 5-8: the k best configurations by metric."""
    cache = store.read_cache(cache_path)
    click.echo(f"# top {k} of {cache.kernel_name} on {cache.device_name} ({', '.join(cache.param_order)})")
    for key, value in landscape.top_k(cache, k):
        click.echo(f"{key}  {value:.6g}")


@analyze.command("centrality")
@click.option("--cache", "cache_path", required=True)
@click.option("--space", "space_path", required=True)
@click.option("--scheme", type=click.Choice([s.value for s in NeighborScheme]), default=None)
@click.option("--p-max", type=float, default=0.15, show_default=True)
@click.option("--p-step", type=float, default=0.005, show_default=True)
@click.option("--damping", type=float, default=landscape.DEFAULT_DAMPING, show_default=True)
@click.option("--out", "out_path", default=None, help="CSV of (p, C_p).")
def analyze_centrality(cache_path, space_path, scheme, p_max, p_step, damping, out_path):
    """Figs. 4/6/8/10a: proportion of PageRank centrality of near-optimal minima."""
    if p_step <= 0 or p_max < 0:
        raise click.UsageError("--p-step must be positive and --p-max non-negative")
    g = landscape.build_ffg(store.read_cache(cache_path), load_space_spec(space_path), scheme)
    curve = landscape.centrality_curve(g, damping=damping, p_grid=landscape.p_grid(p_max, p_step))
    for name, value in (("scheme", g.scheme.value), ("nodes", g.n_nodes), ("edges", g.n_edges),
                        ("minima", curve.minima_count), ("C_0", f"{curve.c_p_values[0]:.6g}"),
                        (f"C_{p_max:g}", f"{curve.c_p_values[-1]:.6g}")):
        click.echo(f"{name:<12} : {value}")
    if out_path:
        landscape.write_centrality_csv(curve, out_path)
        click.echo(f"wrote {out_path}")


@analyze.command("portability")
@click.option("--caches", "cache_list", required=True, help="Comma-separated cache files.")
@click.option("--subset", default=None, help="Comma-separated device names (default: all).")
@click.option("--out", "out_path", default=None, help="JSON report.")
def analyze_portability(cache_list, subset, out_path):
    """Figs. 9/10b: the configuration with the best performance portability."""
    caches = {}
    for path in cache_list.split(","):
        cache = store.read_cache(path)
        if cache.device_name in caches:
            raise click.UsageError(f"duplicate device name {cache.device_name!r} in --caches")
        caches[cache.device_name] = cache
    report = landscape.best_portable_config(caches, subset.split(",") if subset else None)
    click.echo(f"config      : {report.config}")
    for dev, eff in zip(report.devices, report.efficiencies):
        click.echo(f"  {dev:<10}: {eff:.4f}")
    click.echo(f"pp          : {report.pp:.6g}")
    if out_path:
        landscape.write_portability_json(report, out_path)
        click.echo(f"wrote {out_path}")


@cli.group()
def export():
    """Datasets for plotting (distribution CSV, FFG DOT)."""


@export.command("dist")
@click.option("--cache", "cache_path", required=True)
@click.option("--out", "out_path", required=True)
def export_dist(cache_path, out_path):
    """Figs. 3/5/7/9a: performance relative to the optimum, per configuration."""
    data = landscape.export_distribution(store.read_cache(cache_path))
    landscape.write_distribution_csv(data, out_path)
    for q, v in data.quantiles:
        click.echo(f"q{q:<2} : {v:.6g}")
    click.echo(f"wrote {out_path}")


@export.command("ffg")
@click.option("--cache", "cache_path", required=True)
@click.option("--space", "space_path", required=True)
@click.option("--scheme", type=click.Choice([s.value for s in NeighborScheme]), default=None)
@click.option("--out", "out_path", required=True)
def export_ffg(cache_path, space_path, scheme, out_path):
    """Fig. 2: the fitness flow graph as Graphviz DOT."""
    g = landscape.build_ffg(store.read_cache(cache_path), load_space_spec(space_path), scheme)
    with open(out_path, "w", encoding="utf-8") as fh:
        fh.write(landscape.export_dot(g))
    click.echo(f"wrote {out_path}")


@cli.command("import")
@click.option("--from", "source_format", type=click.Choice(["external"]), default="external", show_default=True)
@click.option("--in", "in_path", required=True, help="Kernel-Tuner-format cache file.")
@click.option("--space", "space_path", default=None, help="Validate every configuration against this space.")
@click.option("--device", default=None, help="Device name to record.")
@click.option("--out", "out_path", required=True)
def import_cache(source_format, in_path, space_path, device, out_path):
    """Convert a Kernel Tuner cache into a native cache."""
    space = load_space_spec(space_path) if space_path else None
    cache = store.import_external_cache(in_path, expected_space=space, device_name=device)
    store.write_cache(cache, out_path)
    click.echo(f"records : {len(cache.records)} ({len(cache.ok_records())} ok)")
    click.echo(f"wrote {out_path}")


def main(argv=None):
    """Entry point: domain errors print ``error: <Type>: <msg>`` and exit 1."""
    try:
        cli.main(args=argv, prog_name="paper_2407_11488_b200", standalone_mode=True)
    except TunescapeError as e:
        click.echo(f"error: {type(e).__name__}: {e}", err=True)
        sys.exit(1)
