"""Kernel-Tuner-style facade: ``tune_kernel`` / ``run_kernel``.

The north_star's drop-in surface.  Semantics of the search-space side
(``tune_params`` dict order = canonical parameter order, ``restrictions``
as reference-grammar strings or callables, enumeration order,
strategies, protocol of 1 warmup + ``iterations`` runs, failures as
statuses) are the reference's (`pkg/src/tunescape/paramspace.py`,
`strategies.py`, `measure.py`); the argument conventions follow Kernel
Tuner's public API:

* tunables reach the kernel as ``#define name value`` lines (plus any
  ``defines``), and ``block_size_x/y/z`` (or ``block_size_names``) give
  the thread block (default 256x1x1);
* grid = ceil(problem_size / grid_div), grid_div defaulting to the block
  size per dimension; ``grid_div_*`` may be lists of parameter names
  (their product), expressions in the restriction grammar, or callables;
* ``arguments``: numpy arrays are copied to the device, numpy scalars are
  passed by value; ``cmem_args`` fill ``__constant__`` symbols;
  ``smem_args={"size": int|callable}`` sets dynamic shared memory;
* ``answer`` (list aligned with ``arguments``; None = unchecked) is
  verified after a dedicated run with output buffers zeroed first;
  float32 outputs are compared ON THE DEVICE (allclose semantics:
  |out-ans| <= atol + 1e-5*|ans|), others on the host; ``verify`` may
  override (called as ``verify(answer, result, atol=atol)``);
* ``strategy`` in {brute_force, random_sample, genetic_algorithm,
  greedy_ls}; ``strategy_options`` understands max_fevals, fraction,
  seed, popsize, maxiter, mutation_chance;
* returns ``(results, env)``: one dict per measured configuration (the
  parameters, ``time`` = mean ms, ``times``, metrics, ``status``) and an
  environment dict.  ``cache=`` writes a Kernel Tuner cache file the
  reference's ``import_external_cache`` ingests.

Only CUDA on sm_100a exists: ``lang`` other than "CUDA" is an error (no
HIP/OpenCL dispatch, north_star).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from pathlib import Path
from typing import Any, Callable

import numpy as np

from . import expressions as ex
from . import runtime as rt
from .cuda_backend import Compiler
from .errors import ProtocolError, VerificationError
from .measure import BackendDescriptor, MeasurementProtocol, Observation, Status, aggregate_times
from .paramspace import config_key, space_from_tune_params
from .store import TuningCache, write_kernel_tuner_cache
from .strategies import STRATEGIES, result_to_cache

_RC_STATUS = {rt.ERR_COMPILE: Status.COMPILE_FAILED, rt.ERR_INVALID: Status.INVALID,
              rt.ERR_RUNTIME: Status.RUNTIME_FAILED, rt.ERR_TIMEOUT: Status.TIMEOUT,
              rt.ERR_ARG: Status.INVALID}

_SCALAR_CTYPES = {
    np.dtype(np.int8): C.c_int8, np.dtype(np.int16): C.c_int16, np.dtype(np.int32): C.c_int32,
    np.dtype(np.int64): C.c_int64, np.dtype(np.uint8): C.c_uint8, np.dtype(np.uint16): C.c_uint16,
    np.dtype(np.uint32): C.c_uint32, np.dtype(np.uint64): C.c_uint64,
    np.dtype(np.float32): C.c_float, np.dtype(np.float64): C.c_double,
}


def _source_text(kernel_source) -> str:
    if isinstance(kernel_source, (list, tuple)):
        kernel_source = kernel_source[0]
    if isinstance(kernel_source, Path) or (isinstance(kernel_source, str) and "\n" not in kernel_source
                                           and kernel_source.endswith((".cu", ".cuh"))
                                           and Path(kernel_source).exists()):
        return Path(kernel_source).read_text()
    return str(kernel_source)


def _eval_param_expr(expr, params: dict):
    if callable(expr):
        return expr(params)
    if isinstance(expr, (int, np.integer)):
        return int(expr)
    if isinstance(expr, str):
        if expr in params:
            return params[expr]
        node = ex.parse_expression(expr)
        return ex.evaluate(node, params)
    if isinstance(expr, (list, tuple)):
        v = 1
        for e in expr:
            v *= _eval_param_expr(e, params)
        return v
    raise ProtocolError(f"cannot interpret {expr!r}")


class KernelInstance:
    """Geometry + source of one configuration (Kernel Tuner conventions)."""

    def __init__(self, spec: "KernelSpec", params: dict):
        self.spec, self.params = spec, params
        names = spec.block_size_names
        self.block = tuple(int(params.get(n, d)) for n, d in zip(names, (256, 1, 1)))
        ps = spec.problem_size
        if callable(ps):
            ps = ps(params)
        if not isinstance(ps, (list, tuple)):
            ps = (ps,)
        ps = [int(_eval_param_expr(p, params)) for p in ps] + [1] * (3 - len(ps))
        divs = []
        for d, gd in enumerate(spec.grid_div):
            if gd is None:
                divs.append(self.block[d])
            else:
                divs.append(int(_eval_param_expr(gd, params)))
        self.grid = tuple(max(1, math.ceil(ps[d] / divs[d])) for d in range(3))
        smem = 0
        if spec.smem_args and "size" in spec.smem_args:
            smem = int(_eval_param_expr(spec.smem_args["size"], params))
        self.smem = smem
        lines = [f"#define {k} {v}" for k, v in params.items()]
        lines += [f"#define {k} {_eval_param_expr(v, params) if callable(v) else v}"
                  for k, v in (spec.defines or {}).items()]
        lines.append("#define kernel_tuner 1")
        self.source = "\n".join(lines) + "\n" + spec.source


class KernelSpec:
    def __init__(self, kernel_name, kernel_source, problem_size, arguments, grid_div=(None, None, None),
                 block_size_names=None, smem_args=None, cmem_args=None, compiler_options=None,
                 defines=None):
        self.kernel_name = kernel_name
        self.source = _source_text(kernel_source)
        self.problem_size = problem_size
        self.arguments = list(arguments)
        self.grid_div = grid_div
        self.block_size_names = list(block_size_names or ("block_size_x", "block_size_y", "block_size_z"))
        self.block_size_names += ["block_size_y", "block_size_z"][len(self.block_size_names) - 1:]
        self.smem_args = smem_args
        self.cmem_args = cmem_args or {}
        self.compiler_options = list(compiler_options or [])
        self.defines = defines or {}
        self.templated = "<" in kernel_name

    def options(self) -> list:
        return ["--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo"] + self.compiler_options


class DeviceArgs:
    """Device copies of the argument list (arrays) + by-value scalars."""

    def __init__(self, dev: rt.Device, arguments: list):
        self.dev = dev
        self.host = arguments
        self.bufs: list = []
        for a in arguments:
            if isinstance(a, np.ndarray):
                arr = np.ascontiguousarray(a)
                buf = dev.alloc(max(arr.nbytes, 4))
                if arr.nbytes:
                    buf.upload(arr)
                self.bufs.append(buf)
            elif isinstance(a, (np.generic,)):
                self.bufs.append(None)
            else:
                raise ProtocolError(f"unsupported argument type {type(a).__name__}: use numpy "
                                    "arrays or numpy scalars (np.int32(...), np.float32(...))")

    def ctypes_args(self) -> list:
        out = []
        for a, b in zip(self.host, self.bufs):
            if b is not None:
                out.append(C.c_uint64(b.ptr))
            else:
                out.append(_SCALAR_CTYPES[np.dtype(a.dtype)](a.item()))
        return out

    def restore(self, i: int):
        """Re-upload argument ``i`` from its host array (Kernel Tuner semantics:
        every verified run starts from the caller's original data, so
        read-modify-write kernels and in-place updates verify correctly)."""
        b, a = self.bufs[i], self.host[i]
        if b is not None and a.nbytes:
            b.upload(np.ascontiguousarray(a))

    def download(self, i: int) -> np.ndarray:
        a = self.host[i]
        if self.bufs[i] is None:
            return a
        out = np.empty_like(np.ascontiguousarray(a))
        if out.nbytes:
            self.bufs[i].download(out)
        return out

    def free(self):
        for b in self.bufs:
            if b is not None:
                b.free()


class GenericTarget:
    """cuda-backend target for a user kernel (what tune_kernel measures)."""

    def __init__(self, spec: KernelSpec, space, dev: rt.Device, compiler: Compiler, answer=None,
                 atol: float = 1e-6, verify: Callable | None = None):
        self.spec, self.space, self.dev, self.compiler = spec, space, dev, compiler
        self.args = DeviceArgs(dev, spec.arguments)
        self.answer = answer
        self.atol = atol
        self.verify = verify
        self.answer_bufs: dict = {}
        if answer is not None:
            if len(answer) != len(spec.arguments):
                raise ProtocolError("answer must have one entry per argument (None = unchecked)")
            for i, a in enumerate(answer):
                if a is not None and verify is None and isinstance(a, np.ndarray) \
                        and a.dtype == np.float32 and self.args.bufs[i] is not None:
                    self.answer_bufs[i] = dev.to_device(np.ascontiguousarray(a))
        self.extras: dict = {}
        self.prefetch_depth = 2 * compiler.pool._max_workers
        self._pending: dict = {}

    def _compile(self, inst: KernelInstance):
        name_expr = self.spec.kernel_name if self.spec.templated else None
        key = self.compiler.cache.key(inst.source, self.spec.options(), name_expr)
        hit = self.compiler.cache.get(key)
        if hit is not None:
            return rt.CompileResult(True, hit[0], lowered=hit[1])
        res = rt.compile_source(inst.source, self.spec.options(), name_expr=name_expr)
        if res.ok:
            self.compiler.cache.put(key, res.image, res.lowered)
        return res

    def prefetch(self, configs):
        names = self.space.param_names
        for c in configs:
            k = config_key(c)
            if k in self._pending or len(self._pending) >= self.prefetch_depth:
                continue
            inst = KernelInstance(self.spec, dict(zip(names, c)))
            self._pending[k] = (inst, self.compiler.pool.submit(self._compile, inst))

    def _get(self, config):
        k = config_key(config)
        if k in self._pending:
            inst, fut = self._pending.pop(k)
            return inst, fut.result()
        inst = KernelInstance(self.spec, dict(zip(self.space.param_names, config)))
        return inst, self._compile(inst)

    def _launch(self, inst: KernelInstance, kern) -> rt.Launch:
        return rt.Launch(kern, inst.grid, inst.block, self.args.ctypes_args(), smem=inst.smem)

    def _load(self, inst, res):
        rc, mod = self.dev.load(res.image)
        if rc != rt.OK:
            return None, None, Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(mod))
        for sym, data in self.spec.cmem_args.items():
            if mod.set_constant(sym, np.ascontiguousarray(data)) != rt.OK:
                mod.unload()
                return None, None, Observation(Status.RUNTIME_FAILED, detail=rt.last_error())
        name = res.lowered or self.spec.kernel_name
        try:
            kern = mod.function(name)
        except Exception as e:  # noqa: BLE001 -- missing kernel symbol is a config failure
            mod.unload()
            return None, None, Observation(Status.COMPILE_FAILED, detail=str(e))
        if inst.smem > 48 * 1024 and kern.set_max_dynamic_smem(inst.smem) != rt.OK:
            mod.unload()
            return None, None, Observation(Status.INVALID, detail=rt.last_error())
        return mod, kern, None

    def _check(self, info) -> str | None:
        """Verify outputs of the last run; returns a failure message or None."""
        if self.answer is None:
            return None
        results = []
        for i, a in enumerate(self.answer):
            if a is None:
                results.append(None)
                continue
            if i in self.answer_bufs:
                n = self.answer[i].size
                cmp = self.dev.compare(self.args.bufs[i], self.answer_bufs[i], n, 1e-5, self.atol)
                info.setdefault("verify", []).append(cmp)
                if cmp["n_bad"]:
                    return (f"argument {i}: {cmp['n_bad']} elements differ "
                            f"(max_abs_err={cmp['max_abs_err']:.3e}, atol={self.atol:g})")
                results.append(None)
            else:
                results.append(self.args.download(i))
        if self.verify is not None:
            full = [r if r is not None else (self.args.download(i) if self.answer[i] is not None else None)
                    for i, r in enumerate(results)]
            ok = self.verify(self.answer, full, atol=self.atol)
            return None if ok else "custom verify() rejected the output"
        for i, r in enumerate(results):
            if r is not None and not np.allclose(self.answer[i], r, atol=self.atol):
                return f"argument {i}: output differs from answer (atol={self.atol:g})"
        return None

    def execute(self, config, protocol: MeasurementProtocol) -> Observation:
        if self.dev.poisoned:
            from .cuda_backend import DevicePoisoned

            raise DevicePoisoned(self.dev.index)
        inst, res = self._get(config)
        if not res.ok:
            return Observation(Status.COMPILE_FAILED, detail=(res.error or res.log)[-2000:])
        mod, kern, bad = self._load(inst, res)
        if bad is not None:
            return bad
        info: dict = {"grid": inst.grid, "block": inst.block}
        try:
            launch = [self._launch(inst, kern)]
            if self.answer is not None:
                for i in range(len(self.args.bufs)):
                    self.args.restore(i)
                rc, err = self.dev.run(launch, protocol.timeout_ms)
                if rc != rt.OK:
                    return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=err)
                msg = self._check(info)
                if msg:
                    return Observation(Status.RUNTIME_FAILED, detail=f"verification failed: {msg}")
            rc, times = self.dev.run_timed(launch, protocol.warmup_runs, protocol.benchmark_runs,
                                           protocol.flush_l2, protocol.timeout_ms)
            if rc != rt.OK:
                return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(times))
            info.update(kern.attrs())
        finally:
            mod.unload()
            self.extras[config_key(config)] = info
        return Observation(Status.OK, tuple(times), aggregate_times(protocol, times))

    def run_once(self, config) -> list:
        inst, res = self._get(config)
        if not res.ok:
            raise ProtocolError(f"compilation failed:\n{res.error}\n{res.log}")
        mod, kern, bad = self._load(inst, res)
        if bad is not None:
            raise ProtocolError(f"{bad.status.value}: {bad.detail}")
        try:
            rc, err = self.dev.run([self._launch(inst, kern)])
            if rc != rt.OK:
                raise ProtocolError(f"launch failed: {err}")
            return [self.args.download(i) for i in range(len(self.spec.arguments))]
        finally:
            mod.unload()

    def close(self):
        self.args.free()
        for b in self.answer_bufs.values():
            b.free()


_DEVICES: dict = {}


def _device(index: int) -> rt.Device:
    if index not in _DEVICES:
        _DEVICES[index] = rt.Device(index)
    return _DEVICES[index]


def run_kernel(kernel_name, kernel_source, problem_size, arguments, params, grid_div_x=None,
               grid_div_y=None, grid_div_z=None, lang=None, device=0, platform=0, smem_args=None,
               cmem_args=None, texmem_args=None, compiler=None, compiler_options=None, defines=None,
               block_size_names=None, quiet=False, log=None) -> list:
    """Compile and run ONE configuration; return every argument's device value."""
    if lang not in (None, "CUDA", "cupy", "cuda"):
        raise ProtocolError(f"lang={lang!r}: only CUDA (sm_100a) is supported")
    if texmem_args:
        raise ProtocolError("texmem_args are not supported on this backend")
    spec = KernelSpec(kernel_name, kernel_source, problem_size, arguments,
                      (grid_div_x, grid_div_y, grid_div_z), block_size_names, smem_args, cmem_args,
                      compiler_options, defines)
    space = space_from_tune_params(kernel_name, {k: [v] for k, v in params.items()})
    dev = _device(device)
    comp = Compiler(workers=1)
    tgt = GenericTarget(spec, space, dev, comp)
    try:
        return tgt.run_once(tuple(params.values()))
    finally:
        tgt.close()
        comp.shutdown()


def tune_kernel(kernel_name, kernel_source, problem_size, arguments, tune_params, grid_div_x=None,
                grid_div_y=None, grid_div_z=None, restrictions=None, answer=None, atol=1e-6,
                verify=None, verbose=False, lang=None, device=0, platform=0, smem_args=None,
                cmem_args=None, texmem_args=None, compiler=None, compiler_options=None, defines=None,
                log=None, iterations=7, block_size_names=None, quiet=False, strategy=None,
                strategy_options=None, cache=None, metrics=None, simulation_mode=False,
                observers=None, objective=None, objective_higher_is_better=None):
    """Tune ``kernel_name`` over ``tune_params`` on a B200; returns (results, env)."""
    if lang not in (None, "CUDA", "cupy", "cuda"):
        raise ProtocolError(f"lang={lang!r}: only CUDA (sm_100a) is supported")
    if texmem_args:
        raise ProtocolError("texmem_args are not supported on this backend")
    if simulation_mode:
        raise ProtocolError("simulation_mode: use the simulated backend with a recorded cache")
    opts = dict(strategy_options or {})
    spec = KernelSpec(kernel_name, kernel_source, problem_size, arguments,
                      (grid_div_x, grid_div_y, grid_div_z), block_size_names, smem_args, cmem_args,
                      compiler_options, defines)
    space = space_from_tune_params(kernel_name, tune_params, restrictions)
    dev = _device(device)
    comp = Compiler()
    target = GenericTarget(spec, space, dev, comp, answer=answer, atol=atol, verify=verify)
    backend = BackendDescriptor(kind="cuda", target=target)
    protocol = MeasurementProtocol(warmup_runs=1, benchmark_runs=int(iterations),
                                   flush_l2=bool(opts.get("flush_l2", True)))
    name = (strategy or "brute_force").lower()
    if name not in STRATEGIES:
        raise ProtocolError(f"unknown strategy {strategy!r}; choose from {sorted(STRATEGIES)}")
    seed = int(opts.get("seed", 0))
    size = space.space_size()
    budget = int(opts.get("max_fevals", 0)) or (max(1, int(size * float(opts["fraction"])))
                                                if "fraction" in opts else None)
    t0 = time.perf_counter()
    try:
        if name == "brute_force":
            result, _ = STRATEGIES[name](space, backend, protocol)
        elif name in ("random_sample", "random"):
            result = STRATEGIES[name](space, backend, protocol, budget=budget or size, seed=seed)
        elif name in ("genetic_algorithm", "genetic"):
            result = STRATEGIES[name](space, backend, protocol, budget=budget or min(size, 1000),
                                      seed=seed, popsize=int(opts.get("popsize", 20)),
                                      maxiter=int(opts.get("maxiter", 100)),
                                      mutation_chance=int(opts.get("mutation_chance", 10)))
        else:
            result = STRATEGIES[name](space, backend, protocol, budget=budget or size, seed=seed)
    finally:
        elapsed = time.perf_counter() - t0
    results = []
    for config, obs in result.trace:
        params = dict(zip(space.param_names, config))
        row: dict[str, Any] = dict(params)
        row["status"] = obs.status.value
        if obs.ok:
            row["time"] = obs.time_ms
            row["times"] = list(obs.times_ms)
            if metrics:
                env_p = dict(params)
                env_p["time"] = obs.time_ms
                for mname, fn in metrics.items():
                    row[mname] = fn(env_p) if callable(fn) else ex.evaluate(ex.parse_expression(fn), env_p)
                    env_p[mname] = row[mname]
        else:
            row["time"] = {"compile_failed": "CompilationFailedConfig", "invalid": "InvalidConfig",
                           "timeout": "TimeoutConfig"}.get(obs.status.value, "RuntimeFailedConfig")
            row["error"] = obs.detail
        row.update({k: v for k, v in target.extras.get(config_key(config), {}).items()
                    if k in ("regs", "local_bytes")})
        results.append(row)
    env = {"device_name": dev.info["name"], "compute_capability": f"{dev.info['cc_major']}{dev.info['cc_minor']}",
           "iterations": iterations, "compiler_options": spec.options(), "problem_size": problem_size,
           "kernel_name": kernel_name, "tune_params": tune_params, "strategy": name,
           "space_size": size, "evaluations": result.evaluations_used, "notes": list(result.notes),
           "best_config": dict(zip(space.param_names, result.best)) if result.best else None,
           "best_time_ms": result.best_observation.time_ms if result.best_observation else None,
           "total_time_s": elapsed, "nvrtc": "%d.%d" % rt.nvrtc_version(),
           "compile_stats": dict(comp.stats)}
    if cache:
        tc = result_to_cache(space, result, dev.info["name"])
        write_kernel_tuner_cache(tc, cache, space, target.extras)
    target.close()
    comp.shutdown()
    if not quiet and verbose:
        for r in results:
            print(r)
    return results, env
