"""In-process B200 executor behind the ``cuda`` backend kind.

One :class:`CudaTarget` = one problem instance resident in HBM on one
GPU.  ``execute(config, protocol)`` is the B200 replacement of the
reference's ``command_execute`` (`pkg/src/tunescape/measure.py:218-305`):

1. NVRTC -> sm_100a cubin (host compile pool + on-disk cubin cache),
   failure -> ``compile_failed`` with the NVRTC log in ``detail``;
2. ``cuModuleLoadData``, ``__constant__`` upload, dynamic-smem opt-in,
   failure -> ``invalid``;
3. warmup + benchmark runs in ONE native call, per-run CUDA events on
   the launch stream, optional L2 flush outside the events; a rejected
   launch -> ``invalid``, a device fault -> ``runtime_failed`` (the
   context is poisoned: every later configuration raises
   :class:`DevicePoisoned` instead of recording a fake failure, so the sweep
   stops, nothing unmeasured reaches the cache or the resume log, and a
   restarted process -- a fresh context -- measures the rest), the
   watchdog -> ``timeout``;
4. on-device verification against the answer buffer (no D2H of the
   output), mismatch -> ``runtime_failed`` with the error in ``detail``.

Compilation is pipelined: :meth:`prefetch` queues configurations on a
thread pool (ctypes releases the GIL, NVRTC is thread-safe) while the
GPU times earlier ones.
"""

from __future__ import annotations

import os
import threading
import time
from collections import OrderedDict
from concurrent.futures import Future, ThreadPoolExecutor

import numpy as np

from . import runtime as rt
from .errors import DeviceError
from .measure import MeasurementProtocol, Observation, Status, aggregate_times
from .paramspace import config_key

_RC_STATUS = {rt.ERR_COMPILE: Status.COMPILE_FAILED, rt.ERR_INVALID: Status.INVALID,
              rt.ERR_RUNTIME: Status.RUNTIME_FAILED, rt.ERR_TIMEOUT: Status.TIMEOUT,
              rt.ERR_ARG: Status.INVALID}


class DevicePoisoned(DeviceError):
    """A device fault poisoned this process's CUDA context: no further
    configuration can be measured in it (restart the worker; ``--resume``
    re-measures everything not yet logged)."""

    def __init__(self, index: int):
        super().__init__(f"CUDA context of device {index} poisoned by an earlier fault; "
                         "restart the worker (with --resume) to measure the remaining configurations")


def default_workers() -> int:
    env = os.environ.get("TSG_COMPILE_WORKERS")
    if env:
        return max(1, int(env))
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    # one process per GPU: the node's host threads are shared by the ranks on
    # it (torchrun's LOCAL_WORLD_SIZE), one left for the drivers' main threads
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(1, (n - 1) // local)


class Compiler:
    """Thread pool + cubin cache; futures resolve to CompileResult."""

    def __init__(self, workers: int | None = None, cache: rt.CubinCache | None = None):
        self.pool = ThreadPoolExecutor(max_workers=workers or default_workers(),
                                       thread_name_prefix="nvrtc")
        self.cache = cache if cache is not None else rt.CubinCache()
        self._inflight: dict = {}
        self._lock = threading.Lock()
        # finished compilations kept in memory (a configuration measured again
        # -- e2e pass, re-tune -- skips the disk cache and the pool round trip)
        self._done: "OrderedDict[str, Future]" = OrderedDict()
        self.memory_entries = 1024
        self.stats = {"compiled": 0, "cache_hits": 0, "compile_s": 0.0, "failed": 0}

    def _job(self, source: str, options: list, key: str) -> rt.CompileResult:
        hit = self.cache.get(key)
        if hit is not None:
            with self._lock:
                self.stats["cache_hits"] += 1
            return rt.CompileResult(True, hit[0], lowered=hit[1])
        res = rt.compile_source(source, options)
        with self._lock:
            self.stats["compiled"] += 1
            self.stats["compile_s"] += res.seconds
            if not res.ok:
                self.stats["failed"] += 1
        if res.ok:
            self.cache.put(key, res.image, res.lowered)
        return res

    def submit(self, source: str, options: list) -> Future:
        key = self.cache.key(source, options, None)
        with self._lock:
            done = self._done.get(key)
            if done is not None:
                self._done.move_to_end(key)
                return done
            fut = self._inflight.get(key)
            if fut is None:
                fut = self.pool.submit(self._job, source, options, key)
                self._inflight[key] = fut
                fut.add_done_callback(lambda _f, k=key: self._drop(k))
        return fut

    def _drop(self, key):
        with self._lock:
            fut = self._inflight.pop(key, None)
            if fut is not None and not fut.cancelled() and fut.exception() is None:
                self._done[key] = fut
                while len(self._done) > self.memory_entries:
                    self._done.popitem(last=False)

    def compile(self, source: str, options: list) -> rt.CompileResult:
        return self.submit(source, options).result()

    def shutdown(self):
        self.pool.shutdown(wait=False, cancel_futures=True)


class CudaTarget:
    """A problem instance resident on one GPU, measurable per config."""

    def __init__(self, problem, device: rt.Device | int | None = None,
                 compiler: Compiler | None = None, verify: bool = True,
                 answer: np.ndarray | None = None, prefetch_depth: int | None = None):
        self.problem = problem
        if device is None or isinstance(device, int):
            device = rt.Device(device or 0)
        self.dev = device
        self.compiler = compiler or Compiler()
        self.verify = verify
        self.source = problem.source()
        self.bufs = {}
        for spec in problem.buffers():
            buf = self.dev.alloc(spec.nbytes)
            if spec.init is not None:
                buf.upload(spec.init)
            self.bufs[spec.name] = buf
        self.out = self.bufs[problem.output_name]
        self.n_out = problem.output_count
        self.answer_buf = None
        if verify:
            self.answer_buf = self.dev.alloc(self.n_out * 4)
            if answer is not None:
                self.answer_buf.upload(np.ascontiguousarray(answer, dtype=np.float32))
            else:
                self._compute_answer()
        self.extras: dict = {}
        # modules of measured configurations are unloaded in batches (flush_
        # modules / close), not inside the per-configuration protocol: a
        # cuModuleUnload of a large module occasionally blocks ~0.1-0.6 s in
        # the driver (measured on B200), which would land inside a sweep
        self._retired: list = []
        self.retire_cap = 256
        # modules of upcoming configurations are loaded by one helper thread
        # while the GPU runs the current one (ctypes releases the GIL): an
        # eager cuModuleLoadData occasionally blocks 10-100 ms in the driver
        self._loader = ThreadPoolExecutor(max_workers=1, thread_name_prefix="modload")
        self._preloaded: dict = {}
        self.preload_depth = 2
        self._pending: "OrderedDict[str, Future]" = OrderedDict()
        self.prefetch_depth = prefetch_depth or 4 * self.compiler.pool._max_workers
        self.stats = {"executed": 0, "gpu_ms": 0.0, "verify_failed": 0}
        self._slots_inflight: list = []  # execute_many: enqueued, not yet collected
        # configurations enqueued at once (<= rt.SLOTS); TSG_PIPELINE_DEPTH overrides
        self.pipeline_depth = int(os.environ.get("TSG_PIPELINE_DEPTH", "4"))

    # -- answer ------------------------------------------------------------------
    def _load(self, image: bytes):
        rc, mod = self.dev.load(image)
        if rc != rt.OK:
            raise DeviceError(f"cannot load module: {mod}")
        for sym, data in self.problem.constants().items():
            rc = mod.set_constant(sym, data)
            if rc != rt.OK:
                raise DeviceError(f"cannot set constant {sym}: {rt.last_error()}")
        return mod

    def _compute_answer(self):
        res = self.compiler.compile(self.source, self.problem.options(None) + ["-DREFERENCE_ONLY=1"])
        if not res.ok:
            raise DeviceError(f"reference kernel failed to compile:\n{res.error}")
        mod = self._load(res.image)
        try:
            kern = mod.function(self.problem.reference_kernel)
            bufs = dict(self.bufs)
            bufs[self.problem.output_name] = self.answer_buf
            launches = self.problem.reference_launches(kern, bufs)
            rc, err = self.dev.run(launches, timeout_ms=600_000)
            if rc != rt.OK:
                raise DeviceError(f"reference kernel failed: {err}")
        finally:
            mod.unload()

    def answer(self) -> np.ndarray:
        out = np.empty(self.n_out, dtype=np.float32)
        return self.answer_buf.download(out)

    # -- compile pipeline ------------------------------------------------------------
    def _options(self, cfg: dict) -> list:
        return self.problem.options(cfg)

    def source_for(self, cfg: dict) -> str:
        """Kernel source of one configuration (some problems generate code per config)."""
        return self.problem.source_for(cfg, self.source)

    def prefetch(self, configs) -> None:
        """Queue compilation of upcoming configurations (bounded window)."""
        names = self.problem.space.param_names
        for config in configs:
            if len(self._pending) >= self.prefetch_depth:
                break
            key = config_key(config)
            if key not in self._pending:
                cfg = dict(zip(names, config))
                self._pending[key] = self.compiler.submit(self.source_for(cfg), self._options(cfg))

    def preload(self, configs) -> None:
        """Load the modules of the next ``preload_depth`` configurations in the
        background (their compilation must already be queued by prefetch)."""
        for config in configs[: self.preload_depth]:
            key = config_key(config)
            if key in self._preloaded or key not in self._pending:
                continue
            fut = self._pending[key]
            self._preloaded[key] = self._loader.submit(self._load_when_compiled, fut)

    def _load_when_compiled(self, fut: Future):
        res = fut.result()
        if not res.ok:
            return None
        return self.dev.load(res.image)

    def _compiled(self, key: str, cfg: dict) -> rt.CompileResult:
        fut = self._pending.pop(key, None)
        if fut is None:
            fut = self.compiler.submit(self.source_for(cfg), self._options(cfg))
        return fut.result()

    # -- the protocol ------------------------------------------------------------------
    def execute(self, config, protocol: MeasurementProtocol) -> Observation:
        if self.dev.poisoned:
            raise DevicePoisoned(self.dev.index)
        names = self.problem.space.param_names
        cfg = dict(zip(names, config))
        key = config_key(config)
        info = {}
        t0 = time.perf_counter()
        res = self._compiled(key, cfg)
        info["compile_wait_s"] = time.perf_counter() - t0
        if not res.ok:
            return Observation(Status.COMPILE_FAILED, detail=(res.error or res.log)[-2000:])
        t1 = time.perf_counter()
        pre = self._preloaded.pop(key, None)
        loaded = pre.result() if pre is not None else None
        rc, mod = loaded if loaded is not None else self.dev.load(res.image)
        if rc != rt.OK:
            return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(mod))
        info["t_load_s"] = time.perf_counter() - t1
        info["preloaded"] = pre is not None
        try:
            for sym, data in self.problem.constants().items():
                if mod.set_constant(sym, data) != rt.OK:
                    return Observation(Status.RUNTIME_FAILED, detail=rt.last_error())
            kern = mod.function(self.problem.kernel_name)
            smem = self.problem.smem_bytes(cfg)
            if smem > 48 * 1024:
                if kern.set_max_dynamic_smem(smem) != rt.OK:
                    return Observation(Status.INVALID, detail=rt.last_error())
            if smem > 0:
                kern.set_smem_carveout(100)  # occupancy limited by smem use, not a default carveout
            # register/static-smem attributes are read in batch when the module
            # is retired (flush_modules): fewer driver calls per configuration
            info["smem_bytes"] = smem
            launches = self.problem.launches(cfg, kern, self.bufs)
            t2 = time.perf_counter()
            info["t_setup_s"] = t2 - t1 - info["t_load_s"]
            if self.verify:
                # poison the output so a kernel that skips elements fails
                self.dev._check(self.dev.lib.tsg_memset32(self.dev.ctx, self.out.ptr,
                                                          0x7FC00000, self.n_out))
            rc, times = self.dev.run_timed(launches, protocol.warmup_runs,
                                           protocol.benchmark_runs, protocol.flush_l2,
                                           protocol.timeout_ms)
            if rc != rt.OK:
                return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(times))
            t3 = time.perf_counter()
            info["t_run_s"] = t3 - t2
            info["launch_ms"] = self.dev.last_launch_times(len(launches))
            info["n_launches"] = len(launches)
            if self.verify:
                cmp = self.dev.compare(self.out, self.answer_buf, self.n_out,
                                       self.problem.rtol, self.problem.atol)
                info["verify"] = cmp
                rel = cmp["max_abs_err"] / cmp["max_abs_ref"] if cmp["max_abs_ref"] > 0 else \
                    cmp["max_abs_err"]
                info["verify_rel_err"] = rel
                abs_tol = getattr(self.problem, "abs_tol", None)
                bad = (cmp["max_abs_err"] > abs_tol) if abs_tol is not None else (rel > self.problem.rtol)
                if cmp["n_nonfinite"] or bad:
                    self.stats["verify_failed"] += 1
                    return Observation(
                        Status.RUNTIME_FAILED,
                        detail=(f"verification failed: max_abs_err={cmp['max_abs_err']:.3e} "
                                f"max_abs_ref={cmp['max_abs_ref']:.3e} "
                                f"nonfinite={cmp['n_nonfinite']} bad={cmp['n_bad']}"),
                    )
        finally:
            t4 = time.perf_counter()
            self._retire(mod, key, self.problem.kernel_name)
            info["t_unload_s"] = time.perf_counter() - t4
            info["t_total_s"] = time.perf_counter() - t0
            self.extras[key] = info
        self.stats["executed"] += 1
        self.stats["gpu_ms"] += sum(times)
        return Observation(Status.OK, times_ms=tuple(times),
                           time_ms=aggregate_times(protocol, times))

    # -- pipelined protocol (same measurement, no idle device between configs) --
    def _prepare(self, config, info: dict):
        """Compile wait, module, constants, smem opt-in, launch list: the
        host-side part of one configuration.  Returns (mod, launches) or an
        Observation for a configuration that fails before any launch."""
        cfg = dict(zip(self.problem.space.param_names, config))
        key = config_key(config)
        t0 = time.perf_counter()
        res = self._compiled(key, cfg)
        info["compile_wait_s"] = time.perf_counter() - t0
        if not res.ok:
            return Observation(Status.COMPILE_FAILED, detail=(res.error or res.log)[-2000:])
        t1 = time.perf_counter()
        pre = self._preloaded.pop(key, None)
        loaded = pre.result() if pre is not None else None
        rc, mod = loaded if loaded is not None else self.dev.load(res.image)
        if rc != rt.OK:
            return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(mod))
        info["t_load_s"] = time.perf_counter() - t1
        info["preloaded"] = pre is not None
        for sym, data in self.problem.constants().items():
            if mod.set_constant(sym, data) != rt.OK:
                self._retire(mod, key, self.problem.kernel_name)
                return Observation(Status.RUNTIME_FAILED, detail=rt.last_error())
        kern = mod.function(self.problem.kernel_name)
        smem = self.problem.smem_bytes(cfg)
        if smem > 48 * 1024 and kern.set_max_dynamic_smem(smem) != rt.OK:
            self._retire(mod, key, self.problem.kernel_name)
            return Observation(Status.INVALID, detail=rt.last_error())
        if smem > 0:
            kern.set_smem_carveout(100)
        info["smem_bytes"] = smem
        launches = self.problem.launches(cfg, kern, self.bufs)
        info["t_setup_s"] = time.perf_counter() - t1 - info["t_load_s"]
        return mod, launches

    def _verdict(self, cmp: dict, info: dict) -> Observation | None:
        """Verification outcome (None = passed) of an on-device comparison."""
        info["verify"] = cmp
        rel = cmp["max_abs_err"] / cmp["max_abs_ref"] if cmp["max_abs_ref"] > 0 else cmp["max_abs_err"]
        info["verify_rel_err"] = rel
        abs_tol = getattr(self.problem, "abs_tol", None)
        bad = (cmp["max_abs_err"] > abs_tol) if abs_tol is not None else (rel > self.problem.rtol)
        if cmp["n_nonfinite"] or bad:
            self.stats["verify_failed"] += 1
            return Observation(
                Status.RUNTIME_FAILED,
                detail=(f"verification failed: max_abs_err={cmp['max_abs_err']:.3e} "
                        f"max_abs_ref={cmp['max_abs_ref']:.3e} "
                        f"nonfinite={cmp['n_nonfinite']} bad={cmp['n_bad']}"),
            )
        return None

    def execute_many(self, configs, protocol: MeasurementProtocol, on_config=None):
        """Measure ``configs`` in order; yields (config, Observation) in order.

        Same protocol and measurement as :meth:`execute` (per-run CUDA
        events around each run on the one stream, L2 flush outside them,
        on-device verification), but pipelined through the C ABI's
        submission slots (tsg_submit_timed / tsg_collect): up to
        ``pipeline_depth`` configurations are enqueued at once, and
        configuration i+1 is compile-waited, loaded, set up and ENQUEUED
        before the host waits for the oldest one, so the device never idles
        between configurations.  Compilation prefetch and module preload
        run ahead as in :meth:`execute`.  ``on_config(i)`` (optional) is
        called before each configuration is prepared (bench: clock
        sampling).
        """
        configs = list(configs)

        def finish(p):
            config, key, mod, n_launch, info, sl, t0 = p
            try:
                rc, times, lt, cmp = self.dev.collect(sl, protocol.benchmark_runs, n_launch, protocol.timeout_ms)
                info["t_run_s"] = time.perf_counter() - info["_t_submit"]
                info["t_abs_submit"] = info.pop("_t_submit")  # host timeline (bench --dump)
                info["t_abs_collected"] = time.perf_counter()
                if rc != rt.OK:
                    return Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=str(times))
                info["launch_ms"] = lt
                info["n_launches"] = n_launch
                tl = self.dev.slot_timeline(sl)
                if tl is not None:  # device timeline (ms): bench --dump
                    info["t_dev_start_ms"], info["t_dev_end_ms"], info["t_dev_warmup_ms"] = tl
                if self.verify:
                    bad = self._verdict(cmp, info)
                    if bad is not None:
                        return bad
                self.stats["executed"] += 1
                self.stats["gpu_ms"] += sum(times)
                return Observation(Status.OK, times_ms=tuple(times), time_ms=aggregate_times(protocol, times))
            finally:
                self._retire(mod, key, self.problem.kernel_name)
                info["t_total_s"] = time.perf_counter() - t0
                self.extras[key] = info

        try:
            yield from self._pipeline(configs, protocol, on_config, finish)
        finally:
            # a consumer that stops early leaves no slot in flight
            for p in self._slots_inflight:
                if p[0] == "pending":
                    finish(p[2])
            self._slots_inflight = []

    def _pipeline(self, configs, protocol, on_config, finish):
        # FIFO of ("pending", config, state) / ("done", config, Observation):
        # results leave in input order; up to pipeline_depth configurations
        # are enqueued on the device at once (absorbs host hiccups longer
        # than one configuration's device time)
        fifo = self._slots_inflight = []
        free = list(range(rt.SLOTS))
        depth = max(1, min(self.pipeline_depth, rt.SLOTS))

        def n_pending():
            return sum(1 for e in fifo if e[0] == "pending")

        def drain(limit):
            while fifo and (fifo[0][0] == "done" or n_pending() > limit):
                kind, config, x = fifo.pop(0)
                if kind == "pending":
                    free.append(x[5])
                    yield config, finish(x)
                else:
                    yield config, x

        for i, config in enumerate(configs):
            if i % 4 == 0:
                self.prefetch(configs[i:])
            self.preload(configs[i + 1:])
            if on_config is not None:
                on_config(i)
            yield from drain(depth - 1)  # a slot is free
            key = config_key(config)
            info: dict = {"pipelined": True}
            t0 = time.perf_counter()
            info["t_abs_prepare"] = t0
            immediate = None
            if self.dev.poisoned:
                raise DevicePoisoned(self.dev.index)
            else:
                prep = self._prepare(config, info)
                if isinstance(prep, Observation):
                    immediate = prep
                else:
                    mod, launches = prep
                    slot = free.pop(0)
                    info["_t_submit"] = time.perf_counter()
                    rc, err = self.dev.submit_timed(slot, launches, protocol.warmup_runs, protocol.benchmark_runs,
                                                    protocol.flush_l2, self.out if self.verify else None,
                                                    self.n_out, self.answer_buf if self.verify else None,
                                                    self.problem.rtol, self.problem.atol)
                    if rc != rt.OK:
                        free.append(slot)
                        info.pop("_t_submit", None)
                        self._retire(mod, key, self.problem.kernel_name)
                        self.extras[key] = info
                        immediate = Observation(_RC_STATUS.get(rc, Status.RUNTIME_FAILED), detail=err)
                    else:
                        fifo.append(("pending", config, (config, key, mod, len(launches), info, slot, t0)))
            if immediate is not None:
                self.extras.setdefault(key, info)
                fifo.append(("done", config, immediate))
            yield from drain(depth - 1)
        yield from drain(-1)

    def run_output(self, config, out: np.ndarray | None = None) -> tuple:
        """Run one configuration once and return (Observation-like status, host output).

        ``out`` (optional): a float32 host array of ``output_count`` elements
        to download into (e.g. page-locked memory: no staging copy)."""
        names = self.problem.space.param_names
        cfg = dict(zip(names, config))
        res = self._compiled(config_key(config), cfg)
        if not res.ok:
            return Status.COMPILE_FAILED, res.error
        mod = self._load(res.image)
        try:
            kern = mod.function(self.problem.kernel_name)
            smem = self.problem.smem_bytes(cfg)
            if smem > 48 * 1024 and kern.set_max_dynamic_smem(smem) != rt.OK:
                return Status.INVALID, rt.last_error()
            if smem > 0:
                kern.set_smem_carveout(100)
            self.dev._check(self.dev.lib.tsg_memset32(self.dev.ctx, self.out.ptr, 0x7FC00000,
                                                      self.n_out))
            rc, err = self.dev.run(self.problem.launches(cfg, kern, self.bufs))
            if rc != rt.OK:
                return _RC_STATUS.get(rc, Status.RUNTIME_FAILED), err
            if out is None:
                out = np.empty(self.n_out, dtype=np.float32)
            self.out.download(out)
            return Status.OK, out
        finally:
            self._retire(mod)

    def _retire(self, mod, key: str | None = None, kernel_name: str | None = None) -> None:
        self._retired.append((mod, key, kernel_name))
        if len(self._retired) >= self.retire_cap:
            self.flush_modules()

    def collect_attrs(self) -> None:
        """Fill ``extras[key]`` with register/smem attributes of retired modules."""
        for mod, key, name in self._retired:
            if key is not None and name and "regs" not in self.extras.get(key, {}):
                try:
                    self.extras.setdefault(key, {}).update(mod.function(name).attrs())
                except Exception:  # noqa: BLE001 -- attributes are diagnostics
                    pass

    def flush_modules(self) -> None:
        """Unload the modules of already-measured configurations."""
        self.collect_attrs()
        for mod, _, _ in self._retired:
            mod.unload()
        self._retired.clear()

    def close(self):
        self._loader.shutdown(wait=True)
        for fut in self._preloaded.values():  # preloaded but never executed
            r = fut.result()
            if r is not None and r[0] == rt.OK:
                r[1].unload()
        self._preloaded.clear()
        self.flush_modules()
        for b in self.bufs.values():
            b.free()
        if self.answer_buf:
            self.answer_buf.free()
