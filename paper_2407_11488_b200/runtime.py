"""ctypes binding of ``libtsgpu.so`` (the C ABI in ``include/tsgpu.h``).

This is the "thin C-ABI layer" of the north_star: NVRTC compile to
sm_100a, module load, launch, CUDA-event timing, on-device compare.
There is no fallback: if the library or a GPU is missing, every entry
point raises :class:`DeviceError` -- the tuner never silently measures
something else.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DeviceError, ProtocolError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libtsgpu.so"

OK, ERR_COMPILE, ERR_INVALID, ERR_RUNTIME, ERR_TIMEOUT, ERR_SETUP, ERR_ARG = range(7)
ARCH = "sm_100a"


class LaunchT(C.Structure):
    _fields_ = [
        ("fn", C.c_void_p),
        ("grid", C.c_uint * 3),
        ("block", C.c_uint * 3),
        ("cluster", C.c_uint * 3),
        ("smem_bytes", C.c_uint),
        ("flags", C.c_uint),  # TSG_LAUNCH_PDL
        ("args", C.POINTER(C.c_void_p)),
    ]


class DeviceInfoT(C.Structure):
    _fields_ = [
        ("name", C.c_char * 256),
        ("cc_major", C.c_int),
        ("cc_minor", C.c_int),
        ("sm_count", C.c_int),
        ("max_threads_per_block", C.c_int),
        ("max_smem_per_block_optin", C.c_int),
        ("max_smem_per_sm", C.c_int),
        ("l2_bytes", C.c_int),
        ("regs_per_sm", C.c_int),
        ("clock_khz", C.c_int),
        ("mem_clock_khz", C.c_int),
        ("mem_bus_bits", C.c_int),
        ("total_mem", C.c_size_t),
    ]


# name -> (restype, argtypes); the symbol list doubles as the export check
SIGNATURES = {
    "tsg_last_error": (C.c_char_p, []),
    "tsg_error_string": (C.c_char_p, [C.c_int]),
    "tsg_nvrtc_version": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "tsg_driver_version": (C.c_int, [C.POINTER(C.c_int)]),
    "tsg_init": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "tsg_destroy": (C.c_int, [C.c_void_p]),
    "tsg_device_info": (C.c_int, [C.c_void_p, C.POINTER(DeviceInfoT)]),
    "tsg_launch_count": (C.c_uint64, [C.c_void_p]),
    "tsg_compile": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int,
                              C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
                              C.c_char_p, C.c_size_t]),
    "tsg_free_host": (None, [C.c_void_p]),
    "tsg_module_load": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "tsg_module_unload": (C.c_int, [C.c_void_p]),
    "tsg_get_function": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "tsg_set_constant": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "tsg_func_attrs": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_int)] * 4),
    "tsg_set_max_dynamic_smem": (C.c_int, [C.c_void_p, C.c_int]),
    "tsg_set_smem_carveout": (C.c_int, [C.c_void_p, C.c_int]),
    "tsg_occupancy": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "tsg_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]),
    "tsg_free": (C.c_int, [C.c_void_p, C.c_uint64]),
    "tsg_h2d": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_size_t]),
    "tsg_d2h": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_size_t]),
    "tsg_d2d": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_size_t]),
    "tsg_memset32": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_size_t]),
    "tsg_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "tsg_host_unregister": (C.c_int, [C.c_void_p]),
    "tsg_run": (C.c_int, [C.c_void_p, C.POINTER(LaunchT), C.c_int, C.c_double]),
    "tsg_run_timed": (C.c_int, [C.c_void_p, C.POINTER(LaunchT), C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_double, C.POINTER(C.c_float)]),
    "tsg_last_launch_times": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_int]),
    "tsg_event_record": (C.c_int, [C.c_void_p, C.c_int]),
    "tsg_tma_encode_2d_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_uint32, C.c_uint32, C.c_int]),
    "tsg_event_elapsed": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "tsg_compare_f32": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_size_t, C.c_double,
                                  C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "tsg_submit_timed": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(LaunchT), C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_uint64, C.c_size_t, C.c_uint64, C.c_double, C.c_double]),
    "tsg_collect": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.POINTER(C.c_float), C.POINTER(C.c_float),
                              C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)]),
    "tsg_slot_reset": (C.c_int, [C.c_void_p, C.c_int]),
    "tsg_slot_timeline": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_float)]),
    "tsg_set_flush_bytes": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t]),
    "tsg_stream_handle": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "tsg_stream_wait": (C.c_int, [C.c_void_p, C.c_uint64]),
    "tsg_stream_signal": (C.c_int, [C.c_void_p, C.c_uint64]),
    "tsg_launch_async": (C.c_int, [C.c_void_p, C.POINTER(LaunchT), C.c_int]),
    "tsg_copy_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_size_t]),
    "tsg_sync": (C.c_int, [C.c_void_p, C.c_double]),
}

SLOTS = 16  # include/tsgpu.h TSG_SLOTS (pipelined submission slots)
LAUNCH_PDL = 1  # include/tsgpu.h TSG_LAUNCH_PDL

_lib = None
_lib_lock = threading.Lock()


# Modules are loaded eagerly (all kernels at cuModuleLoadData) unless the user
# chose otherwise: the tuning loop then pays the code upload in one predictable
# call instead of inside the first function lookup / launch.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")


def load_library(path: Path | str | None = None):
    """Load libtsgpu.so (raises DeviceError when it is absent)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"native library {p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    return load_library().tsg_last_error().decode(errors="replace")


class CompileResult:
    __slots__ = ("ok", "image", "log", "lowered", "error", "seconds")

    def __init__(self, ok, image=b"", log="", lowered="", error="", seconds=0.0):
        self.ok, self.image, self.log, self.lowered, self.error = ok, image, log, lowered, error
        self.seconds = seconds


def nvrtc_version() -> tuple:
    lib = load_library()
    a, b = C.c_int(), C.c_int()
    lib.tsg_nvrtc_version(C.byref(a), C.byref(b))
    return (a.value, b.value)


def compile_source(source: str, options: list[str], name_expr: str | None = None,
                   program_name: str = "kernel.cu") -> CompileResult:
    """NVRTC -> cubin (context-free; safe to call from worker threads)."""
    import time

    lib = load_library()
    opts = (C.c_char_p * len(options))(*[o.encode() for o in options])
    img = C.c_void_p()
    size = C.c_size_t()
    lowered = C.create_string_buffer(1024)
    log = C.create_string_buffer(1 << 16)
    t0 = time.perf_counter()
    rc = lib.tsg_compile(source.encode(), program_name.encode(),
                         name_expr.encode() if name_expr else None, opts, len(options),
                         C.byref(img), C.byref(size), lowered, 1024, log, 1 << 16)
    dt = time.perf_counter() - t0
    if rc != OK:
        return CompileResult(False, log=log.value.decode(errors="replace"),
                             error=last_error(), seconds=dt)
    data = C.string_at(img.value, size.value)
    lib.tsg_free_host(img)
    return CompileResult(True, data, log.value.decode(errors="replace"),
                         lowered.value.decode(), seconds=dt)


class CubinCache:
    """On-disk cache of compiled cubins keyed by (source, options, NVRTC).

    Warm sweeps skip NVRTC entirely; the key includes the NVRTC version
    and the arch so a toolkit change never reuses stale code.
    """

    def __init__(self, root: str | Path | None = None):
        root = root or os.environ.get("TSG_CUBIN_CACHE") or (Path.home() / ".cache" / "tsgpu_cubins")
        self.root = Path(root)
        self.root.mkdir(parents=True, exist_ok=True)
        self._ver = None

    def key(self, source: str, options: list[str], name_expr: str | None) -> str:
        if self._ver is None:
            self._ver = "%d.%d" % nvrtc_version()
        h = hashlib.sha256()
        for part in (self._ver, ARCH, source, "\0".join(options), name_expr or ""):
            h.update(part.encode())
            h.update(b"\1")
        return h.hexdigest()

    def get(self, key: str):
        p = self.root / key[:2] / (key + ".cubin")
        try:
            data = p.read_bytes()
        except OSError:
            return None
        name = p.with_suffix(".name")
        lowered = name.read_text() if name.exists() else ""
        return data, lowered

    def put(self, key: str, image: bytes, lowered: str = ""):
        d = self.root / key[:2]
        d.mkdir(parents=True, exist_ok=True)
        tmp = d / f".{key}.{os.getpid()}.{threading.get_ident()}.tmp"
        tmp.write_bytes(image)
        os.replace(tmp, d / (key + ".cubin"))
        if lowered:
            (d / (key + ".name")).write_text(lowered)


class Module:
    def __init__(self, dev: "Device", handle: int):
        self.dev = dev
        self.handle = handle
        self._fns = {}

    def function(self, name: str) -> "Kernel":
        if name not in self._fns:
            h = C.c_void_p()
            self.dev._check(self.dev.lib.tsg_get_function(self.handle, name.encode(), C.byref(h)))
            self._fns[name] = Kernel(self, h.value)
        return self._fns[name]

    def set_constant(self, symbol: str, data: np.ndarray):
        data = np.ascontiguousarray(data)
        return self.dev.lib.tsg_set_constant(self.handle, symbol.encode(),
                                             data.ctypes.data_as(C.c_void_p), data.nbytes)

    def unload(self):
        if self.handle:
            self.dev.lib.tsg_module_unload(self.handle)
            self.handle = None


class Kernel:
    def __init__(self, module: Module, handle: int):
        self.module = module
        self.handle = handle

    def attrs(self) -> dict:
        v = [C.c_int() for _ in range(4)]
        self.module.dev.lib.tsg_func_attrs(self.handle, *[C.byref(x) for x in v])
        return dict(regs=v[0].value, static_smem=v[1].value, max_threads=v[2].value,
                    local_bytes=v[3].value)

    def set_max_dynamic_smem(self, nbytes: int) -> int:
        return self.module.dev.lib.tsg_set_max_dynamic_smem(self.handle, int(nbytes))

    def set_smem_carveout(self, percent: int) -> int:
        return self.module.dev.lib.tsg_set_smem_carveout(self.handle, int(percent))

    def occupancy(self, block_threads: int, dyn_smem: int) -> int:
        """Resident blocks per SM for this launch shape (0 if it cannot launch)."""
        n = C.c_int(0)
        rc = self.module.dev.lib.tsg_occupancy(self.handle, int(block_threads), int(dyn_smem), C.byref(n))
        return n.value if rc == OK else 0

    @property
    def sm_count(self) -> int:
        return int(self.module.dev.info["sm_count"])


class Launch:
    """One launch of a timed sequence: kernel, geometry, typed arguments.

    ``args`` is a list of ctypes scalars (c_uint64 for device pointers,
    c_int / c_float for values); they are kept alive by this object.
    """

    def __init__(self, kernel: Kernel, grid, block, args, smem: int = 0, cluster=(1, 1, 1), pdl: bool = False):
        self.kernel = kernel
        self.grid = tuple(int(g) for g in grid) + (1,) * (3 - len(grid))
        self.block = tuple(int(b) for b in block) + (1,) * (3 - len(block))
        self.cluster = tuple(int(c) for c in cluster) + (1,) * (3 - len(cluster))
        self.smem = int(smem)
        self.pdl = bool(pdl)  # programmatic dependent launch (kernel runs griddepcontrol.wait)
        self.args = list(args)
        self._ptrs = (C.c_void_p * max(1, len(self.args)))(
            *[C.cast(C.pointer(a), C.c_void_p) for a in self.args])

    def to_struct(self) -> LaunchT:
        s = LaunchT()
        s.fn = self.kernel.handle
        s.grid[:] = self.grid
        s.block[:] = self.block
        s.cluster[:] = self.cluster
        s.smem_bytes = self.smem
        s.flags = LAUNCH_PDL if self.pdl else 0
        s.args = C.cast(self._ptrs, C.POINTER(C.c_void_p))
        return s


class Buffer:
    """A device allocation owned by a :class:`Device`."""

    def __init__(self, dev: "Device", ptr: int, nbytes: int):
        self.dev, self.ptr, self.nbytes = dev, ptr, nbytes

    def arg(self):
        return C.c_uint64(self.ptr)

    def upload(self, host: np.ndarray):
        host = np.ascontiguousarray(host)
        if host.nbytes > self.nbytes:
            raise ProtocolError("upload larger than buffer")
        self.dev._check(self.dev.lib.tsg_h2d(self.dev.ctx, self.ptr,
                                             host.ctypes.data_as(C.c_void_p), host.nbytes))

    def download(self, out: np.ndarray) -> np.ndarray:
        self.dev._check(self.dev.lib.tsg_d2h(self.dev.ctx, out.ctypes.data_as(C.c_void_p),
                                             self.ptr, out.nbytes))
        return out

    def free(self):
        if self.ptr:
            self.dev.lib.tsg_free(self.dev.ctx, self.ptr)
            self.ptr = 0


class Device:
    """One CUDA device (primary context + stream) through libtsgpu."""

    def __init__(self, index: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.tsg_init(int(index), C.byref(h))
        if rc != OK:
            raise DeviceError(f"cannot initialise CUDA device {index}: {last_error()}")
        self.ctx = h.value
        self.index = index
        info = DeviceInfoT()
        self.lib.tsg_device_info(self.ctx, C.byref(info))
        self.info = {k: (getattr(info, k).decode() if k == "name" else getattr(info, k))
                     for k, _ in DeviceInfoT._fields_}
        self.poisoned = False

    def _check(self, rc: int):
        if rc != OK:
            if rc in (ERR_RUNTIME, ERR_TIMEOUT):
                self.poisoned = True
            raise DeviceError(f"{self.lib.tsg_error_string(rc).decode()}: {last_error()}")

    @property
    def launch_count(self) -> int:
        return int(self.lib.tsg_launch_count(self.ctx))

    def alloc(self, nbytes: int) -> Buffer:
        p = C.c_uint64()
        self._check(self.lib.tsg_alloc(self.ctx, int(nbytes), C.byref(p)))
        return Buffer(self, p.value, int(nbytes))

    def to_device(self, host: np.ndarray) -> Buffer:
        b = self.alloc(host.nbytes)
        b.upload(host)
        return b

    def load(self, image: bytes):
        """Load a cubin; returns (status_code, Module | error text)."""
        h = C.c_void_p()
        rc = self.lib.tsg_module_load(self.ctx, image, len(image), C.byref(h))
        if rc != OK:
            if rc == ERR_RUNTIME:
                self.poisoned = True
            return rc, last_error()
        return OK, Module(self, h.value)

    def run(self, launches: list, timeout_ms: float = 60000.0) -> tuple:
        arr = (LaunchT * len(launches))(*[l.to_struct() for l in launches])
        rc = self.lib.tsg_run(self.ctx, arr, len(launches), float(timeout_ms))
        if rc in (ERR_RUNTIME, ERR_TIMEOUT):
            self.poisoned = True
        return rc, ("" if rc == OK else last_error())

    # -- ordering against foreign streams (torch / NCCL), include/tsgpu.h --
    @property
    def stream(self) -> int:
        """Handle of the context stream (CUstream value)."""
        h = C.c_uint64()
        self._check(self.lib.tsg_stream_handle(self.ctx, C.byref(h)))
        return int(h.value)

    def wait_stream(self, stream: int) -> None:
        """Later work on the context stream waits for what ``stream`` has enqueued so far."""
        self._check(self.lib.tsg_stream_wait(self.ctx, int(stream)))

    def signal_stream(self, stream: int) -> None:
        """Later work on ``stream`` waits for what the context stream has enqueued so far."""
        self._check(self.lib.tsg_stream_signal(self.ctx, int(stream)))

    def launch_async(self, launches: list) -> None:
        """Enqueue launches on the context stream without waiting."""
        arr = (LaunchT * len(launches))(*[l.to_struct() for l in launches])
        self._check(self.lib.tsg_launch_async(self.ctx, arr, len(launches)))

    def copy_async(self, dst: int, src: int, nbytes: int) -> None:
        self._check(self.lib.tsg_copy_async(self.ctx, int(dst), int(src), int(nbytes)))

    def sync(self, timeout_ms: float = 60000.0) -> None:
        self._check(self.lib.tsg_sync(self.ctx, float(timeout_ms)))

    def run_timed(self, launches: list, warmup: int, runs: int, flush_l2: bool = True,
                  timeout_ms: float = 60000.0):
        """Returns (status_code, times_ms list | error text)."""
        arr = (LaunchT * len(launches))(*[l.to_struct() for l in launches])
        times = (C.c_float * runs)()
        rc = self.lib.tsg_run_timed(self.ctx, arr, len(launches), int(warmup), int(runs),
                                    1 if flush_l2 else 0, float(timeout_ms), times)
        if rc != OK:
            if rc in (ERR_RUNTIME, ERR_TIMEOUT):
                self.poisoned = True
            return rc, last_error()
        return OK, [float(t) for t in times]

    def submit_timed(self, slot: int, launches: list, warmup: int, runs: int, flush_l2: bool,
                     out: "Buffer | None", n_out: int, ref: "Buffer | None", rtol: float = 0.0,
                     atol: float = 0.0) -> tuple:
        """Enqueue one configuration's protocol into ``slot`` without waiting
        (tsg_submit_timed); returns (status_code, error text)."""
        arr = (LaunchT * len(launches))(*[l.to_struct() for l in launches])
        rc = self.lib.tsg_submit_timed(self.ctx, int(slot), arr, len(launches), int(warmup), int(runs),
                                       1 if flush_l2 else 0, out.ptr if out is not None else 0, int(n_out),
                                       ref.ptr if ref is not None else 0, float(rtol), float(atol))
        if rc != OK:
            err = last_error()
            if rc in (ERR_RUNTIME, ERR_TIMEOUT):
                self.poisoned = True
            self.lib.tsg_slot_reset(self.ctx, int(slot))
            return rc, err
        return OK, ""

    def collect(self, slot: int, runs: int, n_launch: int, timeout_ms: float = 60000.0) -> tuple:
        """Wait for ``slot``; returns (status_code, times | error, per-launch times, compare dict)."""
        times = (C.c_float * runs)()
        lt = (C.c_float * n_launch)()
        e, r = C.c_double(), C.c_double()
        bad, nf = C.c_uint64(), C.c_uint64()
        rc = self.lib.tsg_collect(self.ctx, int(slot), float(timeout_ms), times, lt, int(n_launch), C.byref(e),
                                  C.byref(r), C.byref(bad), C.byref(nf))
        if rc != OK:
            if rc in (ERR_RUNTIME, ERR_TIMEOUT):
                self.poisoned = True
            return rc, last_error(), None, None
        cmp = dict(max_abs_err=e.value, max_abs_ref=r.value, n_bad=int(bad.value), n_nonfinite=int(nf.value))
        return OK, [float(t) for t in times], [float(x) for x in lt], cmp

    def slot_timeline(self, slot: int) -> tuple:
        """(start_ms, end_ms, warmup_ms) of a collected slot on the device timeline."""
        a, b, w = C.c_double(), C.c_double(), C.c_float()
        if self.lib.tsg_slot_timeline(self.ctx, int(slot), C.byref(a), C.byref(b), C.byref(w)) != OK:
            return None
        return a.value, b.value, w.value

    def last_launch_times(self, n: int) -> list:
        t = (C.c_float * n)()
        self.lib.tsg_last_launch_times(self.ctx, t, n)
        return [float(x) for x in t]

    def tma_2d_f32(self, buf: "Buffer", dim0: int, dim1: int, stride1_bytes: int, box0: int, box1: int,
                   swizzle: int = 128):
        """CUtensorMap (128 bytes, by-value kernel argument) for a 2-D fp32 tensor."""
        desc = (C.c_ubyte * 128)()
        self._check(self.lib.tsg_tma_encode_2d_f32(self.ctx, desc, buf.ptr, dim0, dim1, stride1_bytes,
                                                   box0, box1, swizzle))
        return desc

    def mark(self, slot: int) -> None:
        """Record stream marker ``slot`` (device-side region timing)."""
        self._check(self.lib.tsg_event_record(self.ctx, int(slot)))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        self._check(self.lib.tsg_event_elapsed(self.ctx, int(a), int(b), C.byref(ms)))
        return float(ms.value)

    def compare(self, out: Buffer, ref: Buffer, n: int, rtol: float, atol: float) -> dict:
        e, r = C.c_double(), C.c_double()
        bad, nf = C.c_uint64(), C.c_uint64()
        self._check(self.lib.tsg_compare_f32(self.ctx, out.ptr, ref.ptr, int(n), float(rtol),
                                             float(atol), C.byref(e), C.byref(r), C.byref(bad),
                                             C.byref(nf)))
        return dict(max_abs_err=e.value, max_abs_ref=r.value, n_bad=int(bad.value),
                    n_nonfinite=int(nf.value))

    def close(self):
        if self.ctx:
            self.lib.tsg_destroy(self.ctx)
            self.ctx = None
