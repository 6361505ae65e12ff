"""ctypes binding of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

Each wrapper takes the same host arrays the product uploads (same
padding/pitch) so tests compare like with like.  Built by
``oracle/Makefile`` (``__graft_entry__.build()`` runs it).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None

_F = C.POINTER(C.c_float)


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.oracle_convolution.argtypes = [_F, _F, C.c_int, C.c_int, C.c_int, _F, C.c_int, C.c_int]
        L.oracle_hotspot.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_int] + [C.c_float] * 5 + [_F]
        L.oracle_hotspot_tuned.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_int] + [C.c_float] * 5 + [_F]
        L.oracle_hotspot_tuned.restype = None
        L.oracle_dedispersion.argtypes = [_F, _F, C.c_int, _F, C.c_int, C.c_int, C.c_int,
                                          C.c_float, C.c_float]
        L.oracle_gemm.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_int]
        L.oracle_threads.restype = C.c_int
        L.oracle_set_threads.argtypes = [C.c_int]
        for f in ("oracle_convolution", "oracle_hotspot", "oracle_dedispersion", "oracle_gemm"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_F)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def threads() -> int:
    return int(lib().oracle_threads())


def convolution(prob, padded: np.ndarray | None = None) -> np.ndarray:
    """Oracle output for a :class:`Convolution` problem (fp32 [H*W])."""
    if padded is None:
        padded = prob.buffers()[0].init
    out = np.empty(prob.W * prob.H, np.float32)
    f = np.ascontiguousarray(prob.filter().ravel())
    lib().oracle_convolution(_p(out), _p(padded), prob.pitch, prob.W, prob.H, _p(f), prob.FW, prob.FH)
    return out


def hotspot(prob, iterations: int | None = None) -> np.ndarray:
    temp = np.ascontiguousarray(prob.temperature())
    power = np.ascontiguousarray(prob.power())
    out = np.empty(prob.W * prob.H, np.float32)
    scratch = np.empty_like(out)
    k = prob.k
    it = prob.iterations if iterations is None else iterations
    lib().oracle_hotspot(_p(out), _p(temp), _p(power), prob.W, prob.H, it, k["sdc"], k["rx1"],
                         k["ry1"], k["rz1"], k["amb"], _p(scratch))
    return out


def hotspot_tuned(prob, iterations: int | None = None) -> np.ndarray:
    """The tuned kernels' folded arithmetic (bit-exact target of every tuned
    hotspot configuration; within rtol 1e-5 of :func:`hotspot`)."""
    temp = np.ascontiguousarray(prob.temperature())
    power = np.ascontiguousarray(prob.power())
    out = np.empty(prob.W * prob.H, np.float32)
    scratch = np.empty_like(out)
    c = prob.tuned_coefficients(prob.k)
    it = prob.iterations if iterations is None else iterations
    lib().oracle_hotspot_tuned(_p(out), _p(temp), _p(power), prob.W, prob.H, it, c["at"], c["ay"], c["ax"],
                               c["ap"], c["ac"], _p(scratch))
    return out


def dedispersion(prob) -> np.ndarray:
    padded = prob.buffers()[0].init
    out = np.empty(prob.NDM * prob.NSAMP, np.float32)
    delay = np.ascontiguousarray(prob.delay)
    lib().oracle_dedispersion(_p(out), _p(padded), prob.pitch, _p(delay), prob.NCH, prob.NSAMP,
                              prob.NDM, prob.dm_first, prob.dm_step)
    return out


def gemm(prob) -> np.ndarray:
    a = np.ascontiguousarray(prob.a())
    b = np.ascontiguousarray(prob.b())
    out = np.empty(prob.M * prob.N, np.float32)
    lib().oracle_gemm(_p(out), _p(a), _p(b), prob.M, prob.N, prob.K)
    return out


def answer(prob) -> np.ndarray:
    """The reference answer (the on-device naive kernel computes the same)."""
    return {"convolution": convolution, "hotspot": hotspot, "dedispersion": dedispersion,
            "gemm": gemm, "gemm_tc": gemm}[prob.space_name](prob)


def tuned(prob) -> np.ndarray:
    """What every tuned configuration must reproduce BIT-FOR-BIT: the answer,
    except where the tuned kernels use a restated operation order (hotspot)."""
    if prob.space_name == "hotspot":
        return hotspot_tuned(prob)
    return answer(prob)


# ---------------------------------------------------------------------------
# independent float64 numpy restatements (pin the C oracle within tolerance)


def convolution_f64(prob) -> np.ndarray:
    img = prob.image().astype(np.float64)
    f = prob.filter().astype(np.float64)
    out = np.zeros((prob.H, prob.W))
    for i in range(prob.FH):
        for j in range(prob.FW):
            out += f[i, j] * img[i:i + prob.H, j:j + prob.W]
    return out.ravel()


def hotspot_f64(prob, iterations: int | None = None) -> np.ndarray:
    t = prob.temperature().astype(np.float64)
    p = prob.power().astype(np.float64)
    k = prob.k
    for _ in range(prob.iterations if iterations is None else iterations):
        n = np.vstack([t[:1], t[:-1]])
        s = np.vstack([t[1:], t[-1:]])
        w = np.hstack([t[:, :1], t[:, :-1]])
        e = np.hstack([t[:, 1:], t[:, -1:]])
        t = t + k["sdc"] * (p + (n + s - 2 * t) * k["ry1"] + (e + w - 2 * t) * k["rx1"]
                            + (k["amb"] - t) * k["rz1"])
    return t.ravel()


def dedispersion_f64(prob) -> np.ndarray:
    from paper_2407_11488_b200.problems import dm_shifts

    data = prob.data().astype(np.float64)
    sh = dm_shifts(prob.delay, prob.NDM, prob.dm_first, prob.dm_step)
    out = np.zeros((prob.NDM, prob.NSAMP))
    for d in range(prob.NDM):
        for ch in range(prob.NCH):
            out[d] += data[ch, sh[d, ch]:sh[d, ch] + prob.NSAMP]
    return out.ravel()


def gemm_f64(prob) -> np.ndarray:
    a = prob.a().astype(np.float64)  # [K][M]
    b = prob.b().astype(np.float64)  # [K][N]
    c = a.T @ b  # [M][N]
    return np.ascontiguousarray(c.T).ravel()  # C[n*M+m]
