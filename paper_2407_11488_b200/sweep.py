"""Sweep helpers shared by bench.py, the multi-GPU runner and tools/.

* :func:`stratified_sample` -- deterministic configuration samples
  (e.g. the hotspot temporal_tiling_factor 1-10 sweep of BASELINE
  config 1), drawn from the valid flat-index set;
* :func:`fp32_peak` -- measured FFMA peak of this GPU (roofline
  denominator for SIMT kernels; MEASURED_PEAKS.json has only HBM/bf16);
* :func:`roofline` -- algorithmic work of one configuration against the
  binding B200 ceiling.
"""

from __future__ import annotations

import ctypes as C
import json
import math
from pathlib import Path

import numpy as np

from . import runtime as rt

ROOT = Path(__file__).resolve().parent.parent
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (driver-measured)",
                "bf16_tflops": float(d.get("bf16_tflops", 0.0))}
    return {"hbm_gbs": FALLBACK_HBM_GBS, "source": "B200_PROFILING.md fallback", "bf16_tflops": 1590.0}


def stratified_sample(space, n: int, seed: int, param: str | None = None, offset: int = 0) -> list:
    """``n`` distinct valid configurations, round-robin over ``param``'s values.

    Deterministic in (space, n, seed, param, offset); ``offset`` selects a
    disjoint block of the same per-stratum permutations (rank / step
    sharding without overlap).
    """
    idx = space.valid_indices()
    rng = np.random.default_rng(seed)
    if param is None:
        perm = rng.permutation(len(idx))
        take = perm[(offset + np.arange(min(n, len(idx)))) % len(idx)]  # wraps on small spaces
        return space.configs_at(idx[take])
    pi = space.param_names.index(param)
    configs = space.configs_at(idx)
    strata: dict = {}
    for k, c in enumerate(configs):
        strata.setdefault(c[pi], []).append(k)
    keys = sorted(strata)
    perms = {v: rng.permutation(len(strata[v])) for v in keys}
    out = []
    per = math.ceil(n / len(keys))
    start = offset // len(keys)
    for j in range(per):
        for v in keys:
            lst = strata[v]
            pos = (start + j) % len(lst)  # wraps once a stratum is exhausted
            if len(out) < n:
                out.append(configs[lst[perms[v][pos]]])
    return out


_PEAK_CACHE: dict = {}


def fp32_peak(dev: rt.Device, iters: int = 2048) -> dict:
    """FFMA throughput of this GPU (TFLOP/s), measured with CUDA events."""
    if dev.index in _PEAK_CACHE:
        return _PEAK_CACHE[dev.index]
    src = (Path(__file__).parent / "kernels" / "peak.cu").read_text()
    res = rt.compile_source(src, ["--gpu-architecture=sm_100a", "-std=c++17"])
    if not res.ok:
        raise RuntimeError(res.error)
    rc, mod = dev.load(res.image)
    if rc != rt.OK:
        raise RuntimeError(mod)
    k = mod.function("ffma_peak")
    # (the same module also holds ffma2_peak, loaded again below)
    blocks = dev.info["sm_count"] * 8
    out = dev.alloc(blocks * 256 * 4)
    launch = rt.Launch(k, (blocks, 1, 1), (256, 1, 1),
                       [C.c_uint64(out.ptr), C.c_int(iters), C.c_float(0.999), C.c_float(1e-3)])
    rc, times = dev.run_timed([launch], 2, 5, flush_l2=False)
    mod.unload()
    out.free()
    if rc != rt.OK:
        raise RuntimeError(times)
    flop = 2.0 * blocks * 256 * iters * 8 * 16
    best = min(times)
    # packed fp32x2 FMA (FFMA2): same probe with two FMAs per instruction
    rc2, mod2 = dev.load(res.image)
    k2 = mod2.function("ffma2_peak")
    out2 = dev.alloc(blocks * 256 * 4)
    launch2 = rt.Launch(k2, (blocks, 1, 1), (256, 1, 1),
                        [C.c_uint64(out2.ptr), C.c_int(iters), C.c_float(0.999), C.c_float(1e-3)])
    rc2, times2 = dev.run_timed([launch2], 2, 5, flush_l2=False)
    mod2.unload()
    out2.free()
    f2 = (2.0 * flop / (min(times2) * 1e-3) / 1e12) if rc2 == rt.OK else 0.0
    scalar = flop / (best * 1e-3) / 1e12
    r = {"fp32_tflops": max(scalar, f2), "ffma_tflops": scalar, "ffma2_tflops": f2, "probe_ms": best,
         "nominal_tflops_at_max_clock": dev.info["sm_count"] * 128 * 2 * dev.info["clock_khz"] * 1e3 / 1e12}
    _PEAK_CACHE[dev.index] = r
    return r


def cublas_tf32(n: int = 4096, reps: int = 10) -> dict:
    """cuBLAS TF32 GEMM (torch.matmul on fp32, TF32 allowed) on the tuned
    problem's shape, best of ``reps`` after warm-up, CUDA events: the library
    baseline the tcgen05 kernel is compared with (bench `alt.vs_cublas`).
    torch is plumbing here; the tuned kernels never go through it."""
    import torch

    if not torch.cuda.is_available():
        return {}
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.rand(n, n, device="cuda")
        b = torch.rand(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(a, b)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        del a, b
        torch.cuda.empty_cache()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return {"cublas_tf32_tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "cublas_tf32_ms": best}


def tf32_peak(dev: rt.Device, iters: int = 4096) -> dict:
    """Dense tf32 tcgen05 throughput of this GPU (TFLOP/s), measured with CUDA
    events: kernels/peak.cu tf32_mma_peak, one CTA per SM issuing back-to-back
    M=128 N=256 K=8 MMAs from shared memory (the GEMM's instruction shape)."""
    key = ("tf32", dev.index)
    if key in _PEAK_CACHE:
        return _PEAK_CACHE[key]
    src = (Path(__file__).parent / "kernels" / "peak.cu").read_text()
    res = rt.compile_source(src, ["--gpu-architecture=sm_100a", "-std=c++17"])
    if not res.ok:
        raise RuntimeError(res.error)
    rc, mod = dev.load(res.image)
    if rc != rt.OK:
        raise RuntimeError(mod)
    k = mod.function("tf32_mma_peak")
    smem = 1024 + 128 * 128 + 256 * 128 + 64
    k.set_max_dynamic_smem(smem)
    blocks = dev.info["sm_count"]
    out = dev.alloc(blocks * 4)
    launch = rt.Launch(k, (blocks, 1, 1), (128, 1, 1), [C.c_uint64(out.ptr), C.c_int(iters)], smem=smem)
    rc, times = dev.run_timed([launch], 2, 5, flush_l2=False)
    mod.unload()
    out.free()
    if rc != rt.OK:
        raise RuntimeError(times)
    flop = 2.0 * 128 * 256 * 8 * 4 * iters * blocks
    r = {"tf32_tflops": flop / (min(times) * 1e-3) / 1e12, "tf32_probe_ms": min(times),
         "tf32_source": "measured in-run: tcgen05.mma kind::tf32 M128 N256 K8 back to back, one CTA per SM "
                        "(kernels/peak.cu tf32_mma_peak)"}
    _PEAK_CACHE[key] = r
    return r


def roofline(problem, cfg: dict, info: dict, peaks: dict) -> dict:
    """Roofline of the dominant launch of one configuration.

    achieved = algorithmic work of that launch / its CUDA-event duration
    (``info['launch_ms']`` from the last timed run).  The binding bound is
    the larger of compulsory-HBM time and FP32 time.
    """
    launch_ms = info.get("launch_ms") or []
    if not launch_ms:
        return {}
    n = len(launch_ms)
    dom = int(np.argmax(launch_ms))
    t = launch_ms[dom] * 1e-3
    flop = problem.flops(cfg) / n
    byts = problem.compulsory_bytes(cfg) / n
    hbm_peak = peaks["hbm_gbs"] * 1e9
    if getattr(problem, "space_name", "") == "hotspot":
        # one launch advancing k steps: 12 B/cell compulsory (read T, P; write
        # T).  The tuned form needs 5 FP32-pipe operations per cell update (+1
        # per cell for the power term), so the FP32 time of a launch stays
        # below its HBM time at every T <= 10: the binding roofline is HBM.
        steps = problem.step_plan(cfg["temporal_tiling_factor"])
        cells = problem.W * problem.H
        byts = 12.0 * cells
        gbs = byts / t / 1e9
        fp_ops = cells * (5.0 * steps[dom] + 1.0)
        pipe = peaks.get("fp32_tflops", 0.0) * 1e12 / 2.0  # FMA-pipe operations per second
        return {"bound": "hbm", "achieved": round(gbs, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "traffic": None,
                "bytes_per_launch": byts, "launch_us": round(t * 1e6, 3), "steps_in_launch": steps[dom],
                "alt": {"paper_gflops": round(problem.FLOP_PER_CELL * cells * steps[dom] / t / 1e9, 1),
                        "fp32_pipe_frac": round(fp_ops / t / pipe, 4) if pipe else None,
                        "hbm_floor_us": round(byts / hbm_peak * 1e6, 2)}}
    if getattr(problem, "space_name", "") == "gemm_tc":
        # tf32 tensor pipe: the in-run tcgen05 tf32 probe (sweep.tf32_peak);
        # fallback half the driver-measured bf16 burst
        if peaks.get("tf32_tflops"):
            tf32, src = peaks["tf32_tflops"], peaks.get("tf32_source", "in-run tf32 probe")
        else:
            tf32, src = 0.5 * peaks.get("bf16_tflops", 1639.7), "0.5 x MEASURED_PEAKS bf16_tflops (fallback)"
        tfs = flop / t / 1e12
        alt = {"hbm_gbs": round(byts / t / 1e9, 2)}
        if peaks.get("cublas_tf32_tflops"):  # the library GEMM on the same problem, same run
            alt["cublas_tf32_tflops"] = round(peaks["cublas_tf32_tflops"], 1)
            alt["vs_cublas"] = round(tfs / peaks["cublas_tf32_tflops"], 3)
        return {"bound": "tensor", "achieved": round(tfs, 2), "peak": round(tf32, 2), "unit": "TFLOP/s",
                "frac": round(tfs / tf32, 4), "traffic": None, "peak_source": src, "alt": alt}
    fp32 = peaks.get("fp32_tflops", 0.0) * 1e12
    if getattr(problem, "space_name", "") == "dedispersion":
        # add-only kernel: the FP32 pipe retires one FADD per lane per cycle
        # (FADD2 = two adds in two cycles), i.e. half the FFMA FLOP rate
        tadd = 0.5 * fp32
        ta = flop / t
        return {"bound": "fp32", "achieved": round(ta / 1e12, 3), "peak": round(tadd / 1e12, 3),
                "unit": "Tadd/s", "frac": round(ta / tadd, 4), "traffic": None,
                "peak_source": "0.5 x in-run FFMA probe (FADD = 1 FLOP per FMA-pipe slot)",
                "alt": {"paper_gbs": round(4.0 * flop / t / 1e9, 1),
                        "hbm_gbs": round(byts / t / 1e9, 2)}}
    t_hbm = byts / hbm_peak
    t_fp = flop / fp32 if fp32 else 0.0
    gbs = byts / t / 1e9
    tfs = flop / t / 1e12
    if t_hbm >= t_fp:
        return {"bound": "hbm", "achieved": round(gbs, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "traffic": None,
                "alt": {"fp32_tflops": round(tfs, 3), "fp32_frac": round(tfs * 1e12 / fp32, 4) if fp32 else None}}
    return {"bound": "fp32", "achieved": round(tfs, 3), "peak": round(fp32 / 1e12, 3), "unit": "TFLOP/s",
            "frac": round(tfs * 1e12 / fp32, 4), "traffic": None,
            "alt": {"hbm_gbs": round(gbs, 2), "hbm_frac": round(gbs / peaks["hbm_gbs"], 4)}}
