"""Build the native pieces in-tree (sm_100a): libtsgpu.so and the C oracle.

``python -m paper_2407_11488_b200.build`` or ``__graft_entry__.build()``.
NVRTC kernel sources under ``kernels/`` are compiled per configuration
at tuning time; here we additionally compile a sample configuration of
each with nvcc so a broken kernel fails the build, not the sweep.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def _stale(target: Path, *sources: Path) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_libtsgpu(force: bool = False) -> Path:
    out = HERE / "libtsgpu.so"
    srcs = [HERE / "csrc" / "tsgpu.cu", HERE / "csrc" / "driver_table.h", ROOT / "include" / "tsgpu.h"]
    if force or _stale(out, *srcs):
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-o", str(out), str(srcs[0]), f"-L{CUDA}/lib64", "-lnvrtc", "-ldl",
              "-Xlinker", f"-rpath,{CUDA}/lib64"])
    return out


SAMPLES = {
    "convolution.cu": "-DBSX=32 -DBSY=8 -DTSX=4 -DTSY=4 -DREAD_ONLY=1 -DUSE_PADDING=0 -DUSE_SHMEM=1 "
                      "-DIMG_W=4096 -DIMG_H=4096 -DIN_PITCH=4112",
    "hotspot.cu": "-DBSX=32 -DBSY=8 -DTSX=2 -DTSY=2 -DTT=4 -DUNROLL=2 -DSH_POWER=1 -DGW=4096 -DGH=4096",
    "dedispersion.cu": "-DBSX=8 -DBSY=64 -DTSX=2 -DTSY=4 -DSTX=1 -DSTY=0 -DNCH=1536 -DNSAMP=25000 "
                       "-DNDM=2048 -DIN_PITCH=25792",
    "gemm.cu": "-DMWG=128 -DNWG=128 -DKWG=16 -DMDIMC=16 -DNDIMC=16 -DMDIMA=16 -DNDIMB=16 -DVWM=4 "
               "-DVWN=4 -DSTRM=0 -DSTRN=0 -DSA=1 -DSB=1 -DGM=4096 -DGN=4096 -DGK=4096",
}


def check_kernels(tmp: Path | None = None) -> None:
    """nvcc-compile one configuration of every tunable kernel (sm_100a)."""
    tmp = tmp or (ROOT / "build")
    tmp.mkdir(exist_ok=True)
    for name, defs in SAMPLES.items():
        src = HERE / "kernels" / name
        extra = ["--fmad=false"] if name == "hotspot.cu" else []
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-cubin", *extra, *defs.split(),
              "-o", str(tmp / (src.stem + ".cubin")), str(src)])
    for name in ("gemm_tc.cu",):
        src = HERE / "kernels" / name
        if src.exists():
            _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-cubin", "-DGM=4096", "-DGN=4096",
                  "-DGK=4096", "-o", str(tmp / (src.stem + ".cubin")), str(src)])


def build_oracle() -> None:
    oracle = ROOT / "oracle"
    if (oracle / "Makefile").exists() and shutil.which("make"):
        _run(["make", "-s", "-C", str(oracle)])


def install_reference() -> None:
    """The UNMODIFIED reference under baseline/_ref (git-ignored, travels to
    the GPU box with the snapshot) for bench.py's reference arm -- only where
    /root/reference exists (this container), only if missing."""
    recipe = ROOT / "baseline" / "install_reference.sh"
    if (Path("/root/reference/pkg").is_dir() and recipe.exists()
            and not (ROOT / "baseline" / "_ref" / "tunescape" / "__init__.py").exists()):
        _run(["bash", str(recipe)])


def build_all(force: bool = False, kernels: bool = True) -> None:
    build_libtsgpu(force)
    build_oracle()
    install_reference()
    if kernels:
        check_kernels()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
