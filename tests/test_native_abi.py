"""The C ABI (include/tsgpu.h) without a GPU.

* libtsgpu.so loads on a host with no NVIDIA driver (the driver is
  dlopen'ed at tsg_init) and exports every function the header declares;
* NVRTC compiles sample configurations of every kernel for sm_100a
  (context-free), and compile errors surface as compile_failed;
* tsg_init reports a setup error (never a crash) when no driver exists.
"""

import re
from pathlib import Path

import pytest

from paper_2407_11488_b200 import runtime as rt
from paper_2407_11488_b200.problems import make_problem

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "tsgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = rt.load_library()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(rt.SIGNATURES), set(declared) ^ set(rt.SIGNATURES)


def test_nvrtc_version():
    major, minor = rt.nvrtc_version()
    assert major >= 12


SAMPLE = {
    "convolution": (32, 8, 4, 4, 1, 0, 1),
    "hotspot": (32, 8, 2, 2, 4, 2, 1),
    "dedispersion": (8, 64, 2, 4, 1, 0),
    "gemm": (128, 128, 16, 16, 16, 16, 16, 4, 4, 0, 0, 1, 1),
}


@pytest.mark.parametrize("name", sorted(SAMPLE))
def test_nvrtc_compiles_each_kernel(name):
    prob = make_problem(name)
    cfg = dict(zip(prob.space.param_names, SAMPLE[name]))
    assert prob.space.is_valid(SAMPLE[name])
    res = rt.compile_source(prob.source(), prob.options(cfg))
    assert res.ok, res.error
    assert res.image[:4] == b"\x7fELF"
    ref = rt.compile_source(prob.source(), prob.options(None) + ["-DREFERENCE_ONLY=1"])
    assert ref.ok, ref.error


def test_compile_error_is_reported():
    res = rt.compile_source("extern \"C\" __global__ void k() { this is not cuda; }",
                            ["--gpu-architecture=sm_100a"])
    assert not res.ok and "error" in (res.error + res.log).lower()


def test_init_without_driver_is_a_clean_error():
    import ctypes as C

    lib = rt.load_library()
    h = C.c_void_p()
    rc = lib.tsg_init(0, C.byref(h))
    if rc == rt.OK:
        lib.tsg_destroy(h)
        pytest.skip("a GPU is present on this host")
    assert rc == rt.ERR_SETUP
    assert rt.last_error()


def test_launch_record_layout_matches_header():
    """tsg_launch_t (include/tsgpu.h): the ctypes mirror has the header's
    field order and offsets (`flags`, TSG_LAUNCH_PDL, sits between
    `smem_bytes` and `args`)."""
    import ctypes as C
    import re
    from pathlib import Path

    from paper_2407_11488_b200.runtime import LAUNCH_PDL, LaunchT

    hdr = (Path(__file__).resolve().parents[1] / "include" / "tsgpu.h").read_text()
    body = re.search(r"typedef struct \{([^}]*)\} tsg_launch_t;", hdr).group(1)
    names = re.findall(r"(\w+)(?:\[\d\])?;", body)
    assert names == [f[0] for f in LaunchT._fields_]
    assert int(re.search(r"#define TSG_LAUNCH_PDL (\d+)u", hdr).group(1)) == LAUNCH_PDL
    assert LaunchT.smem_bytes.offset == 44 and LaunchT.flags.offset == 48
    assert LaunchT.args.offset == 56 and C.sizeof(LaunchT) == 64
