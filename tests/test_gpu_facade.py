"""tune_kernel / run_kernel on the GPU (Kernel-Tuner-style facade)."""

import numpy as np
import pytest

from paper_2407_11488_b200 import run_kernel, tune_kernel
from paper_2407_11488_b200.paramspace import space_from_tune_params
from paper_2407_11488_b200.store import import_external_cache

pytestmark = pytest.mark.gpu

VADD = r"""
extern "C" __global__ void vector_add(float* c, const float* a, const float* b, int n) {
    int i = blockIdx.x * block_size_x * tile + threadIdx.x;
    #pragma unroll
    for (int k = 0; k < tile; ++k, i += block_size_x)
        if (i < n) c[i] = a[i] + b[i];
}
"""

SCALE = r"""
__constant__ float coef[4];
template <typename T>
__global__ void scale(T* out, const T* in, int n) {
    int i = blockIdx.x * block_size_x + threadIdx.x;
    if (i < n) out[i] = in[i] * coef[i % 4];
}
"""


def test_tune_vector_add_with_answer(tmp_path):
    n = np.int32(1_000_003)
    a = np.random.default_rng(0).random(n, dtype=np.float32)
    b = np.random.default_rng(1).random(n, dtype=np.float32)
    c = np.zeros_like(a)
    tune_params = {"block_size_x": [64, 128, 256, 512, 1024, 2048], "tile": [1, 2, 4]}
    cache = tmp_path / "kt.json"
    results, env = tune_kernel("vector_add", VADD, n, [c, a, b, n], tune_params,
                               grid_div_x=["block_size_x", "tile"], answer=[a + b, None, None, None],
                               restrictions=["block_size_x * tile <= 4096"], cache=str(cache),
                               metrics={"GB/s": lambda p: 12 * n / (p["time"] * 1e6)})
    assert env["space_size"] == 17 and len(results) == 17
    ok = [r for r in results if r["status"] == "ok"]
    bad = [r for r in results if r["status"] != "ok"]
    assert all(r["block_size_x"] == 2048 for r in bad) and len(bad) == 2  # > 1024 threads
    assert all(r["status"] == "invalid" for r in bad)
    assert len(ok) == 15 and all(r["GB/s"] > 0 for r in ok)
    space = space_from_tune_params("vector_add", tune_params, ["block_size_x * tile <= 4096"])
    imported = import_external_cache(cache, expected_space=space)
    assert len(imported.records) == 17


def test_wrong_answer_is_runtime_failed():
    n = np.int32(4096)
    a = np.ones(n, np.float32)
    c = np.zeros_like(a)
    results, _ = tune_kernel("vector_add", VADD, n, [c, a, a, n], {"block_size_x": [128], "tile": [1]},
                             grid_div_x=["block_size_x", "tile"], answer=[a * 3, None, None, None])
    assert results[0]["status"] == "runtime_failed" and "verification" in results[0]["error"]


def test_run_kernel_template_and_cmem():
    n = np.int32(1000)
    x = np.arange(n, dtype=np.float32)
    out = np.zeros_like(x)
    coef = np.array([1, 2, 3, 4], np.float32)
    res = run_kernel("scale<float>", SCALE, n, [out, x, n], {"block_size_x": 128},
                     cmem_args={"coef": coef})
    np.testing.assert_array_equal(res[0], x * coef[np.arange(n) % 4])


@pytest.mark.parametrize("strategy", ["random_sample", "genetic_algorithm", "greedy_ls"])
def test_strategies_through_facade(strategy):
    n = np.int32(1 << 20)
    a = np.ones(n, np.float32)
    c = np.zeros_like(a)
    tp = {"block_size_x": [32, 64, 128, 256, 512, 1024], "tile": [1, 2, 4, 8]}
    results, env = tune_kernel("vector_add", VADD, n, [c, a, a, n], tp,
                               grid_div_x=["block_size_x", "tile"], strategy=strategy,
                               strategy_options={"max_fevals": 8, "seed": 3})
    assert 1 <= len(results) <= 8 and env["best_config"] is not None


def test_tsbench_through_command_backend():
    """The reference's cmd: route (same stdout contract) drives B200 kernels."""
    import sys

    from paper_2407_11488_b200.measure import MeasurementProtocol, command_backend, measure
    from paper_2407_11488_b200.paramspace import bundled_space

    space = bundled_space("hotspot")
    tpl = (f"{sys.executable} -m paper_2407_11488_b200.tsbench --kernel hotspot --size width=512,height=512 "
           "--config {block_size_x},{block_size_y},{tile_size_x},{tile_size_y},"
           "{temporal_tiling_factor},{loop_unroll_factor_t},{sh_power}")
    be = command_backend(tpl)
    obs = measure(be, (32, 8, 2, 2, 5, 5, 1), MeasurementProtocol(), space.param_names)
    assert obs.ok and len(obs.times_ms) == 7, obs


def test_unmodified_reference_tune_drives_b200_kernels(tmp_path):
    """The UNMODIFIED reference (tunescape installed under baseline/_ref by
    baseline/install_reference.sh) runs its own ``tune`` command line with a
    ``cmd:`` backend over tsbench: its random search, process protocol and
    stdout parsing measure B200 kernels, and its cache holds them."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    ref = root / "baseline" / "_ref"
    if not (ref / "tunescape" / "__init__.py").exists():
        pytest.skip("reference not installed (baseline/install_reference.sh)")
    tpl = (f"{sys.executable} -m paper_2407_11488_b200.tsbench --kernel hotspot --size width=1024,height=1024 "
           "--config {block_size_x},{block_size_y},{tile_size_x},{tile_size_y},"
           "{temporal_tiling_factor},{loop_unroll_factor_t},{sh_power}")
    out = tmp_path / "b200_via_reference.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ref), str(root)]))
    proc = subprocess.run([sys.executable, "-c", "import sys, tunescape.cli as c; "
                           "assert 'baseline/_ref' in c.__file__, c.__file__; sys.argv[0] = 'tunescape'; c.main()",
                           "tune", "--space", "hotspot", "--backend", f"cmd:{tpl}", "--strategy", "random",
                           "--budget", "3", "--seed", "5", "--out", str(out)],
                          capture_output=True, text=True, env=env, timeout=900, cwd=str(root))
    assert proc.returncode == 0, proc.stderr[-3000:]
    assert "evaluations : 3" in proc.stdout and "best config : " in proc.stdout, proc.stdout
    doc = json.loads(out.read_text())
    oks = [r for r in doc["records"].values() if r["status"] == "ok"]
    assert len(doc["records"]) == 3 and oks and all(len(r["times_ms"]) == 7 for r in oks)


TRAP_KERNEL = r"""
extern "C" __global__ void maybe_trap(float* c, const float* a, int n) {
  int i = blockIdx.x * block_size_x + threadIdx.x;
  if (block_size_x == 64) __trap();  // a device fault in exactly one configuration
  if (i < n) c[i] = a[i] * 2.0f;
}
"""

TRAP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2407_11488_b200 import tune_kernel
from paper_2407_11488_b200.cuda_backend import DevicePoisoned
n = 4096
a = np.ones(n, np.float32)
c = np.zeros_like(a)
try:
    tune_kernel("maybe_trap", sys.argv[2], n, [c, a, np.int32(n)], {"block_size_x": [32, 64, 128, 256]})
    print("NO-RAISE")
except DevicePoisoned as e:
    print("POISONED", e)
"""


def test_device_fault_stops_the_sweep(tmp_path):
    """A configuration that faults the device poisons the process's CUDA
    context; the sweep must stop with DevicePoisoned instead of recording
    fake failures for the configurations after it (they are re-measured by a
    restarted, resumed run).  Isolated in a subprocess: the context is dead
    afterwards."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    proc = subprocess.run([sys.executable, "-c", TRAP_SCRIPT, str(root), TRAP_KERNEL], capture_output=True,
                          text=True, timeout=600)
    assert "POISONED" in proc.stdout, (proc.stdout[-2000:], proc.stderr[-2000:])
