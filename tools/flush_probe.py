"""Is the L2 flush big enough?  Times an L2-resident-sized read (96 MiB,
< the 126 MB L2) right after flushes of several sizes, inside the normal
protocol (tsg_run_timed: flush, event, kernel, event).  A flush that evicts
the buffer makes the read run at HBM speed like the 3 x L2 reference; a
too-small one leaves part of it in L2 and the read gets faster.

    python tools/flush_probe.py          (prints one JSON line per size)
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200 import runtime as rt  # noqa: E402

SRC = r'''
extern "C" __global__ void __launch_bounds__(512) read_sum(const float4* __restrict__ a, size_t n, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcg(a + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.678f) out[blockIdx.x] = s;  // keeps the loads alive
}
'''

dev = rt.Device(0)
l2 = dev.info["l2_bytes"]
res = rt.compile_source(SRC, ["--gpu-architecture=sm_100a"])
assert res.ok, res.error
rc, mod = dev.load(res.image)
k = mod.function("read_sum")
for mb in (96, 64):
    nbytes = mb << 20
    buf = dev.alloc(nbytes)
    out = dev.alloc(4 * 4096)
    dev.lib.tsg_memset32(dev.ctx, buf.ptr, 0, nbytes // 4)
    launch = rt.Launch(k, (dev.info["sm_count"] * 4, 1, 1), (512, 1, 1),
                       [C.c_uint64(buf.ptr), C.c_size_t(nbytes // 16), C.c_uint64(out.ptr)])
    for w, r in ((0, 0), (3.0, 0), (1.0, 0), (0.0, 1.0), (0.0, 1.5), (1.0, 1.0), (1.25, 1.25), (3.0, 1.5),
                 (1.0, 1.5)):
        if w or r:
            dev.lib.tsg_set_flush_bytes(dev.ctx, max(16, int(w * l2)), int(r * l2))
        rc, times = dev.run_timed([launch], 2, 15, flush_l2=bool(w or r))
        assert rc == rt.OK, times
        t = sorted(times)[len(times) // 2]
        print(json.dumps({"buffer_mib": mb, "write_x_l2": w, "read_x_l2": r, "median_us": round(t * 1e3, 2),
                          "gbs": round(nbytes / (t * 1e-3) / 1e9, 1), "l2_bytes": l2}), flush=True)
    buf.free()
    out.free()
dev.lib.tsg_set_flush_bytes(dev.ctx, 0, 0)
