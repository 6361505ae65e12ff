import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_11488_b200 import runtime as rt  # noqa: E402

dev = rt.Device(0)
src = (Path(__file__).parent / "cuda" / "tmem_probe.cu").read_text()
res = rt.compile_source(src, ["--gpu-architecture=sm_100a"])
assert res.ok, res.error
rc, mod = dev.load(res.image)
k = mod.function("tmem_probe")
out = dev.alloc(4 * 1024)
for variant in (0, 1):
    dev._check(dev.lib.tsg_memset32(dev.ctx, out.ptr, 0x7FC00000, 1024))
    rc, err = dev.run([rt.Launch(k, (1, 1, 1), (128, 1, 1), [C.c_uint64(out.ptr), C.c_int(variant)])])
    h = np.empty(1024, np.float32)
    out.download(h)
    print("variant", variant, "rc", rc, err, "thread 37:", h[37 * 4: 37 * 4 + 4], "expect", [37 * 100 + 4 + j for j in range(4)],
          "tmem", hex(h.view(np.uint32)[512]))
