import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_11488_b200 import runtime as rt  # noqa: E402

dev = rt.Device(0)
src = (Path(__file__).parent / "cuda" / "mma_probe.cu").read_text()
res = rt.compile_source(src, ["--gpu-architecture=sm_100a"])
assert res.ok, res.error
rc, mod = dev.load(res.image)
k = mod.function("mma_probe")
k.set_max_dynamic_smem(64 * 1024)
out = dev.alloc(4 * 1024)
cases = [(0, 128, 256), (0, 256, 128), (1, 128, 1024), (1, 1024, 128), (3, 1024, 4096), (3, 4096, 1024),
         (2, 16, 1024), (0, 16, 128)]
for variant, lbo, sbo in cases:
    dev._check(dev.lib.tsg_memset32(dev.ctx, out.ptr, 0x7FC00000, 1024))
    rc, err = dev.run([rt.Launch(k, (1, 1, 1), (128, 1, 1), [C.c_uint64(out.ptr), C.c_int(variant),
                                                             C.c_uint32(lbo), C.c_uint32(sbo)], smem=64 * 1024)],
                      timeout_ms=3000)
    h = np.empty(1024, np.float32)
    if rc == 0:
        out.download(h)
    print(f"variant {variant} lbo {lbo} sbo {sbo}: rc {rc} {err} D[0,:4]={h[:4]} D[77,:]={h[77*4:77*4+4]}"
          f" base={hex(h.view(np.uint32)[600])}", flush=True)
    if rc != 0:
        break
