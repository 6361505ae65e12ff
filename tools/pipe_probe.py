"""FMA-pipe latency/throughput of FFMA vs packed FFMA2 on this GPU.

Prints cycles per instruction per warp for C chains x W warps/SM:
latency ~ cycles at C=1,W=1; issue interval ~ cycles at large C*W.
"""
import ctypes as Cty
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_11488_b200 import runtime as rt  # noqa: E402

src = (Path(__file__).parent / "cuda" / "pipe_probe.cu").read_text()
dev = rt.Device(0)
sms = dev.info["sm_count"]
clk = dev.info["clock_khz"] * 1e3
out = dev.alloc(1 << 16)
iters = 4096
res = []
for c in (1, 2, 4, 8):
    r = rt.compile_source(src, ["--gpu-architecture=sm_100a", f"-DC={c}"])
    rc, mod = dev.load(r.image)
    for name in ("ffma_chain", "ffma2_chain"):
        k = mod.function(name)
        for w in (1, 2, 4, 8, 16):
            la = rt.Launch(k, (sms, 1, 1), (32 * w, 1, 1),
                           [Cty.c_uint64(out.ptr), Cty.c_int(iters), Cty.c_float(0.999), Cty.c_float(1e-3)])
            rc, t = dev.run_timed([la], 1, 3, flush_l2=False)
            ms = min(t)
            n_inst = iters * 16 * c  # per thread (= per warp, in order)
            cyc = ms * 1e-3 * clk
            res.append({"op": name, "chains": c, "warps_per_sm": w, "ms": ms,
                        "cycles_per_inst_per_warp": cyc / n_inst,
                        "sm_inst_per_cycle": n_inst * w / cyc})
    mod.unload()
for x in res:
    print(json.dumps(x))
