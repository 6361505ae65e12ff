"""Real ptxas register counts of the hotspot stream kernel vs the host estimate.

    python tools/hs_regs.py        (no GPU needed: NVRTC + cuobjdump)

Prints (TSX, T, two-rows-per-iteration, ptxas regs, estimate) for a sample
of stream configurations; problems.Hotspot.stream_geometry's estimate gates
stream eligibility against the __launch_bounds__ register budget.
"""
import math
import random
import re
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_11488_b200 import runtime as rt  # noqa: E402
from paper_2407_11488_b200.problems import Hotspot  # noqa: E402

h = Hotspot()
names = h.space.param_names
random.seed(1)
cands = [(32, 2, tsx, 1, t, u, 1) for tsx in (1, 2, 3, 4, 5, 6, 8) for t in (1, 2, 3, 4, 5, 6, 7, 8, 10)
         for u in (1, 2) if t % u == 0]
random.shuffle(cands)
rows = []
for c in cands[:40]:
    if not h.space.is_valid(c):
        continue
    d = dict(zip(names, c))
    t, tsx = d["temporal_tiling_factor"], d["tile_size_x"]
    est = math.ceil(3.5 * t * tsx) + Hotspot.STREAM_REG_BASE + (12 * t if tsx % 2 else 0)
    opts = [o for o in h.options(d) if not o.startswith("-DHS_STREAM")] + ["-DHS_STREAM=1"]
    r = rt.compile_source(h.source(), opts)
    if not r.ok:
        print("compile failed", c, r.error[:200])
        continue
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(r.image)
        f.flush()
        out = subprocess.run(["cuobjdump", "-res-usage", f.name], capture_output=True, text=True).stdout
    m = re.findall(r"Function hotspot_kernel:\s*REG:(\d+)", out)
    rows.append((tsx, t, d["loop_unroll_factor_t"] > 1, int(m[0]) if m else None, est))
for r in sorted(rows):
    print(r)
