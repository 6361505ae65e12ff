"""Collect per-launch DRAM traffic from the committed ncu summaries.

    python tools/traffic_table.py [profiles/round1 profiles/round1/final ...] > profiles/traffic.json

Each ``ncu_<kernel>[_<mode>]_<c-o-n-f-i-g>.md`` summary (tools/ncu_summary.py
output of one ``ncu --set full`` capture) gives dram__bytes_read.sum +
dram__bytes_write.sum for one launch of that configuration; bench.py reports
it as ``roofline.traffic`` when its best configuration was profiled.
Files are read in name order; later captures of a configuration win.
"""

import json
import re
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(*dirs: str) -> None:
    out: dict = {}
    files = [f for d in (dirs or ("profiles/round1", "profiles/round1/final")) for f in sorted(Path(d).glob("ncu_*.md"))]
    for f in files:  # directories in order: later captures win
        m = re.match(r"ncu_([a-z_]+?)(?:_(?:stream|window|staged))?_([0-9-]+)\.md$", f.name)
        if not m:
            continue
        kernel, cfg = m.group(1), m.group(2).replace("-", ",")
        text = f.read_text()
        vals = {}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            mm = re.search(r"`" + re.escape(key) + r"`\) \| ([0-9.]+) (\w+)", text)
            if mm:
                vals[key] = (float(mm.group(1)), mm.group(2))
        if "dram__bytes_read.sum" not in vals:
            continue
        b = sum(v * SCALE.get(u, 1) for k, (v, u) in vals.items() if k.startswith("dram"))
        out.setdefault(kernel, {})[cfg] = {"dram_bytes": b, "source": str(f)}
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(*sys.argv[1:])
