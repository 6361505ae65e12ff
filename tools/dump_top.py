"""Top configurations of a bench --dump file: python tools/dump_top.py dump.json [N] [param_index]"""
import collections
import json
import sys

d = json.load(open(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
rows = sorted((r for r in d["rows"] if r["status"] == "ok"), key=lambda r: r["time_ms"])
bad = collections.Counter(r["status"] for r in d["rows"] if r["status"] != "ok")
for r in rows[:n]:
    print(r["config"], round(r["time_ms"], 4), "regs", r["regs"], "smem", r["smem"],
          "launch_ms", [round(x, 4) for x in (r.get("launch_ms") or [])][:4])
print("ok", len(rows), "failed", dict(bad))
if len(sys.argv) > 3:
    pi = int(sys.argv[3])
    best = {}
    for r in rows:
        best.setdefault(r["config"][pi], r["time_ms"])
    print("best per param[%d]:" % pi, sorted((k, round(v, 4)) for k, v in best.items()))
