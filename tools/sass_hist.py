"""SASS opcode histogram + ptxas resources of one tuned configuration (no GPU needed).

    python tools/sass_hist.py hotspot 32,2,4,1,8,2,1 [--json out.json]

NVRTC compiles the configuration exactly as the tuner does (same source,
same options), then ``cuobjdump -sass`` / ``--dump-resource-usage`` read
the cubin.  Prints registers, spill bytes, shared memory and the opcode
counts per kernel (base mnemonic, modifiers stripped), e.g. to prove that
the tf32 GEMM issues UTCHMMA/UTMALDG and the hotspot stream kernel FFMA2.
"""
from __future__ import annotations

import argparse
import collections
import json
import re
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200 import runtime as rt  # noqa: E402
from paper_2407_11488_b200.problems import make_problem  # noqa: E402

CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"


def analyse(problem: str, config: tuple, **kw) -> dict:
    prob = make_problem(problem, **kw)
    cfg = dict(zip(prob.space.param_names, config))
    res = rt.compile_source(prob.source_for(cfg), prob.options(cfg))
    if not res.ok:
        raise SystemExit(f"compile failed: {res.error[:2000]}")
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(res.image)
        f.flush()
        sass = subprocess.run([CUOBJDUMP, "-sass", f.name], capture_output=True, text=True).stdout
        usage = subprocess.run([CUOBJDUMP, "--dump-resource-usage", f.name], capture_output=True,
                               text=True).stdout
    kernels: dict = {}
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = kernels.setdefault(m.group(1), collections.Counter())
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[\w.]+)?", ln)
        if m and cur is not None:
            cur[m.group(1)] += 1
    res_by_k = {}
    name = None
    for ln in usage.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", ln)
        if m and name:
            res_by_k[name] = dict(regs=int(m.group(1)), stack=int(m.group(2)), shared=int(m.group(3)),
                                  local=int(m.group(4)))
    out = {"problem": problem, "config": cfg, "compile_s": round(res.seconds, 3), "kernels": {}}
    for k, ops in kernels.items():
        out["kernels"][k] = {"resources": res_by_k.get(k), "total": sum(ops.values()),
                             "opcodes": dict(ops.most_common())}
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("problem")
    ap.add_argument("config")
    ap.add_argument("--json")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    r = analyse(a.problem, tuple(int(x) for x in a.config.split(",")))
    for k, v in r["kernels"].items():
        print(f"{k}: {v['resources']} total {v['total']} (NVRTC {r['compile_s']} s)")
        print("  " + ", ".join(f"{op} {n}" for op, n in list(v["opcodes"].items())[: a.top]))
    if a.json:
        Path(a.json).write_text(json.dumps(r, indent=1))


if __name__ == "__main__":
    main()
