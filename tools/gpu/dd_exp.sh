#!/bin/bash
# Dedispersion experiment: time configs under TSG_EXTRA_DEFINES variants.
#   gpurun -- 'bash tools/gpu/dd_exp.sh tag "cfg;cfg" "" "DD_PF=1" ...'
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
out=gpurun_out/dd_exp_$tag.jsonl; : > $out
for v in "$@"; do
  TSG_EXTRA_DEFINES="$v" timeout 900 python tools/run_configs.py dedispersion "$cfgs" --runs 7 \
    2>>gpurun_out/dd_exp_$tag.err | sed "s/^{/{\"variant\": \"$v\", /" >> $out
done
python - "$out" <<'PY'
import json, sys, collections
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
by = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows: by[tuple(r["config"])][r["variant"]].append(r["time_ms"] if r["status"] == "ok" else r["status"])
for c, v in by.items():
    print(c, "  ".join(f"[{k}]: " + "/".join(str(round(t, 4)) if isinstance(t, float) else str(t) for t in ts) for k, ts in v.items()))
PY
