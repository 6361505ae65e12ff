#!/bin/bash
# Time configurations of one problem under -D variants (TSG_EXTRA_DEFINES).
#   gpurun -- 'bash tools/gpu/exp.sh dedispersion tag "cfg;cfg" "" "DD_NOSLOTS=1" ...'
prob=$1; tag=$2; cfgs=$3; shift 3
mkdir -p gpurun_out
out=gpurun_out/exp_${prob}_$tag.jsonl; : > $out
for v in "$@"; do
  TSG_EXTRA_DEFINES="$v" timeout 900 python tools/run_configs.py $prob "$cfgs" --runs 7 \
    2>>gpurun_out/exp_${prob}_$tag.err | sed "s/^{/{\"variant\": \"$v\", /" >> $out
done
python - "$out" <<'PY'
import json, sys, collections
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
by = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows: by[tuple(r["config"])][r["variant"]].append(r["time_ms"] if r["status"] == "ok" else r["status"])
for c, v in by.items():
    print(c, "  ".join(f"[{k}]: " + "/".join(str(round(t, 4)) if isinstance(t, float) else str(t) for t in ts) for k, ts in v.items()))
PY
