#!/bin/bash
# Hotspot stream-kernel experiment: time a config list under env variants
# (input ring depth TSG_HS_NR, power prefetch distance TSG_HS_PD, ...).
#   gpurun -- 'bash tools/gpu/hs_exp.sh tag "cfg;cfg" "NR=16,PD=14" "NR=16,PD=6" ...'
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
out=gpurun_out/hs_exp_$tag.jsonl; : > $out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hs_exp_build.log 2>&1
for v in "$@"; do
  envs=$(echo "$v" | tr ',' '\n' | sed 's/^/TSG_HS_/' | tr '\n' ' ')
  env $envs timeout 600 python tools/run_configs.py hotspot "$cfgs" --runs 7 2>>gpurun_out/hs_exp_$tag.err \
    | sed "s/^{/{\"variant\": \"$v\", /" >> $out
done
python - "$out" <<'PY'
import json, sys, collections
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
by = collections.defaultdict(dict)
for r in rows: by[tuple(r["config"])][r["variant"]] = (r["time_ms"], r["status"], r.get("launch_ms"))
for c, v in by.items():
    print(c, "  ".join(f"{k}: {t[0] if t[0] is None else round(t[0], 4)} {t[1] if t[1] != 'ok' else ''}" for k, t in v.items()))
PY
