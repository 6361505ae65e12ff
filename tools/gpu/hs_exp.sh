#!/bin/bash
# Hotspot stream-kernel experiment: time a config list under env variants
# (input ring depth TSG_HS_NR, power prefetch distance TSG_HS_PD, ...;
# "X=Y" sets TSG_HS_X=Y, "D:NAME=V" adds -DNAME=V via TSG_EXTRA_DEFINES).
#   gpurun -- 'bash tools/gpu/hs_exp.sh tag "cfg;cfg" "NR=16,PD=14" "NR=16,PD=6" ...'
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
out=gpurun_out/hs_exp_$tag.jsonl; : > $out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hs_exp_build.log 2>&1
for v in "$@"; do
  envs=""; defs=""
  for kv in $(echo "$v" | tr ',' ' '); do
    case $kv in D:*) defs="$defs,${kv#D:}";; *) envs="$envs TSG_HS_$kv";; esac
  done
  env $envs TSG_EXTRA_DEFINES="${defs#,}" timeout 600 python tools/run_configs.py hotspot "$cfgs" --runs 7 \
    2>>gpurun_out/hs_exp_$tag.err | sed "s/^{/{\"variant\": \"$v\", /" >> $out
done
python - "$out" <<'PY'
import json, sys, collections
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
by = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows: by[tuple(r["config"])][r["variant"]].append(r["time_ms"] if r["status"] == "ok" else r["status"])
for c, v in by.items():
    print(c, "  ".join(f"{k}: " + "/".join(str(round(t, 4)) if isinstance(t, float) else str(t) for t in ts) for k, ts in v.items()))
PY
