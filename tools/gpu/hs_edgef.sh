set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/hs_edgef.jsonl
for f in 0.25 0.35 0.45; do
  TSG_HS_EDGE_SEG=$f timeout 600 python tools/run_configs.py hotspot "$1" | sed "s/^/$f /" >> gpurun_out/hs_edgef.jsonl 2>> gpurun_out/hs_edgef.err
done
