set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/hs_nr.jsonl
for nr in 4 8 16; do
  TSG_HS_NR=$nr timeout 600 python tools/run_configs.py hotspot "$1" | sed "s/^/$nr /" >> gpurun_out/hs_nr.jsonl 2>> gpurun_out/hs_nr.err
done
