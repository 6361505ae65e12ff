set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 16,4,4,1,4,2,1 32,2,4,1,8,2,1 32,16,3,2,6,6,1; do
timeout 600 python tools/dd_hotspot_bench.py --config $c >> gpurun_out/dd.jsonl 2>> gpurun_out/dd.err
done
