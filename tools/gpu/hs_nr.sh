set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CF="32,2,4,1,8,2,1;32,4,4,1,7,7,1;32,4,4,1,8,2,1;64,1,4,1,8,2,1;32,2,4,1,7,2,1;64,2,4,1,8,2,1;32,8,4,1,8,2,1;32,2,4,1,6,2,1;32,2,4,1,8,1,1;32,4,4,1,7,1,1"
for nr in 4 6 16; do
TSG_HS_NR=$nr timeout 600 python tools/run_configs.py hotspot "$CF" --runs 7 > gpurun_out/hs_nr_$nr.jsonl 2> gpurun_out/hs_nr_$nr.err
done
