set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CF="32,2,4,1,8,2,1;32,4,4,1,7,7,1;32,2,4,1,10,1,1;32,2,4,1,6,2,1;32,4,4,1,8,2,1;64,1,4,1,8,2,1;32,1,4,1,8,2,1;32,2,2,1,8,2,1;32,4,4,1,5,5,1;32,2,4,1,7,2,1;64,2,4,1,8,2,1;32,1,4,1,7,1,1;32,8,4,1,8,2,1;32,2,8,1,8,2,1;32,2,4,1,4,2,1"
for f in 1 0.75 0.5 0.34; do
TSG_HS_OCC_FRAC=$f timeout 600 python tools/run_configs.py hotspot "$CF" --runs 7 > gpurun_out/hs_occ_$f.jsonl 2> gpurun_out/hs_occ.err
done
