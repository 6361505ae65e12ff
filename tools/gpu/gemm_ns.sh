mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CF="64,128,16,8,8,8,8,8,4,1,1,1,1;64,128,16,8,8,16,32,4,4,0,0,1,1;128,128,16,16,16,16,16,4,4,0,0,1,1;128,64,16,16,8,16,8,4,4,1,1,1,1"
for ns in 2 3 4; do TSG_GEMM_NS=$ns timeout 600 python tools/run_configs.py gemm "$CF" --runs 5 > gpurun_out/gemm_ns$ns.jsonl 2>> gpurun_out/gemm_ns.err; done
