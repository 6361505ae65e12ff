set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dedispersion" > gpurun_out/pytest_dd.log 2>&1
CF="2,48,3,4,1,1;1,40,1,1,0,0;16,64,4,3,1,0;4,256,2,8,0,1;8,128,3,7,1,1;32,32,4,8,1,0"
TSG_DD_STG=all timeout 900 python tools/run_configs.py dedispersion "$CF" --sample 40 --seed 3 --param block_size_x --runs 3 > gpurun_out/dd_stg1.jsonl 2> gpurun_out/dd_stg1.err
TSG_DD_STG=0 timeout 900 python tools/run_configs.py dedispersion "$CF" --sample 40 --seed 3 --param block_size_x --runs 3 > gpurun_out/dd_stg0.jsonl 2> gpurun_out/dd_stg0.err
