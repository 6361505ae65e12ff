set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dedispersion" > gpurun_out/pytest_dd.log 2>&1
timeout 900 python tools/run_configs.py dedispersion "32,32,4,8,1,0;32,32,2,8,1,0;32,32,3,8,1,0;32,32,4,4,1,0;32,32,1,8,0,0;32,32,4,6,1,0;2,48,3,4,1,1;32,32,4,8,1,1" --runs 3 > gpurun_out/dd_cfgs.jsonl 2> gpurun_out/dd_cfgs.err
