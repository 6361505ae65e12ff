set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm" > gpurun_out/pytest_gemm.log 2>&1
timeout 900 python tools/run_configs.py gemm "128,128,16,32,8,16,16,4,4,0,0,1,1;128,128,32,32,8,16,16,4,4,0,0,1,1;128,128,16,16,16,16,16,4,4,0,0,1,1;128,128,16,16,16,16,16,8,8,0,0,1,1;128,128,16,32,8,32,8,4,4,0,0,1,1;128,64,16,16,16,16,16,4,4,0,0,1,1;64,128,16,16,16,16,16,4,4,0,0,1,1;128,128,32,16,16,16,16,8,8,0,0,1,1;128,128,16,8,32,8,32,8,4,0,0,1,1;128,128,16,16,8,16,8,8,4,0,0,1,1" --runs 3 > gpurun_out/gemm_cfgs.jsonl 2> gpurun_out/gemm_cfgs.err
