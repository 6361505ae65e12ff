set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dd_hotspot.py -q -x -m gpu -k "hotspot or stream or cuda_run" > gpurun_out/pytest_hs.log 2>&1
timeout 900 python tools/run_configs.py hotspot "$1" > gpurun_out/hs_cfgs.jsonl 2> gpurun_out/hs_cfgs.err
