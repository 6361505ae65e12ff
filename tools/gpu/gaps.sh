mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/sweep_gaps.py hotspot --n 40 > gpurun_out/gaps_hotspot.jsonl 2> gpurun_out/gaps.err
timeout 600 python tools/sweep_gaps.py convolution --n 40 > gpurun_out/gaps_conv.jsonl 2>> gpurun_out/gaps.err
timeout 900 python -m pytest tests/test_gpu_facade.py tests/test_gpu_pipeline.py -q > gpurun_out/pytest_facade.log 2>&1
