mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/sweep_gaps.py hotspot --n 40 > gpurun_out/gaps_hotspot.jsonl 2> gpurun_out/gaps.err
timeout 600 python tools/sweep_gaps.py convolution --n 40 > gpurun_out/gaps_conv.jsonl 2>> gpurun_out/gaps.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
TSG_NVML_NO_SAMPLES=1 timeout 600 python bench.py --no-e2e > gpurun_out/bench_nosample.json 2> gpurun_out/bench_nosample.err
