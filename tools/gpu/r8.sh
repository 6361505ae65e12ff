mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_facade.py tests/test_cli.py -q -m gpu > gpurun_out/pytest_pipe.log 2>&1
for i in 1 2; do
timeout 600 python tools/sweep_gaps.py convolution --n 40 > gpurun_out/gaps_conv_$i.jsonl 2>> gpurun_out/gaps.err
timeout 600 python bench.py --no-e2e > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
done
