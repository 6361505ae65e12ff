set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_cli.py -q -x -m gpu > gpurun_out/pytest_cli.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small_problem" > gpurun_out/pytest_small.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload dedispersion > gpurun_out/bench_dd.json 2> gpurun_out/bench_dd.err
