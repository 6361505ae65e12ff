set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hotspot.json > gpurun_out/bench_hotspot.json 2> gpurun_out/bench_hotspot.err
timeout 600 python bench.py --workload gemm --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_gemm.json > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err
