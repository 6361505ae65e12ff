set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dd_hotspot.py -q -x -m gpu -k "hotspot or stream or cuda_run" > gpurun_out/pytest_hs.log 2>&1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_f$i.json > gpurun_out/bench_hs_f$i.json 2>/dev/null; done
