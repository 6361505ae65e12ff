set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hotspot" > gpurun_out/pytest_hotspot.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --batch 60 --dump gpurun_out/dump_hotspot.json > gpurun_out/bench_hotspot.json 2> gpurun_out/bench_hotspot.err
