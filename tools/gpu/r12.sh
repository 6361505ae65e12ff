mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_hotspot_geometry.py tests/test_dd_hotspot.py -q -k "hotspot or stream" > gpurun_out/pytest_hs.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
for i in 1 2; do timeout 600 python bench.py --no-e2e > gpurun_out/bench_nr_$i.json 2> gpurun_out/bench_nr_$i.err; done
