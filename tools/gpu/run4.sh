set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "hotspot" > gpurun_out/pytest_hotspot.log 2>&1
timeout 600 python -m pytest tests/test_gpu_facade.py -q > gpurun_out/pytest_facade.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_hotspot.json 2> gpurun_out/bench_hotspot.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hotspot_kernel -s 2 -c 1 -o gpurun_out/prof_hotspot2 -f python tools/run_config.py hotspot 16,16,4,2,10,1,1 --runs 2 > gpurun_out/ncu_hotspot2.log 2>&1
