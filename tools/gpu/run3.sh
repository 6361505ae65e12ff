set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "hotspot" > gpurun_out/pytest_hotspot.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_hotspot.json 2> gpurun_out/bench_hotspot.err
timeout 600 python bench.py --workload convolution --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_conv.json 2> gpurun_out/bench_conv.err
timeout 600 python bench.py --workload gemm --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err
timeout 600 python bench.py --workload dedispersion --steps 1 --warmup 1 --batch 6 --no-cpu-baseline --no-e2e > gpurun_out/bench_dedisp.json 2> gpurun_out/bench_dedisp.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hotspot_kernel -s 2 -c 1 -o gpurun_out/prof_hotspot -f python tools/run_config.py hotspot 16,16,4,2,10,1,1 --runs 2 > gpurun_out/ncu_hotspot.log 2>&1
