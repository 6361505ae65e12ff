set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm_tc or dedispersion" > gpurun_out/pytest_gemmtc.log 2>&1
timeout 600 python bench.py --workload gemm_tc --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_gemmtc.json 2> gpurun_out/bench_gemmtc.err
timeout 600 python bench.py --workload dedispersion --steps 1 --warmup 1 --batch 6 --no-cpu-baseline --no-e2e > gpurun_out/bench_dedisp.json 2> gpurun_out/bench_dedisp.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/prof_gemmtc -f python tools/run_config.py gemm_tc 256,4 --runs 1 > gpurun_out/ncu_gemmtc.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dedispersion_kernel -s 1 -c 1 -o gpurun_out/prof_dedisp2 -f python tools/run_config.py dedispersion 2,48,3,4,1,1 --runs 1 > gpurun_out/ncu_dedisp2.log 2>&1
