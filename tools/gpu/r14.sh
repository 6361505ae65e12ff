mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_1.json 2> gpurun_out/bench_e2e_1.err
TSG_E2E_FLUSH_MODULES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_0.json 2> gpurun_out/bench_e2e_0.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_2.json 2> gpurun_out/bench_e2e_2.err
