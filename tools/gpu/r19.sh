mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -k "dedispersion or pipeline or pipelined" > gpurun_out/pytest_dd2.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
TSG_DD_STG=all timeout 900 python tools/run_configs.py dedispersion "4,256,4,8,0,0;8,256,4,8,1,1;16,64,4,8,0,1;32,32,4,8,0,0;4,256,4,7,1,0" --runs 2 > gpurun_out/dd_wide.jsonl 2> gpurun_out/dd_wide.err
timeout 900 python bench.py --workload dedispersion --steps 2 --warmup 1 --batch 12 --no-cpu-baseline --no-e2e > gpurun_out/bench_dd.json 2> gpurun_out/bench_dd.err
