set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TSG_NO_CLOCK_SAMPLER=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_ns.json > gpurun_out/bench_hs_ns.json 2> gpurun_out/bench_hs_ns.err
CUDA_MODULE_LOADING=EAGER timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_eager.json > gpurun_out/bench_hs_eager.json 2> gpurun_out/bench_hs_eager.err
