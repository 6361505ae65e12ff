set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_p$i.json > gpurun_out/bench_hs_p$i.json 2>/dev/null; done
timeout 600 python bench.py --workload convolution --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_conv_p.json 2>/dev/null
