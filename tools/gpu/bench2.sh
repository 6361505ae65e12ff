set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --workload convolution --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_conv_r.json > gpurun_out/bench_conv_r.json 2> gpurun_out/bench_conv_r.err
timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_r.json > gpurun_out/bench_hs_r.json 2> gpurun_out/bench_hs_r.err
nvidia-smi -q | grep -i -A3 "persistence\|clocks event" > gpurun_out/nvsmi_q.txt 2>&1
