mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
uptime > gpurun_out/r20_uptime.txt; nproc >> gpurun_out/r20_uptime.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_r20_1.json > gpurun_out/bench_r20_1.json 2> gpurun_out/bench_r20_1.err
uptime >> gpurun_out/r20_uptime.txt
sleep 60
uptime >> gpurun_out/r20_uptime.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_r20_2.json > gpurun_out/bench_r20_2.json 2> gpurun_out/bench_r20_2.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_r20_3.json > gpurun_out/bench_r20_3.json 2> gpurun_out/bench_r20_3.err
uptime >> gpurun_out/r20_uptime.txt
