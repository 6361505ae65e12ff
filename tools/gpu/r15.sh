mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_v_$i.json > gpurun_out/bench_v_$i.json 2> gpurun_out/bench_v_$i.err; done
