mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for d in 8 4 8 4; do TSG_PIPELINE_DEPTH=$d timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_d${d}_$RANDOM.json 2>> gpurun_out/bench_d.err; done
