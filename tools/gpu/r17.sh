mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cap in 32 16384 32 16384 8; do TSG_RETIRE_CAP=$cap timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cap${cap}_$RANDOM.json 2>> gpurun_out/bench_cap.err; done
