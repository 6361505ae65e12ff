mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for f in 1 0 1 0 1; do TSG_PRE_FLUSH_MODULES=$f timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pf${f}_$RANDOM.json 2>> gpurun_out/bench_pf.err; done
