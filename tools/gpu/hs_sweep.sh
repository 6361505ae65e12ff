set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 1 --batch 300 --seed 99 --dump gpurun_out/dump_hs_sweep.json > gpurun_out/bench_hs_sweep.json 2> gpurun_out/bench_hs_sweep.err
