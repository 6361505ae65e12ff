# ncu --set full of the current best hotspot configuration (+ source page)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hotspot_kernel -s 4 -c 1 -o gpurun_out/prof_hotspot_best -f python tools/run_config.py hotspot 32,16,3,2,6,6,1 --runs 2 > gpurun_out/ncu_hotspot_best.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --batch 60 --dump gpurun_out/dump_hotspot.json > gpurun_out/bench_hotspot.json 2> gpurun_out/bench_hotspot.err
