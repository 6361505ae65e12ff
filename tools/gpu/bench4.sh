set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
TSG_NVML_NO_SAMPLES=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_nvmlinit$i.json > gpurun_out/bench_hs_nvmlinit$i.json 2> /dev/null
TSG_NO_CLOCK_SAMPLER=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --dump gpurun_out/dump_hs_none$i.json > gpurun_out/bench_hs_none$i.json 2> /dev/null
done
