# bench-only refresh of the final pass (all workloads + launch list)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --dump gpurun_out/dump_hotspot_main.json > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in convolution gemm gemm_tc; do
  timeout 600 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_$w.json > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 900 python bench.py --workload dedispersion --steps 2 --warmup 1 --batch 12 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_dedispersion.json > gpurun_out/bench_dedispersion.json 2> gpurun_out/bench_dedispersion.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --batch 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
