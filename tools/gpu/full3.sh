# Full GPU pass: build, smoke, GPU tests, bench (all workloads), launch list,
# ncu --set full of each bench's best configuration (for roofline.traffic)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --dump gpurun_out/dump_hotspot_main.json > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in convolution gemm gemm_tc; do
  timeout 600 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_$w.json > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 900 python bench.py --workload dedispersion --steps 2 --warmup 1 --batch 12 --no-cpu-baseline --no-e2e --dump gpurun_out/dump_dedispersion.json > gpurun_out/bench_dedispersion.json 2> gpurun_out/bench_dedispersion.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --batch 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
for w in hotspot convolution gemm dedispersion; do
  f=gpurun_out/bench.json; [ $w != hotspot ] && f=gpurun_out/bench_$w.json
  cfg=$(python -c "import json,sys; d=json.loads(open('$f').read().splitlines()[-1]); print(','.join(str(v) for v in d['best_config']['config'].values()))" 2>/dev/null)
  [ -z "$cfg" ] && continue
  tag=$(echo $cfg | tr ',' '-')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${w}_kernel -s 1 -c 1 -o gpurun_out/prof_best_${w}_${tag} -f python tools/run_config.py $w $cfg --runs 1 > gpurun_out/ncu_best_$w.log 2>&1
done
# staged generic dedispersion (DD_STG) evidence
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dedispersion_kernel -s 1 -c 1 -o gpurun_out/prof_dd_staged_16-64-4-3-1-0 -f python tools/run_config.py dedispersion 16,64,4,3,1,0 --runs 1 > gpurun_out/ncu_dd_staged.log 2>&1
