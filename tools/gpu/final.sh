#!/bin/bash
# Round-end validation on one B200: GPU suite, smoke, bench lines (default,
# reference arm, domain-decomposed hotspot), ncu of the headline optimum.
mkdir -p gpurun_out
bash tools/gpu/check.sh
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --workload dd_hotspot --steps 5 --warmup 3 > gpurun_out/bench_final_dd.json 2> gpurun_out/bench_final_dd.err; echo "dd rc=$?"
bash tools/gpu/ncu_one.sh hotspot 8,8,4,1,7,7,1 hotspot_kernel hotspot_stream_8-8-4-1-7-7-1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/ncu/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu/bench_under_ncu.log 2>&1
echo "launches rc=$?"
