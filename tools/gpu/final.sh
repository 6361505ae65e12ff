#!/bin/bash
# Round-end validation on one B200: GPU suite, smoke, bench lines (default,
# reference arm, domain-decomposed hotspot), experiment A/B, ncu of the
# dedispersion best.
mkdir -p gpurun_out
bash tools/gpu/check.sh
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --workload dd_hotspot --steps 5 --warmup 3 > gpurun_out/bench_final_dd.json 2> gpurun_out/bench_final_dd.err; echo "dd rc=$?"
bash tools/gpu/ncu_one.sh dedispersion 32,32,4,8,1,0 dedispersion_kernel dedispersion_window_32-32-4-8-1-0
bash tools/gpu/ncu_one.sh gemm 128,64,16,8,8,16,16,4,4,1,1,1,1 gemm_kernel gemm_128-64-16-8-8-16-16-4-4-1-1-1-1
