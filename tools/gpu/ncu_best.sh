#!/bin/bash
# ncu --set full of each kernel's best configuration (the bench line's
# roofline.traffic source) + the bench launch list, into gpurun_out/ncu/.
#   gpurun --timeout 2400 -- 'bash tools/gpu/ncu_best.sh'
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu/build.log 2>&1
cap() {  # problem config kernel-regex tag
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^($3)\$" -s 1 -c 1 \
    -o gpurun_out/ncu/ncu_$4 -f python tools/run_config.py $1 $2 --runs 2 > gpurun_out/ncu/$4.log 2>&1
  echo "$4 rc=$?"
}
cap hotspot 32,1,4,1,7,7,1 hotspot_kernel hotspot_stream_32-1-4-1-7-7-1
cap hotspot 32,2,4,1,8,2,1 hotspot_kernel hotspot_stream_32-2-4-1-8-2-1
cap convolution 256,2,4,4,1,0,0 convolution_kernel convolution_256-2-4-4-1-0-0
cap dedispersion 32,32,4,8,1,0 dedispersion_kernel dedispersion_window_32-32-4-8-1-0
cap gemm 128,64,16,16,8,16,8,4,4,1,1,1,1 gemm_kernel gemm_128-64-16-16-8-16-8-4-4-1-1-1-1
cap gemm_tc 256,6,2 gemm_tc_kernel gemm_tc_256-6-2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/ncu/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu/bench_under_ncu.log 2>&1
echo "launches rc=$?"
ls -la gpurun_out/ncu
