#!/bin/bash
# Bench lines (default workload + options given as args), stdout to gpurun_out/bench_<tag>.json
#   gpurun -- 'bash tools/gpu/bench.sh v1 --steps 5 --warmup 3'
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "rc=$?"
tail -c 3000 gpurun_out/bench_$tag.json
