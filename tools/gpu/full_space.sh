#!/bin/bash
# Whole-space brute-force sweep of one kernel through the command line,
# resumable (the log survives a lost box), native + Kernel-Tuner caches.
#   gpurun --timeout 3600 -- 'bash tools/gpu/full_space.sh hotspot 3000'
k=$1; lim=${2:-3000}
mkdir -p gpurun_out/caches
timeout $lim python -m paper_2407_11488_b200 tune --space $k --backend cuda:$k --strategy brute \
  --resume gpurun_out/caches/$k.log.jsonl --out gpurun_out/caches/$k.tunescape.json \
  --kt-out gpurun_out/caches/$k.kerneltuner.json --chunk 64 > gpurun_out/caches/$k.out 2> gpurun_out/caches/$k.err
echo "sweep $k rc=$?"; tail -5 gpurun_out/caches/$k.out; tail -3 gpurun_out/caches/$k.err
