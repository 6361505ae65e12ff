#!/bin/bash
# Whole-space brute-force sweep of one kernel through the command line,
# resumable (the log survives a lost box), native + Kernel-Tuner caches,
# summary (tools/sweep_summary.py) and the UNMODIFIED reference's own
# `analyze stats` on the Kernel-Tuner cache; caches gzipped (gpurun copies
# back <= 64 MiB).
#   gpurun --timeout 3600 -- 'bash tools/gpu/full_space.sh hotspot 3000'
k=$1; lim=${2:-3000}
d=gpurun_out/caches; mkdir -p $d
t0=$(date +%s)
timeout $lim python -m paper_2407_11488_b200 tune --space $k --backend cuda:$k --strategy brute \
  --resume $d/$k.log.jsonl --out $d/$k.tunescape.json \
  --kt-out $d/$k.kerneltuner.json --chunk 64 > $d/$k.out 2> $d/$k.err
rc=$?; t1=$(date +%s)
echo "sweep $k rc=$rc wall=$((t1-t0))s"; tail -5 $d/$k.out; tail -3 $d/$k.err
if [ -f $d/$k.tunescape.json ]; then
  python tools/sweep_summary.py $k $d/$k.tunescape.json --wall-s $((t1-t0)) --out $d/$k.summary.json \
    --command "python -m paper_2407_11488_b200 tune --space $k --backend cuda:$k --strategy brute --out ... --kt-out ... --resume ..."
  PYTHONPATH=baseline/_ref python -m tunescape analyze stats --cache $d/$k.tunescape.json > $d/$k.reference_stats.txt 2>&1
  cat $d/$k.reference_stats.txt
  gzip -9f $d/$k.tunescape.json $d/$k.kerneltuner.json
  rm -f $d/$k.log.jsonl*
fi
du -sh gpurun_out
