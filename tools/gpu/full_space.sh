#!/bin/bash
# Whole-space brute-force sweep of one kernel through the command line,
# resumable across gpurun calls: the resume log comes back gzipped in
# gpurun_out/caches/ -- move it to sweeps/ (git-ignored, travels with the
# snapshot) and the next call continues from it.  When complete: native +
# Kernel-Tuner caches (gzipped; gpurun copies back <= 64 MiB), summary
# (tools/sweep_summary.py) and the UNMODIFIED reference's `analyze stats`.
#   gpurun --timeout 3600 -- 'bash tools/gpu/full_space.sh hotspot 3000'
k=$1; lim=${2:-3000}
d=gpurun_out/caches; mkdir -p $d
[ -f sweeps/$k.log.jsonl.gz ] && gunzip -c sweeps/$k.log.jsonl.gz > $d/$k.log.jsonl && echo "resuming: $(wc -l < $d/$k.log.jsonl) logged"
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
else
  gzip -9f $d/$k.log.jsonl  # partial: bring the resume log back
fi
du -sh gpurun_out
