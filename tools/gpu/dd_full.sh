mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
date +%s > gpurun_out/dd_full_t0.txt
timeout 2700 python -m paper_2407_11488_b200 tune --space dedispersion --backend cuda:dedispersion --strategy brute \
  --out gpurun_out/dedispersion_full.json --kt-out gpurun_out/dedispersion_full.kerneltuner.json \
  --resume gpurun_out/dedispersion_full.log.jsonl > gpurun_out/dd_full.log 2> gpurun_out/dd_full.err
echo rc=$? >> gpurun_out/dd_full.log
date +%s >> gpurun_out/dd_full_t0.txt
