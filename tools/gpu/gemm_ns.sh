set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/gemm_ns.jsonl
for ns in 2 3 4; do
  TSG_GEMM_NS=$ns timeout 600 python tools/run_configs.py gemm "$1" --runs 5 | sed "s/^/$ns /" >> gpurun_out/gemm_ns.jsonl 2>> gpurun_out/gemm_ns.err
done
