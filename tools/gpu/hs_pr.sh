set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hotspot" > gpurun_out/pytest_hs.log 2>&1
CF="32,2,4,1,8,2,1;32,4,4,1,7,7,1;32,2,4,1,10,1,1;32,2,4,1,9,2,1;32,2,4,1,6,2,1;32,4,4,1,8,2,1;64,1,4,1,8,2,1;32,1,4,1,8,2,1;32,2,2,1,8,2,1;32,2,6,1,7,2,1;32,4,4,1,5,5,1;32,2,4,1,7,2,1;64,2,4,1,8,2,1;32,1,4,1,7,1,1;32,2,4,2,8,2,1"
for rep in 1 2; do
TSG_HS_PR=exact timeout 600 python tools/run_configs.py hotspot "$CF" --runs 7 > gpurun_out/hs_pr_exact_$rep.jsonl 2> gpurun_out/hs_pr_exact.err
TSG_HS_PR=pow2 timeout 600 python tools/run_configs.py hotspot "$CF" --runs 7 > gpurun_out/hs_pr_pow2_$rep.jsonl 2> gpurun_out/hs_pr_pow2.err
done
