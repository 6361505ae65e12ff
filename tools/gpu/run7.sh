set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/debug_gemm_tc.py > gpurun_out/debug_gemmtc.log 2>&1
timeout 600 python tools/dd_hotspot_bench.py --config 32,16,3,2,6,6,1 > gpurun_out/dd1.json 2> gpurun_out/dd1.err
