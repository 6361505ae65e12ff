#!/bin/bash
# Parity of the window dedispersion and tf32 GEMM changes, then A/B timings.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dedispersion or gemm_tc" > gpurun_out/pytest_ab.log 2>&1
tail -3 gpurun_out/pytest_ab.log
bash tools/gpu/exp.sh dedispersion win "32,32,4,8,1,0;32,32,3,7,1,0;32,16,4,8,1,0;32,32,4,6,1,0" "" "DD_ONE=1" "DD_NOSLOTS=1" ""
bash tools/gpu/exp.sh gemm_tc band "256,6,2;256,5,2;256,4,1;256,4,2" "" "GEMM_BAND=1024" ""
