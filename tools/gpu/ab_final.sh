#!/bin/bash
# A/B of the last experiment macros (verified on the device by run_configs).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abf_build.log 2>&1
bash tools/gpu/exp.sh hotspot skip "32,1,4,1,7,7,1;32,2,4,1,8,2,1;64,1,4,1,5,5,1;1,32,4,1,10,5,1;32,4,4,1,7,7,1" "" "HS_SKIP=1" "" "HS_SKIP=1"
bash tools/gpu/exp.sh dedispersion quad "32,32,4,8,1,0;32,16,4,8,1,0" "" "DD_QUAD=1" "" "DD_QUAD=1"
