#!/bin/bash
# tf32 tcgen05 GEMM parity + timing of its space; dedispersion window-mode ncu capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tc_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gemm_tc" > gpurun_out/pytest_tc.log 2>&1
tail -3 gpurun_out/pytest_tc.log
timeout 600 python tools/run_configs.py gemm_tc --sample 24 --seed 1 > gpurun_out/tc_times.jsonl 2> gpurun_out/tc_times.err
cat gpurun_out/tc_times.jsonl | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], r['status'], r['time_ms'] and round(r['time_ms'],4), r['time_ms'] and round(2*4096**3/r['time_ms']/1e9,1), 'TFLOP/s')"
