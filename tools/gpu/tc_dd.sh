#!/bin/bash
# tf32 tcgen05 GEMM: parity, its whole space timed (clocks sampled), cuBLAS
# tf32 for reference; dedispersion window-mode ncu capture + variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tc_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gemm_tc" > gpurun_out/pytest_tc.log 2>&1
tail -3 gpurun_out/pytest_tc.log
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 100 > gpurun_out/tc_clocks.csv 2>&1 &
smi=$!
timeout 900 python tools/run_configs.py gemm_tc --sample 24 --seed 1 > gpurun_out/tc_times.jsonl 2> gpurun_out/tc_times.err
kill $smi
python - <<'PY'
import json
for l in open("gpurun_out/tc_times.jsonl"):
    r = json.loads(l)
    t = r["time_ms"]
    print(r["config"], r["status"], t and round(t, 4), t and round(2 * 4096 ** 3 / t / 1e9, 1), "TFLOP/s")
PY
awk -F, 'NR>1 {print $2}' gpurun_out/tc_clocks.csv | sort | uniq -c | sort -rn | head -5
timeout 300 python tools/cublas_tf32.py
