set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2407_11488_b200 import runtime as rt
from paper_2407_11488_b200.sweep import fp32_peak
print(fp32_peak(rt.Device(0)))
" > gpurun_out/peak.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hotspot_kernel -s 4 -c 1 -o gpurun_out/prof_hotspot_best -f python tools/run_config.py hotspot 32,16,3,2,6,6,1 --runs 2 > gpurun_out/ncu_hotspot_best.log 2>&1
