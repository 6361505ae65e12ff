#!/bin/bash
# One ncu --set full capture (source-correlated) of one configuration's kernel,
# report + raw/source CSV pages into gpurun_out/ncu/.
#   gpurun -- 'bash tools/gpu/ncu_one.sh hotspot 32,2,4,1,8,2,1 hotspot_kernel tag [ENV=V ...]'
prob=$1; cfg=$2; kern=$3; tag=$4; shift 4
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu/build.log 2>&1
env "$@" timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^($kern)\$" -s 1 -c 1 \
  -o gpurun_out/ncu/ncu_$tag -f python tools/run_config.py $prob $cfg --runs 2 > gpurun_out/ncu/$tag.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ncu/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu/ncu_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu/ncu_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/ncu_${tag}_sass.csv 2>/dev/null
ls -la gpurun_out/ncu | tail -5
