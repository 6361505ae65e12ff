# usage: bash tools/gpu/ncu_cfg.sh <problem> <config> <tag> [kernel-regex] [skip]
set -x
mkdir -p gpurun_out
[ -f paper_2407_11488_b200/libtsgpu.so ] || python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${4:-$1_kernel} -s ${5:-2} -c 1 -o gpurun_out/prof_$3 -f python tools/run_config.py $1 $2 --runs 2 > gpurun_out/ncu_$3.log 2>&1
