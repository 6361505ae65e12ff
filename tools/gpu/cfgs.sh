# usage: bash tools/gpu/cfgs.sh <problem> "<cfg;cfg;...>" [pytest -k expr]
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
[ -n "$3" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "$3" > gpurun_out/pytest_cfgs.log 2>&1
timeout 900 python tools/run_configs.py $1 "$2" > gpurun_out/cfgs.jsonl 2> gpurun_out/cfgs.err
