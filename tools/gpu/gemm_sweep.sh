set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --workload gemm --no-cpu-baseline --no-e2e --steps 4 --warmup 1 --batch 80 --seed 7 --dump gpurun_out/dump_gemm_sweep.json > gpurun_out/bench_gemm_sweep.json 2> gpurun_out/bench_gemm_sweep.err
