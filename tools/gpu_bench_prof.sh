#!/bin/bash
# One gpurun call: GPU tests, bench line, ncu launch list, ncu full capture of the factor kernel.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL:-factor_kernel}" -s 2 -c ${NCU_COUNT:-2} \
  -o gpurun_out/prof_${NCU_NAME:-factor} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
