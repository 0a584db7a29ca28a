#!/bin/bash
# One gpurun call: GPU tests (optional filter), bench line, ncu launch list.
#   TAG=r02b TESTS="tests/test_ldlt_gpu.py" BENCH_ARGS="..." NCU=1 tools/gpu_run.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/${T}_gpu.txt
if [ "${TESTS}" != "none" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/${T}_gpu_tests.log 2>&1
  echo "tests rc=$?"; tail -3 gpurun_out/${T}_gpu_tests.log
fi
if [ "${BENCH}" != "none" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  echo "bench rc=$?"; tail -c 2500 gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/${T}_ncu_launch.log 2>&1
  echo "ncu rc=$?"
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
