#!/bin/bash
# One gpurun call producing every artefact profiles/ keeps for a round:
# traffic (ncu dram bytes of one refactorization) -> profiles/factor_traffic_<grid>x<K>.json,
# GPU tests, smoke, the bench line (reads that traffic), the reference arm,
# the ncu launch list, one ncu --set full capture of the factor kernels and a
# per-task timeline of one factorization.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve \
  > gpurun_out/ncu_traffic.log 2>&1
python tools/factor_traffic.py gpurun_out/traffic.csv activsg500x256 && cp profiles/factor_traffic_activsg500x256.json gpurun_out/
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/traffic2000.csv python bench.py --grid activsg2000 --K 64 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-solve > gpurun_out/ncu_traffic2000.log 2>&1
python tools/factor_traffic.py gpurun_out/traffic2000.csv activsg2000x64 && cp profiles/factor_traffic_activsg2000x64.json gpurun_out/
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 1500 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --grid activsg2000 --K 64 --steps 10 --warmup 3 --no-solve > gpurun_out/bench_2000x64.json 2> gpurun_out/bench_2000x64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"factor_kernel" -s 4 -c 4 \
  -o gpurun_out/prof_factor -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve \
  > gpurun_out/ncu_full.log 2>&1
NCL_TASK_TRACE=gpurun_out/trace.bin NCL_SOLVE_TRACE=gpurun_out/strace.bin timeout 300 python bench.py --steps 3 --warmup 1 \
  --no-cpu-baseline --no-solve > gpurun_out/trace.log 2>&1
# the B200 NCL solve's full-precision iterate trace (tools/parity_record.py against the committed reference traces)
NCL_ANALYZE_TIMING=1 timeout 600 python tools/gpu_solve.py activsg500 256 --trace gpurun_out/b200_trace_500x256.json \
  > gpurun_out/solve_500x256.log 2>&1
ls gpurun_out
