#!/bin/bash
# round-2 call A: split-phase shard tests, FP64 peaks, traces, ncu of the IPM kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/a_gpu.txt
timeout 900 python -m pytest tests/test_shard.py -m gpu -x -q > gpurun_out/a_shard_tests.log 2>&1; echo "shard rc=$?"; tail -3 gpurun_out/a_shard_tests.log
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak fp64_peak.cu && timeout 120 /tmp/fp64_peak) > gpurun_out/a_fp64_peak.txt 2>&1; cat gpurun_out/a_fp64_peak.txt
timeout 600 python tools/gpu_solve.py activsg500 256 --trace gpurun_out/a_trace_500x256.json > gpurun_out/a_solve.log 2>&1; echo "solve rc=$?"; head -c 1500 gpurun_out/a_solve.log
timeout 300 python tools/gpu_solve.py activsg500 16 --trace gpurun_out/a_trace_500x16.json > gpurun_out/a_solve16.log 2>&1
for k in eval_kernel gather_sum64 kkt_assemble_kernel elem_kernel reduce_kernel csr_mv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 2 -c 1 \
    -o gpurun_out/a_prof_${k} -f python tools/prof_ipm.py > gpurun_out/a_ncu_${k}.log 2>&1; echo "ncu $k rc=$?"
done
for k in fwd_kernel bwd_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k}" -s 3 -c 3 \
    -o gpurun_out/a_prof_${k} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/a_ncu_${k}.log 2>&1; echo "ncu $k rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bf_syrk_dmma" -s 4 -c 2 \
  -o gpurun_out/a_prof_bf_syrk_dmma -f python bench.py --grid activsg2000 --K 64 --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/a_ncu_dmma.log 2>&1; echo "ncu dmma rc=$?"
ls gpurun_out
