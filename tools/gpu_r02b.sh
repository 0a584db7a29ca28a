#!/bin/bash
# round-2 call B: ncu --set full of the current factor / solve / assembly kernels at 500x256
# (KERNELS = regexes over demangled names; default: the factor and solve kernels)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
KL=${KERNELS:-"reg_factor_kernel factor_kernel<.int.32> factor_kernel<.int.256> reg_solve_kernel fwd_kernel<.int.32> bwd_kernel<.int.32> fwd_kernel<.int.256> bwd_kernel<.int.256> maxdiag_kernel"}
for k in $KL; do
  n=$(echo "$k" | tr -d '<>.' )
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${k}" -s 1 -c 1 \
    -o gpurun_out/b_prof_${n} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/b_ncu_${n}.log 2>&1; echo "ncu $k rc=$?"
done
if [ -z "$KERNELS" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kkt_assemble_compact -s 2 -c 1 \
  -o gpurun_out/b_prof_kkt_assemble_compact -f python tools/prof_ipm.py > gpurun_out/b_ncu_kkt.log 2>&1; echo "ncu kkt rc=$?"
fi
ls gpurun_out | grep b_prof
