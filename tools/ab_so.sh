#!/bin/bash
# A/B of library builds on one box: ab/<variant>.so files (built here from
# different sources) swapped in turn into the package, bench alternated
# ROUNDS times (default 2) so box drift shows. VARIANTS default "base new".
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIB=paper_2510_13333_b200/libnclopf_b200.so
cp $LIB /tmp/keep.so
for r in $(seq ${ROUNDS:-2}); do
  for v in ${VARIANTS:-base new}; do
    cp ab/$v.so $LIB
    timeout 600 python bench.py ${BENCH_ARGS:---no-solve --no-cpu-baseline --steps 30 --warmup 5} > gpurun_out/ab_$v.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$v','value',round(d['value'],4),'factor',round(d['config'].get('factor_ms'),4),'solve',round(d['config'].get('solve_ms'),4),'e2e',round(d['e2e']['value'],4))"
  done
done
cp /tmp/keep.so $LIB
