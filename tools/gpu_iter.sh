#!/bin/bash
# iteration call: GPU tests (TESTS filter), bench (BENCH_ARGS), optional A/B env runs (AB), launch list (NCU=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-it}
if [ "${TESTS}" != "none" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
  echo "tests rc=$?"; tail -4 gpurun_out/${T}_tests.log
fi
if [ "${BENCH}" != "none" ]; then
  timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS:---no-solve --no-cpu-baseline --steps 20 --warmup 5} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  echo "bench rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'factor',d['config'].get('factor_ms'),'solve',d['config'].get('solve_ms'),'e2e',d['e2e']['value'])
" ; tail -2 gpurun_out/${T}_bench.err
fi
if [ -n "$AB" ]; then
  for e in $AB; do
    env $e timeout 900 python bench.py --no-solve --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${T}_ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/${T}_ab.json').read().strip().splitlines()[-1])
print('$e','value',d['value'],'factor',d['config'].get('factor_ms'),'solve',d['config'].get('solve_ms'))"
  done
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/${T}_ncu_launch.log 2>&1
  echo "ncu rc=$?"
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
