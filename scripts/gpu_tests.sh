#!/bin/bash
# GPU session: selected -m gpu tests (PYTEST_ARGS) then an optional bench (BENCH_ARGS).  Outputs -> gpurun_out/
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${PYTEST_ARGS:-tests} -m gpu -v -x --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
if [ -n "$BENCH_ARGS" ]; then
  timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
true
