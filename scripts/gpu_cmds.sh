#!/bin/bash
# GPU session: optional -m gpu tests (PYTEST_ARGS, skipped when empty) then
# each ';'-separated command of CMDS, output appended to gpurun_out/cmds.txt.
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
if [ -n "$PYTEST_ARGS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest $PYTEST_ARGS -m gpu -q -rf --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
fi
IFS=';' read -ra CS <<< "${CMDS}"
for c in "${CS[@]}"; do
  echo "### $c" >> gpurun_out/cmds.txt
  timeout ${CMD_TIMEOUT:-300} bash -c "$c" >> gpurun_out/cmds.txt 2>&1
  echo "### rc=$?" >> gpurun_out/cmds.txt
done
true
