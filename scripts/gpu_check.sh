#!/bin/bash
# GPU session: -m gpu tests (PYTEST_ARGS) + quick per-mapping timings.  Outputs -> gpurun_out/
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
python -m paper_1308_1419_b200.build > gpurun_out/build.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-2400} python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q -rf --timeout 900 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
fi
for spec in ${TIME_SPECS}; do
  IFS=',' read -ra a <<< "$spec"
  timeout 300 python scripts/prof_driver.py ${a[0]} --n ${a[1]} --strategy ${a[2]} --mode ${a[3]} --time --reps 7 >> gpurun_out/times.txt 2>&1
done
ls gpurun_out > /dev/null
