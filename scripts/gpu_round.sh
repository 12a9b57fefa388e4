#!/bin/bash
# One GPU session: tests, bench, A/B variants, ncu evidence.  Outputs -> gpurun_out/
#   PYTEST_ARGS   extra pytest args (default: all -m gpu tests)
#   AB_VARIANTS   space-separated env assignments, each runs a --quick bench
#   NCU_KERNELS   kernel regexes captured with ncu --set full from a --quick bench
#   NCU_PROF      ';'-separated "regex|driver args" pairs captured from scripts/prof_driver.py
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
python -m paper_1308_1419_b200.build > gpurun_out/build.txt 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${PYTEST_ARGS:-tests} -m gpu -v --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
for v in ${AB_VARIANTS}; do
  env $v timeout 300 python bench.py --quick --no-cpu --steps 20 --warmup 5 --e2e-steps 1 > "gpurun_out/bench_ab_$(echo $v | tr -c 'a-zA-Z0-9' '_' | cut -c1-60).json" 2>> gpurun_out/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --quick --no-cpu --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
for k in ${NCU_KERNELS}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py --quick --no-cpu --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_full_$k.log 2>&1
  for pg in raw details; do ncu -i gpurun_out/prof_$k.ncu-rep --page $pg --csv > gpurun_out/prof_$k.$pg.csv 2>/dev/null; done
  [ -z "$NCU_KEEP" ] && rm -f gpurun_out/prof_$k.ncu-rep
done
IFS=';' read -ra PROFS <<< "${NCU_PROF}"
for p in "${PROFS[@]}"; do
  k="${p%%|*}"; args="${p#*|}"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python scripts/prof_driver.py $args > gpurun_out/ncu_full_$k.log 2>&1
  # reports are too big to bring back (64 MiB cap): export the pages ncu_summary.py reads
  for pg in raw details; do ncu -i gpurun_out/prof_$k.ncu-rep --page $pg --csv > gpurun_out/prof_$k.$pg.csv 2>/dev/null; done
  ncu -i gpurun_out/prof_$k.ncu-rep --page source --csv --print-source=sass > gpurun_out/prof_$k.source.csv 2>/dev/null
  [ -z "$NCU_KEEP" ] && rm -f gpurun_out/prof_$k.ncu-rep
done
ls -la gpurun_out
