#!/bin/bash
# ncu --set full captures of single kernels driven by scripts/prof_driver.py.
#   NCU_PROF  ';'-separated "name|kernel-regex|prof_driver args" triples
# Outputs gpurun_out/prof_<name>.{raw,details,source}.csv (ncu_summary.py input).
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -m paper_1308_1419_b200.build > gpurun_out/build.txt 2>&1
IFS=';' read -ra PROFS <<< "${NCU_PROF}"
for p in "${PROFS[@]}"; do
  name="${p%%|*}"; rest="${p#*|}"; k="${rest%%|*}"; args="${rest#*|}"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-1} -c 1 \
      -o gpurun_out/prof_$name python scripts/prof_driver.py $args > gpurun_out/ncu_full_$name.log 2>&1
  for pg in raw details; do ncu -i gpurun_out/prof_$name.ncu-rep --page $pg --csv > gpurun_out/prof_$name.$pg.csv 2>/dev/null; done
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source=sass > gpurun_out/prof_$name.source.csv 2>/dev/null
  rm -f gpurun_out/prof_$name.ncu-rep
  python scripts/prof_driver.py $args --time --reps 5 >> gpurun_out/times.txt 2>&1
done
ls -la gpurun_out
