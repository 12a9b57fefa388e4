#!/bin/bash
# A/B of the span UTM super-block width (TG_UTM_RUNS = run widths per super-block) -> gpurun_out/utm_ab.txt
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for r in ${UTM_RUNS:-1 4 16 64}; do
  for k in edm write; do
    echo "runs=$r $(TG_UTM_RUNS=$r timeout 120 python scripts/prof_driver.py $k --n 65536 --strategy utm --mode span --time --reps 7 | head -1)" >> gpurun_out/utm_ab.txt
  done
done
