#!/bin/bash
# span write/EDM at small N vs TG_SPAN_MIN_UNITS (launch-time unit shrink) -> gpurun_out/smalln_ab.txt
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for mu in ${MIN_UNITS:-1 1184 2368 4736 9472 18944}; do
  for n in 4096 16384; do
    for s in ltm-r bb; do
      echo "min_units=$mu $(TG_SPAN_MIN_UNITS=$mu timeout 120 python scripts/prof_driver.py write --n $n --strategy $s --mode span --time --reps 31 | head -1)" >> gpurun_out/smalln_ab.txt
    done
  done
done
