#!/bin/bash
# compute-sanitizer memcheck + racecheck (+ synccheck for the smem-staged kernels)
# on small invocations of every product kernel -> gpurun_out/sanitize_*.txt
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CS=compute-sanitizer
run() {  # name tool args...
  local name=$1 tool=$2; shift 2
  timeout 600 $CS --tool $tool --error-exitcode 99 --print-limit 20 python scripts/prof_driver.py "$@" --reps 1 \
      > gpurun_out/sanitize_${tool}_${name}.txt 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${name}.txt | tail -1)" >> gpurun_out/sanitize_summary.txt
}
for tool in memcheck racecheck; do
  run edm_ltm $tool edm --n 3000 --d 3 --strategy ltm-r --mode span
  run edm_rb $tool edm --n 3001 --d 3 --strategy rb --mode span
  run edm_utm $tool edm --n 2999 --d 2 --strategy utm --mode span
  run edm_rec $tool edm --n 3072 --d 4 --strategy rec --mode span
  run edm_bb_grid $tool edm --n 1000 --d 3 --strategy bb --mode grid
  run write_ltm $tool write --n 3000 --strategy ltm-r --mode span
  run write_utm $tool write --n 3000 --strategy utm --mode span
  run collide $tool collide --n 3000 --strategy ltm-r
  run collide_bb $tool collide --n 2047 --strategy bb
  run write_rb $tool write --n 2999 --strategy rb --mode span
  run write_bb $tool write --n 3001 --strategy bb --mode span
  run edm_d64_direct $tool edm --n 1500 --d 64 --strategy ltm-r --mode span
  run edm_d64_gram $tool edm --n 1500 --d 64 --strategy ltm-r --mode gram
  run edm_d200_gram $tool edm --n 700 --d 200 --strategy ltm-r --mode gram
done
run edm_d64_gram synccheck edm --n 1500 --d 64 --strategy ltm-r --mode gram
run edm_d64_direct synccheck edm --n 1500 --d 64 --strategy ltm-r --mode span
run collide synccheck collide --n 3000 --strategy ltm-r
cat gpurun_out/sanitize_summary.txt
