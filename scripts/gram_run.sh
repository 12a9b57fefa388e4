#!/bin/bash
# Gram-kernel GPU session: tests, timing, A/B variants (GRAM_VARIANTS="name:DEF=1,DEF2=3 ..."), optional ncu (NCU=1)
python -m paper_1308_1419_b200.build > gpurun_out/build.txt 2>&1
timeout 240 python -m pytest tests/test_gpu_gram.py -x -q --timeout 200 -p no:cacheprovider > gpurun_out/gram_tests.txt 2>&1
timeout 60 python scripts/prof_driver.py edm --n 65536 --d 64 --mode gram --reps 7 --time > gpurun_out/gram_time.txt 2>&1
for vd in $GRAM_VARIANTS; do v=${vd%%:*}; defs=${vd#*:}; python -m paper_1308_1419_b200.build --variant $v ${defs//,/ } > /dev/null 2>&1; TG_LIB_PATH=paper_1308_1419_b200/libtrigrid_b200_$v.so timeout 60 python scripts/prof_driver.py edm --n 65536 --d 64 --mode gram --reps 7 --time 2>&1 | sed "s/^/$v: /" >> gpurun_out/gram_time.txt; done
[ -n "$NCU" ] && timeout 300 ncu --set full --clock-control none --import-source on -k regex:gram2 -s 1 -c 1 -o gpurun_out/prof_gram2 python scripts/prof_driver.py edm --n 65536 --d 64 --mode gram --reps 2 > gpurun_out/ncu_gram2.log 2>&1
tail -3 gpurun_out/gram_tests.txt; cat gpurun_out/gram_time.txt
