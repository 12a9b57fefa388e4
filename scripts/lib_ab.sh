#!/bin/bash
# A/B of prebuilt library variants (LIBS="base sq1 ..." -> paper_1308_1419_b200/libtrigrid_b200_<v>.so)
# running CMD (a prof_driver command line) REPS times each, interleaved -> gpurun_out/lib_ab.txt
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rep in $(seq 1 ${ROUNDS:-2}); do
  for v in ${LIBS}; do
    lib=paper_1308_1419_b200/libtrigrid_b200.so
    [ "$v" != "base" ] && lib=paper_1308_1419_b200/libtrigrid_b200_$v.so
    echo "$v $(TG_LIB_PATH=$lib timeout 180 python scripts/prof_driver.py $CMD --time --reps ${REPS:-7} | head -1)" >> gpurun_out/lib_ab.txt
  done
done
if [ -n "$TEST_LIBS" ]; then
  for v in $TEST_LIBS; do
    TG_LIB_PATH=paper_1308_1419_b200/libtrigrid_b200_$v.so timeout 900 python -m pytest ${TESTS:-tests/test_gpu_gram.py} -q -x -m gpu -p no:cacheprovider > gpurun_out/lib_ab_test_$v.txt 2>&1
    echo "test $v rc=$? $(tail -1 gpurun_out/lib_ab_test_$v.txt)" >> gpurun_out/lib_ab.txt
  done
fi
