#!/bin/bash
# Build-time A/B on the GPU box: VARIANTS="name:DEF=1,DEF2=3 ..." each built as
# libtrigrid_b200_<name>.so and run with CMD (default: quick bench) via TG_LIB_PATH.
# The baseline (in-tree defaults) runs first.  Results -> gpurun_out/ab.txt
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CMD=${CMD:-"python bench.py --quick --no-cpu --steps 10 --warmup 3 --e2e-steps 1"}
python -m paper_1308_1419_b200.build > gpurun_out/build.txt 2>&1
echo "== base" >> gpurun_out/ab.txt
timeout ${AB_TIMEOUT:-180} $CMD >> gpurun_out/ab.txt 2>&1
for vd in $VARIANTS; do
  v=${vd%%:*}; defs=${vd#*:}
  python -m paper_1308_1419_b200.build --variant $v ${defs//,/ } > /dev/null 2>&1
  echo "== $v ($defs)" >> gpurun_out/ab.txt
  TG_LIB_PATH=paper_1308_1419_b200/libtrigrid_b200_$v.so timeout ${AB_TIMEOUT:-180} $CMD >> gpurun_out/ab.txt 2>&1
done
