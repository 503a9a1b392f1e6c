#!/bin/bash
# ncu kernel times of one config's step for build variants in .variants/ (experiments only; restores the
# product library afterwards):  bash scripts/variant_ncu.sh <tag> <config> <kernel regex> <variant> ...
TAG=$1; C=$2; K=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
LIB=paper_2306_06528_b200/libpush_b200.so
cp $LIB /tmp/lib_product.so
for V in product "$@"; do
  if [ "$V" != product ]; then cp .variants/lib_$V.so $LIB; else cp /tmp/lib_product.so $LIB; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -s 3 -c 3 \
    python scripts/step_once.py --config $C --steps 2 > $OUT/ncu_${C}_$V.log 2>&1
  echo "== $V"; grep -E "^  [a-z_ ]|gpu__time" $OUT/ncu_${C}_$V.log | sed 's/(CUtensorMap.*//' | paste - - | awk '{print $1, $2, $NF}'
done
cp /tmp/lib_product.so $LIB
