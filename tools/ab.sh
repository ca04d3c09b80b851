#!/bin/bash
# A/B of sweep variants on one box: tools/ab.sh tag1 tag2 ... (lib/variants/libscenopt_b200_<tag>.so; "main" = lib/)
for rep in 1 2; do
  for t in "$@"; do
    if [ "$t" = main ]; then lib=$PWD/paper_2107_01745_b200/lib/libscenopt_b200.so; else lib=$PWD/paper_2107_01745_b200/lib/variants/libscenopt_b200_$t.so; fi
    echo "== $t"; SCENOPT_LIBRARY=$lib SHAPE=${SHAPE:-c3} timeout 200 python tools/sweep_perf.py 2>&1 | grep "aff" | cut -c1-60
  done
done
