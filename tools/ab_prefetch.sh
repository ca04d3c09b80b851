set -e
L=$PWD/paper_2107_01745_b200/lib
for rep in 1 2; do
for v in pf0 pf8 main pf32 pf64; do
  if [ $v = main ]; then lib=$L/libscenopt_b200.so; else lib=$L/variants/libscenopt_b200_$v.so; fi
  for cfg in "c3 1 1" "c3 2 0" "c5b 1 1"; do set -- $cfg
    echo -n "$v rep$rep: "; SCENOPT_LIBRARY=$lib SHAPE=$1 NRHS=$2 AFF=$3 K=50 python tools/prof_sweep.py 2>&1 | cut -c1-70
  done
done
done
