# A/B of library variants on sweeps and C3 solves: bash tools/ab_solve.sh main nopdl ...
L=$PWD/paper_2107_01745_b200/lib
VARIANTS="$*"
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = main ]; then lib=$L/libscenopt_b200.so; else lib=$L/variants/libscenopt_b200_$v.so; fi
  for cfg in "c3 1 1" "c3 2 0"; do set -- $cfg
    echo -n "$v rep$rep: "; SCENOPT_LIBRARY=$lib SHAPE=$1 NRHS=$2 AFF=$3 K=50 python tools/prof_sweep.py 2>&1 | cut -c1-70
  done
  echo -n "$v rep$rep: "; SCENOPT_LIBRARY=$lib python tools/solve_times.py 2>&1 | tail -1
done
done
