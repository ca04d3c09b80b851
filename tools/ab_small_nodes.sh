L=$PWD/paper_2107_01745_b200/lib
for v in p6t4 p6t4s2 p6t4q24; do for kb in 16 20 24 32; do for sh in c5b c5a; do
 echo -n "$v kb=$kb: "; SCENOPT_LIBRARY=$L/variants/libscenopt_b200_$v.so SCENOPT_ITEM_KB=$kb SHAPE=$sh NRHS=1 AFF=1 K=20 timeout 300 python tools/prof_sweep.py 2>&1 | tail -1 | cut -c1-200
done; done; done
