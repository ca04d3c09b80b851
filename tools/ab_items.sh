# item-size A/B on small-state trees (layout knobs, no rebuild)
for cfg in "24 32" "32 48" "40 64" "48 64" "64 96"; do set -- $cfg
  for sh in c5b c5a; do
    echo -n "ITEM_KB=$1 MAX_NODES=$2: "; SCENOPT_ITEM_KB=$1 SCENOPT_ITEM_MAX_NODES=$2 SHAPE=$sh NRHS=1 AFF=1 K=30 python tools/prof_sweep.py 2>&1 | cut -c1-200
  done
done
