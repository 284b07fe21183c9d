export PYTHONPATH=$PWD
for cfg in 4 5; do
  python scripts/walk_time.py $cfg 3
  BVC_HINTGRID_N=512 python scripts/walk_time.py $cfg 3
  BVC_HINTGRID_N=640 python scripts/walk_time.py $cfg 3
done
