# A/B of the 2D entry frontiers: cache-generation time of C1 and C3 with one entry node per cell
# (BVC_FRONT=0), with frontiers (default) and with finer grids
export PYTHONPATH=$PWD
for cfg in 1 3; do
  BVC_FRONT=0 python scripts/walk_time.py $cfg 5
  python scripts/walk_time.py $cfg 5
  BVC_HINTGRID_N=2048 python scripts/walk_time.py $cfg 5
  BVC_HINTGRID_N=4096 python scripts/walk_time.py $cfg 5
  BVC_FRONT=0 BVC_HINTGRID_N=4096 python scripts/walk_time.py $cfg 5
done
