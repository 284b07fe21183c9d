export PYTHONPATH=$PWD
for cfg in 4 5; do
  python scripts/walk_time.py $cfg 3
  for V in front2 front8 front16; do
    BVC_LIB=paper_2302_11825_b200/_build/variants/$V/libbvc_b200.so python scripts/walk_time.py $cfg 3
  done
  BVC_HINTGRID_N=512 BVC_LIB=paper_2302_11825_b200/_build/variants/front8/libbvc_b200.so python scripts/walk_time.py $cfg 3
done
