# A/B of a walk3.cu compile-time variant (BVC_LIB) against the main build: C4 / C5 walk time
export PYTHONPATH=$PWD
V=${1:-nospec}
for cfg in 4 5; do
  BVC_LIB=paper_2302_11825_b200/_build/variants/$V/libbvc_b200.so python scripts/walk_time.py $cfg 3
  python scripts/walk_time.py $cfg 3
done
