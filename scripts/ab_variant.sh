# A/B of compile-time variants (scripts/variant_lib.py NAME ...) against the main build: C4 / C5 walk time
#   VARIANTS="a b" bash scripts/ab_variant.sh
export PYTHONPATH=$PWD
for cfg in ${CFGS:-4 5}; do
  python scripts/walk_time.py $cfg 3
  for V in $VARIANTS; do
    BVC_LIB=paper_2302_11825_b200/_build/variants/$V/libbvc_b200.so python scripts/walk_time.py $cfg 3
  done
done
