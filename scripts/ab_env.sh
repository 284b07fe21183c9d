# A/B of a runtime knob on the 3D walks: bash scripts/ab_env.sh VAR=VALUE  (C4 and C5 walk time)
export PYTHONPATH=$PWD
for cfg in 4 5; do
  env $1 python scripts/walk_time.py $cfg 3
  python scripts/walk_time.py $cfg 3
done
