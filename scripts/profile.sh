#!/bin/bash
# one profiling pass on the GPU box (B200_PROFILING.md recipe); outputs in gpurun_out/
#   bash scripts/profile.sh [config] [tag]   (default: config 2, files prof_{walk,gather}[_tag])
export PYTHONPATH=$PWD
CFG=${1:-2}
TAG=${2:+_$2}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --no-probe --no-extra"
$CMD > gpurun_out/plain$TAG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches$TAG.csv $CMD > gpurun_out/ncu_list$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 2 -c 1 -o gpurun_out/prof_gather$TAG -f $CMD > gpurun_out/ncu_gather$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:walk -s 0 -c 1 -o gpurun_out/prof_walk$TAG -f $CMD > gpurun_out/ncu_walk$TAG.log 2>&1
ls -la gpurun_out/
