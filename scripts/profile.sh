#!/bin/bash
# one profiling pass on the GPU box (B200_PROFILING.md recipe); outputs in gpurun_out/
export PYTHONPATH=$PWD
CMD="python bench.py --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 2 -c 1 -o gpurun_out/prof_gather -f $CMD > gpurun_out/ncu_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/prof_walk -f $CMD > gpurun_out/ncu_walk.log 2>&1
ls -la gpurun_out/
