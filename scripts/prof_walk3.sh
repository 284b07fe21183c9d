export PYTHONPATH=$PWD
python scripts/walk_profile_case.py 4 0.25 > gpurun_out/wp4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:walk3_kernel -s 0 -c 1 -o gpurun_out/src_walk_c4 -f python scripts/walk_profile_case.py 4 0.25 > gpurun_out/ncu_src_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:walk3_kernel -s 0 -c 1 -o gpurun_out/src_walk_c5 -f python scripts/walk_profile_case.py 5 0.125 > gpurun_out/ncu_src_c5.log 2>&1
ls -la gpurun_out
