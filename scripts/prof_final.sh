# final-state ncu captures of the 3D walk kernels (C4 at 1/4, C5 at 1/8 of the samples) and C3's walk launches
export PYTHONPATH=$PWD
bash scripts/prof_walk3.sh
python scripts/walk_profile_case.py 3 0.25 > gpurun_out/wp3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 0 -c 6 -o gpurun_out/src_walk_c3 -f python scripts/walk_profile_case.py 3 0.25 > gpurun_out/ncu_src_c3.log 2>&1
ls -la gpurun_out
