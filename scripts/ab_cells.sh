# walk time of C1, C3, C4, C5 and the walk kernels' DRAM bytes (C4 1/4, C5 1/8 of the samples)
export PYTHONPATH=$PWD
for cfg in 1 3 4 5; do python scripts/walk_time.py $cfg 3; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__thread_inst_executed_per_inst_executed.ratio
for case in "4 0.25" "5 0.125"; do
  set -- $case
  ncu --metrics $M --clock-control none -k regex:walk3_ -s 0 -c 1 python scripts/walk_profile_case.py $1 $2 2>&1 | grep -E "walk3_kernel|dram__|gpu__time|lts__|l1tex__|smsp__"
done
