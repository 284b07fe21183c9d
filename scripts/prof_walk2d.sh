export PYTHONPATH=$PWD
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,launch__grid_size,launch__registers_per_thread,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio
for c in 1 2; do
ncu --metrics $M --clock-control none -k regex:walk_kernel -s 0 -c 3 python scripts/walk_profile_case.py $c 1.0 2>&1 | grep -E "walk_kernel|gpu__time|smsp__|sm__|l1tex|launch__"
done
