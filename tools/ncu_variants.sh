# Warm-L2 ncu metrics of the iteration kernels for each operator variant
# (matrix_free = $MF list); CSVs in gpurun_out/m_<mf>.csv.
M="gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,launch__grid_size,launch__registers_per_thread,sm__cycles_elapsed.avg"
for mf in ${MF:-3 2 0}; do
PDLP_OPTS="{\"matrix_free\": $mf}" timeout 300 ncu --cache-control none --clock-control none --metrics $M -k regex:"seg_kernel|te_kernel|col_pipe|row_step" --launch-skip 40 -c 6 --csv python tools/profile_c1.py 200 > gpurun_out/m_$mf.csv 2>gpurun_out/m_$mf.err
done
