M=gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,launch__occupancy_limit_registers,sm__ctas_launched.sum,sm__ctas_launched.max
for X in "" "--noexact"; do
tag=$([ -z "$X" ] && echo x || echo t)
for c in "cfg4" "cfg5 --levels 7"; do
ncu --metrics $M --clock-control none -k regex:"op3d[xt]_kernel" -c 1 --csv python tools/kbench.py --config $c --mode full --reps 1 $X > gpurun_out/m3d_${tag}_${c// /_}.csv 2>/dev/null
done
done
