python tools/dbg/miehe_det.py cfg1 > gpurun_out/dbg_miehe.txt 2>&1
for S in 0 2; do
  for m in full chebbd u; do PFFMG_2D_SCHED=$S python tools/kbench.py --config cfg2 --mode $m --reps 200 >> gpurun_out/sched2d_$S.txt 2>&1; done
done
for S in 0 1 2; do
  for c in "cfg4" "cfg5 --levels 7"; do
    for m in full u phi; do PFFMG_3D_SCHED=$S python tools/kbench.py --config $c --mode $m --reps 30 >> gpurun_out/sched3d_$S.txt 2>&1; done
  done
done
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for S in 0 1 2; do
PFFMG_3D_SCHED=$S ncu --metrics $M --clock-control none -k regex:"op3dt" -c 1 --csv python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 1 > gpurun_out/c5m_s$S.csv 2>/dev/null
done
for S in 0 2; do
PFFMG_2D_SCHED=$S ncu --metrics $M --clock-control none -k regex:"op2dw" -c 1 --csv python tools/kbench.py --config cfg2 --mode full --reps 1 > gpurun_out/c2m_s$S.csv 2>/dev/null
done
