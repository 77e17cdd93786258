# ncu --set full capture of the block-diagonal Chebyshev step (the V-cycle's dominant kernel) at cfg2 and cfg4's u-block step
SHA=$(python -c "import bench; print(bench.src_sha())")
timeout 600 ncu --set full --import-source on --clock-control none -k regex:op2dw_kernel --launch-skip 3 -c 1 -o /tmp/cap_chebbd \
  python tools/kbench.py --config cfg2 --mode chebbd --pre --reps 4 > gpurun_out/cap_chebbd.log 2>&1
python tools/ncu_summary.py --rep /tmp/cap_chebbd.ncu-rep --name chebbd_cfg2_r2 --src-sha $SHA \
  --note "block-diagonal Chebyshev step (pffmg_cheb_step_bd, pre-masked input, a_phiphi table): tools/kbench.py --config cfg2 --mode chebbd --pre" >> gpurun_out/cap_summary2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:op3dt_kernel --launch-skip 3 -c 1 -o /tmp/cap_chebu \
  python tools/kbench.py --config cfg4 --mode chebu --pre --reps 4 > gpurun_out/cap_chebu.log 2>&1
python tools/ncu_summary.py --rep /tmp/cap_chebu.ncu-rep --name chebu_cfg4_r2 --src-sha $SHA \
  --note "u-block Chebyshev step (pffmg_cheb_step_dc, pre-masked input): tools/kbench.py --config cfg4 --mode chebu --pre" >> gpurun_out/cap_summary2.log 2>&1
cp profiles/ncu_chebbd_cfg2_r2.* profiles/ncu_chebu_cfg4_r2.* gpurun_out/ 2>/dev/null
tail -5 gpurun_out/cap_summary2.log
