for X in "" "--noexact"; do
  tag=$([ -z "$X" ] && echo x || echo t)
  ncu --set full --import-source on --clock-control none -k regex:"op3d[xt]_kernel" -c 1 -o /tmp/p3d_$tag \
    python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 1 $X > gpurun_out/p3d_$tag.log 2>&1
  ncu -i /tmp/p3d_$tag.ncu-rep --page raw --csv > gpurun_out/p3d_${tag}_raw.csv
  ncu -i /tmp/p3d_$tag.ncu-rep --page source --csv --print-source cuda > gpurun_out/p3d_${tag}_cuda.csv 2>gpurun_out/p3d_${tag}_cuda.err
  ncu -i /tmp/p3d_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/p3d_${tag}_sass.csv 2>/dev/null
done
ls -la gpurun_out/
