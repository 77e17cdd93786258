# A/B of kernel variants by ncu gpu__time_duration (the event timer ticks in ~2 us steps)
# usage: bash tools/var/ncu_ab.sh KREGEX "kbench args" ...
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
K=$1; shift
for v in tools/var/lib_*.so; do
  cp $v $LIB
  for args in "$@"; do
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv python tools/kbench.py $args --reps 12 2>/dev/null \
      | python -c "
import sys,csv
r=[x for x in csv.reader(sys.stdin) if len(x)>10 and x[-3]=='gpu__time_duration.sum']
d=[float(x[-1].replace(',','')) for x in r][3:]
print('$(basename $v)', '$args', 'n=%d mean %.2f us min %.2f'%(len(d), sum(d)/len(d)/1e3, min(d)/1e3) if d else 'none')"
  done
done
cp /tmp/lib_orig.so $LIB
