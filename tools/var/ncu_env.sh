# ncu-duration sweep of an env var: bash tools/var/ncu_env.sh KREGEX VAR "v1 v2 .." "kbench args"
K=$1; VAR=$2; VALS=$3; shift 3
for val in $VALS; do
  for args in "$@"; do
    env $VAR=$val ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K --csv python tools/kbench.py $args --reps 12 2>/dev/null \
      | python -c "
import sys,csv
r=[x for x in csv.reader(sys.stdin) if len(x)>10 and x[-3]=='gpu__time_duration.sum']
d=[float(x[-1].replace(',',''))/1e3 for x in r][3:]
print('$VAR=$val', '$args', 'n=%d mean %.2f us min %.2f'%(len(d), sum(d)/len(d), min(d)) if d else 'none')"
  done
done
