for v in 1099511627776 200000 ; do
  for c in cfg2 cfg3; do echo "== BD_MAXV2=$v $c"; PFFMG_BD_MAXV2=$v python tools/prof_vcycle.py $c 2>/dev/null | head -1; done
done
for v in 131072 1000000 1099511627776 8192; do
  for c in cfg4; do echo "== BD_MAXV3=$v $c"; PFFMG_BD_MAXV3=$v python tools/prof_vcycle.py $c 2>/dev/null | head -1; done
done
for m in chebu chebp chebbd; do python tools/kbench.py --config cfg2 --mode $m --pre --reps 100; python tools/kbench.py --config cfg3 --mode $m --pre --reps 100; done
