# ncu launch list of the bench's Newton-step solve (cfg2): every kernel of the
# setup graph, the V-cycle graphs and GMRES, per-launch durations (cold, serialised)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv \
  python tools/prof_newton.py cfg2 > gpurun_out/solve_launches.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/solve_launches.csv")) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4][:70]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values())
print("launches", len(rows), "total us", round(tot, 1))
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{100 * t / tot:5.1f}%  {n:6d}  {t / n:8.2f} us  {k}")
PY
