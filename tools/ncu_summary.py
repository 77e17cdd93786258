"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --rep gpurun_out/prof_bench.ncu-rep \
        --launches gpurun_out/launches.csv --name vmult_cfg2_r1 --bench gpurun_out/bench.json

(name the summaries per round: bench.py reads profiles/ncu_vmult_cfg2_r<N>.json)

Writes profiles/ncu_<name>.json (the numbers bench.py reads: DRAM bytes per
launch, duration, pipe utilisation) and profiles/ncu_<name>.md.
"""
import argparse
import csv
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "lts__t_bytes.sum": "l2_bytes",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def opcode_counts(rep):
    """Warp-level executed instructions per SASS opcode of the first captured kernel."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--print-metric-instances", "details",
                          "--metrics", "sass__inst_executed_per_opcode"], capture_output=True, text=True).stdout
    flat = " ".join(out.split())
    i = flat.find("sass__inst_executed_per_opcode")
    if i < 0 or "(" not in flat[i:]:
        return {}
    body = flat[flat.index("(", i) + 1:flat.index(")", i)]
    counts = {}
    for part in body.split(";"):
        if ":" in part:
            k, v = part.split(":", 1)
            try:
                counts[k.strip()] = float(v.strip().replace(",", ""))
            except ValueError:
                pass
    return counts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--name", required=True)
    ap.add_argument("--bench")
    ap.add_argument("--note", default="")
    ap.add_argument("--src-sha", default=None,
                    help="bench.src_sha() of the sources the capture ran (default: the bench line's)")
    a = ap.parse_args()
    h, units, rows = raw(a.rep)
    kernels = []
    for r in rows:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for m, key in METRICS.items():
            if m in h:
                v = r[h.index(m)].replace(",", "")
                try:
                    d[key] = float(v)
                except ValueError:
                    d[key] = v
            if m in h and units[h.index(m)]:
                d[key + "_unit"] = units[h.index(m)]
        stalls = {}
        for k, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
                try:
                    v = float(r[k])
                except ValueError:
                    continue
                if v > 0.05:
                    stalls[name.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")] = round(v, 3)
        d["stalls_per_issue"] = stalls
        kernels.append(d)
    k0 = kernels[0]
    scale = {"Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Gbyte": 1e9}
    rb = k0["dram_read_MB"] * scale.get(k0.get("dram_read_MB_unit", "Mbyte"), 1e6)
    wb = k0["dram_write_MB"] * scale.get(k0.get("dram_write_MB_unit", "Mbyte"), 1e6)
    summary = {"name": a.name, "source": os.path.basename(a.rep), "kernels": kernels,
               "dram_bytes_per_launch": rb + wb, "note": a.note}
    ops = opcode_counts(a.rep)
    if ops:
        # FP64 flops per launch: DFMA = 2, DADD / DMUL = 1, per thread (32 per warp instruction)
        summary["fp64_flops_per_launch"] = 32.0 * (2.0 * ops.get("DFMA", 0.0) + ops.get("DADD", 0.0)
                                                   + ops.get("DMUL", 0.0))
        summary["opcodes_top"] = dict(sorted(ops.items(), key=lambda kv: -kv[1])[:16])
    if a.launches:
        lines = [l for l in open(a.launches) if not l.startswith("==")]
        lr = list(csv.reader(lines))
        hh = lr[0]
        i, j = hh.index("Kernel Name"), hh.index("Metric Value")
        agg = defaultdict(list)
        for r in lr[1:]:
            agg[r[i]].append(float(r[j].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        summary["launch_list"] = [{"kernel": k[:120], "launches": len(v), "mean_us": sum(v) / len(v) / 1e3,
                                   "share": sum(v) / tot}
                                  for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]
    if a.bench:
        summary["bench_line"] = json.load(open(a.bench))
        if a.src_sha is None:
            a.src_sha = summary["bench_line"].get("roofline", {}).get("profile", {}).get("src_sha")
    summary["src_sha"] = a.src_sha
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.name}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    md = [f"# ncu summary: {a.name}", "", a.note, "",
          f"Source capture: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none`, one launch).", ""]
    for d in kernels:
        md.append(f"## `{d['kernel']}`")
        md.append("")
        for key in METRICS.values():
            if key in d:
                md.append(f"- {key}: {d[key]} {d.get(key + '_unit', '')}")
        md.append(f"- stalls (warps per issue): {d['stalls_per_issue']}")
        md.append("")
    md.append(f"DRAM bytes per launch (read + write): {summary['dram_bytes_per_launch'] / 1e6:.2f} MB")
    if "fp64_flops_per_launch" in summary:
        md.append(f"FP64 flops per launch (SASS DFMA x2 + DADD + DMUL): "
                  f"{summary['fp64_flops_per_launch'] / 1e6:.1f} MFLOP")
        md.append(f"Top opcodes (warp instructions): {summary['opcodes_top']}")
    if "launch_list" in summary:
        md += ["", "## Launch list (ncu --metrics gpu__time_duration.sum, serialised, cold)", "",
               "| share | launches | mean us | kernel |", "|---|---|---|---|"]
        for e in summary["launch_list"]:
            md.append(f"| {e['share'] * 100:.1f}% | {e['launches']} | {e['mean_us']:.2f} | `{e['kernel'][:80]}` |")
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.name}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
