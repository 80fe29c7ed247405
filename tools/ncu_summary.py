"""Summarise ncu outputs into profiles/ (tracked).

  python tools/ncu_summary.py launches <launches.csv> <out.md>      # per-kernel share of one step
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [json] # key metrics per captured launch
"""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__cycles_active.avg", "sm_cycles_active"),
    ("sm__cycles_elapsed.avg", "sm_cycles_elapsed"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster_x"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]


EXCLUDE = {"init_kernel"}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = data[0]["Metric Unit"] if data else "ns"
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1.0)
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("detgpu::<unnamed>::", "").replace("unnamed>::", "")
        if name in EXCLUDE:   # engine construction (weight generation), not part of the step
            continue
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list: {path}", "", "gpu__time_duration.sum per kernel (ncu, --clock-control none, "
             "serialised and cold-cache: compare shares, not absolutes; engine weight initialisation excluded)", "",
             "| kernel | launches | total µs | share | mean µs |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0]:.2f} |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, json_out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("detgpu::<unnamed>::", "")
               .replace("unnamed>::", "")}
        for m, short in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[short] = r[i] + (f" {units[i]}" if units[i] else "")
        recs.append(rec)
    cols = ["kernel"] + [s for _, s in FULL_METRICS]
    lines = [f"# ncu --set full: {rep}", "", "| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for rec in recs:
        lines.append("| " + " | ".join(str(rec.get(c, "")) for c in cols) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if json_out:
        json.dump(recs, open(json_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
