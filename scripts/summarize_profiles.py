"""Condense the ncu CSV logs of scripts/profile_round.sh into profiles/ (dev tool).

  python scripts/summarize_profiles.py <tag>     # reads gpurun_out/prof_*.csv
"""
import csv
import io
import sys
from collections import defaultdict

tag = sys.argv[1]
wl = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].endswith(".ncu-rep") else "cfg3"
src = "gpurun_out/"


def table(path):
    """Rows of an ncu --csv log (skips ==PROF==/==WARNING== lines); [] if absent."""
    try:
        lines = [ln for ln in open(path) if ln.startswith('"')]
    except FileNotFoundError:
        return []
    return list(csv.reader(io.StringIO("".join(lines))))


# launch list: one row per (launch, metric) in --page details csv, or raw
rows = table(src + "prof_launches.csv")
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(lambda: [0, 0.0])
raw = []
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    unit = r[mi + 1] if len(r) > mi + 1 else ""
    v = float(r[vi].replace(",", ""))
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
    name = r[ki].split("(")[0].replace("void ", "")
    per[name][0] += 1
    per[name][1] += ms
    raw.append((name, ms))
tot = sum(v[1] for v in per.values())
with open(f"profiles/{tag}_launches_summary.csv", "w") as f:
    f.write(f"# {tag} launch list: `python bench.py --workload {wl} --steps 1 --warmup 1 --no-cpu-baseline` under\n")
    f.write("# `ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares)\n")
    f.write("kernel,launches,total_ms,share\n")
    for name, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{name},{n},{ms:.3f},{ms / tot:.4f}\n")
with open(f"profiles/{tag}_launches_raw.csv", "w") as f:
    f.write("kernel,ms\n")
    for name, ms in raw:
        f.write(f"{name},{ms:.4f}\n")

keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
for name in ("sweep", "ilu", "matvec"):
    rows = table(src + f"prof_{name}_full.csv")
    if not rows:
        continue
    hdr = rows[0]
    cols = ["Kernel Name"] + [k for k in keep if k in hdr]
    idx = [hdr.index(c) for c in cols]
    with open(f"profiles/{tag}_{wl}_{name}_full.csv", "w") as f:
        f.write(f"# ncu --set full --clock-control none --page raw, launches of the {name} kernel inside "
                f"python bench.py --workload {wl} --steps 1 --warmup 1\n")
        w = csv.writer(f)
        w.writerow(cols)
        w.writerow([rows[1][i] for i in idx])   # units row
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
print(open(f"profiles/{tag}_launches_summary.csv").read())
for name in ("sweep", "ilu", "matvec"):
    try:
        print(open(f"profiles/{tag}_{wl}_{name}_full.csv").read())
    except FileNotFoundError:
        pass


def summarize_rep(rep, out, note):
    """Selected raw metrics of an `ncu -o` report into profiles/<out> (per launch)."""
    import subprocess
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return
    hdr = rows[0]
    cols = ["Kernel Name"] + [k for k in keep if k in hdr]
    idx = [hdr.index(c) for c in cols]
    with open(f"profiles/{out}", "w") as f:
        f.write(f"# {note}\n")
        w = csv.writer(f)
        w.writerow(cols)
        for r in rows[1:]:
            w.writerow([r[i] for i in idx])
    print(open(f"profiles/{out}").read())


if len(sys.argv) > 3:
    # extra captures: <rep> <out.csv> <note>, repeated
    extra = sys.argv[3:]
    for k in range(0, len(extra) - 2, 3):
        summarize_rep(extra[k], extra[k + 1], extra[k + 2])
