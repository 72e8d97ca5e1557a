"""Summarise ncu captures from tools/profile_round.sh into profiles/.

    python tools/summarize_profiles.py r01

Writes profiles/<tag>_launches.csv (per-kernel launch list: name, count,
mean/min/max duration, DRAM bytes), profiles/<tag>_kernels.md (the --set full
headline metrics of each captured kernel) and profiles/<tag>_traffic.json
(dram read+write bytes per launch of each kernel, consumed by bench.py's
roofline.traffic).
"""

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
]


def _num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def launches(tag):
    path = OUT / f"{tag}_launches.csv"
    if not path.exists():
        return
    rows = list(csv.reader(path.open()))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = defaultdict(lambda: defaultdict(list))
    idi = hdr.index("ID")
    for r in rows[start + 1:]:
        per[r[ki].split("(")[0]][r[mi]].append((int(r[idi]), _num(r[vi])))
    with (PROF / f"{tag}_launches.csv").open("w") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "mean_us", "min_us", "max_us", "dram_read_B_mean", "dram_write_B_mean"])
        for k, m in sorted(per.items(), key=lambda kv: -sum(v for _, v in kv[1]["gpu__time_duration.sum"])):
            d = [v / 1e3 for _, v in m["gpu__time_duration.sum"]]
            rd = [v for _, v in m.get("dram__bytes_read.sum", [])]
            wr = [v for _, v in m.get("dram__bytes_write.sum", [])]
            w.writerow([k, len(d), f"{sum(d) / len(d):.2f}", f"{min(d):.2f}", f"{max(d):.2f}",
                        f"{sum(rd) / max(len(rd), 1):.0f}", f"{sum(wr) / max(len(wr), 1):.0f}"])


def kernels(tag):
    lines = [f"# {tag}: ncu --set full captures (cold caches, --clock-control none)\n"]
    traffic = {}
    for rep in sorted(OUT.glob(f"{tag}_*.ncu-rep")):
        res = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
        rows = list(csv.reader(res.stdout.splitlines()))
        if len(rows) < 3:
            continue
        h, v = rows[0], rows[2]
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep.stem
        lines.append(f"\n## {rep.stem}\n\n`{name[:160]}`\n\n| metric | value |\n|---|---|")
        vals = {}
        for m in METRICS:
            if m in h:
                vals[m] = v[h.index(m)]
                lines.append(f"| {m} | {vals[m]} |")
        rd, wr = _num(vals.get("dram__bytes_read.sum")), _num(vals.get("dram__bytes_write.sum"))
        if rd is not None and wr is not None:
            unit_r = rows[1][h.index("dram__bytes_read.sum")]
            unit_w = rows[1][h.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic[rep.stem] = rd * scale.get(unit_r, 1) + wr * scale.get(unit_w, 1)
    (PROF / f"{tag}_kernels.md").write_text("\n".join(lines) + "\n")
    (PROF / f"{tag}_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    launches(tag)
    kernels(tag)
    print("written", sorted(p.name for p in PROF.glob(f"{tag}_*")))
