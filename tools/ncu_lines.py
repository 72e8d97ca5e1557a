"""Per-source-line warp-stall attribution from an ncu report (cuda,sass view).

    python tools/ncu_lines.py gpurun_out/k4_prof.ncu-rep [top_n]

Prints, per file:line, all warp-state samples and the no_instructions /
long_scoreboard shares (columns from the SASS rows under each line)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = defaultdict(lambda: [0, 0, 0, 0])
    fname, hdr, line, src = "?", None, None, ""
    tot = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            i_all = hdr.index("Warp Stall Sampling (All Samples)")
            i_ex = hdr.index("Instructions Executed")
            cols = {c: k for k, c in enumerate(hdr)}
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if not r[0]:
            continue  # SASS rows: the line row above already aggregates them

        def num(x):
            try:
                return int(float(x))
            except ValueError:
                return 0
        v = num(r[i_all])
        tot += v
        a = agg[(fname, r[0])]
        a[0] += v
        a[1] += num(r[i_ex])
        a[3] = r[1]
    print("total samples", tot)
    for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{a[0]:6d} {100.0 * a[0] / max(tot, 1):5.1f}%  {f}:{ln:5s} inst {a[1]:7d}  {str(a[3]).strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
