"""Summarise a dense warp-sampling ncu capture of K5 (SourceCounters):
stall reasons of the single-thread code (accept, dependent walks) and the
executed instruction footprint.

    ncu --section WarpStateStats --section SourceCounters --import-source on \\
        --warp-sampling-interval 0 --warp-sampling-max-passes 50 \\
        -k regex:fill_kernel -s 10 -c 1 -o gpurun_out/k5_now \\
        python tools/step_driver.py --mode k5 --steps 16
    python tools/stall_summary.py gpurun_out/k5_now.ncu-rep > profiles/r01_k5_stalls.md
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, data = rows[1], rows[2:]
    ia, iex, ith = h.index("Address"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]

    def agg(sel):
        c = collections.Counter()
        for r in sel:
            for x in reasons:
                c[x] += int(r[h.index(x)] or 0)
        return c

    single = [r for r in data if int(r[iex] or 0) > 0 and int(r[ith]) == int(r[iex])]
    print(f"# K5 warp-state sampling ({rep.split('/')[-1]})\n")
    print("| code | samples | top stall reasons |\n|---|---|---|")
    for name, sel in [("all warps", data), ("single-thread (accept, dependent walks, setup)", single),
                      ("single-thread, once per CTA (accept)", [r for r in single if int(r[iex]) <= 140])]:
        c = agg(sel)
        tot = sum(c.values())
        top = ", ".join(f"{k[6:]} {v / tot:.0%}" for k, v in c.most_common(4))
        print(f"| {name} | {tot} | {top} |")
    lines = collections.defaultdict(int)
    base = int(data[0][ia], 16)
    for r in data:
        e = int(r[iex] or 0)
        if e:
            k = (int(r[ia], 16) - base) // 128
            lines[k] = max(lines[k], e)
    print("\nExecuted instruction footprint (128-B lines touched in this launch):\n")
    print("| executed by ≥ N warps-instances | KB |\n|---|---|")
    for thr in (1, 100, 128, 1000):
        print(f"| {thr} | {sum(1 for v in lines.values() if v >= thr) * 128 / 1024:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
