"""Per-source-line share of warp-stall samples and executed instructions
from an ncu report (source page, cuda+sass view).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [min_share]
"""
import collections
import csv
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    agg = collections.OrderedDict()
    cur = fname = hdr = None
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 9:
            continue
        if r[0] != "":
            cur = (fname, int(r[0]), r[1][:72])
            agg.setdefault(cur, [0.0, 0.0, 0.0])
            continue
        a = agg[cur]
        a[0] += num(r[4])
        a[1] += num(r[7])
        a[2] += num(r[8])
    tot = sum(a[0] for a in agg.values()) or 1
    tot_e = sum(a[1] for a in agg.values()) or 1
    print(f"samples {tot:.0f}  warp instructions {tot_e:.0f}")
    for k, a in agg.items():
        if a[0] > thr * tot or a[1] > thr * tot_e:
            print(f"{k[0][:14]:14s}{k[1]:5d} {a[0] / tot * 100:5.1f}% smp {a[1] / tot_e * 100:5.1f}% "
                  f"inst  lanes {a[2] / max(a[1], 1):4.1f}  {k[2]}")


if __name__ == "__main__":
    main()
