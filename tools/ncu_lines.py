"""Per-source-line instruction and stall shares from an ncu report (needs -lineinfo).

  python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=30):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, h, agg = None, None, {}
    for r in csv.reader(txt.splitlines()):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 2 and r[0] == "Line No":
            h = r
            continue
        if h is None or len(r) < 8 or r[0] == "":
            continue
        agg[(cur, int(r[0]))] = (f(r[7]), f(r[4]), r[1].strip()[:90])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"instructions {ti:.3e}  stall samples {ts:.0f}")
    for k, (ie, si, src) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{100 * ie / ti:5.1f}%inst {100 * si / ts:5.1f}%stall  {k[0]}:{k[1]}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
