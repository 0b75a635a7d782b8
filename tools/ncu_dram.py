"""Per-kernel time, DRAM bytes and achieved bandwidth over the last step of an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (cold-cache, serialised).
usage: python tools/ncu_dram.py launches.csv [launches_per_step]"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, per_step):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    iid, ik, im, iu, iv = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    L = collections.OrderedDict()
    for r in rows:
        d = L.setdefault(int(r[iid]), {"k": r[ik]})
        d[r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    ids = sorted(L)[-per_step:]
    agg = collections.OrderedDict()
    for i in ids:
        d = L[i]
        a = agg.setdefault(d["k"].split("(")[0][:48], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"]
        a[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    tot = sum(a[1] for a in agg.values())
    print(f"# last {per_step} launches of {path}: {tot / 1e3:.3f} ms (cold-cache, serialised)")
    print(f"# {'kernel':48s} {'n':>4s} {'ms':>8s} {'share':>6s} {'GB':>7s} {'GB/s':>7s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:50s} {a[0]:4d} {a[1] / 1e3:8.3f} {a[1] / tot:6.1%} {a[2] / 1e9:7.3f} {a[2] / a[1] / 1e3:7.0f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 126)
