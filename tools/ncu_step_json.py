"""From an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum) of
`bench.py --steps 1`, write the DRAM bytes of the last step: profiles/dram_step_<config>.json (whole step)
and profiles/traffic_<config>.json (joint-stage groups: k_joint_fwd_* / k_joint_bwd_* + k_gy_reduce).
bench.py reads both (hbm.dram_bytes_per_step_ncu, roofline.traffic).
usage: python tools/ncu_step_json.py launches.csv launches_per_step config batch"""
import collections
import csv
import json
import os
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def main(path, per_step, config, batch):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    iid, ik, im, iu, iv = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    L = collections.OrderedDict()
    for r in rows:
        d = L.setdefault(int(r[iid]), {"k": r[ik]})
        d[r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    ids = sorted(L)[-per_step:]
    tot = sum(L[i]["dram__bytes_read.sum"] + L[i]["dram__bytes_write.sum"] for i in ids)
    grp = {"joint_fwd": 0.0, "joint_bwd": 0.0}
    for i in ids:
        k = L[i]["k"]
        b = L[i]["dram__bytes_read.sum"] + L[i]["dram__bytes_write.sum"]
        if "k_joint_fwd" in k:
            grp["joint_fwd"] += b
        elif "k_joint_bwd" in k or "k_gy_reduce" in k:
            grp["joint_bwd"] += b
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = os.path.relpath(path, root)
    json.dump({"dram_bytes_per_step": tot, "batch": batch, "launches": per_step, "source": src},
              open(os.path.join(root, "profiles", f"dram_step_{config}.json"), "w"), indent=1)
    json.dump({k: {"dram_bytes_per_step": v} for k, v in grp.items()} | {"batch": batch, "source": src},
              open(os.path.join(root, "profiles", f"traffic_{config}.json"), "w"), indent=1)
    print(config, tot / 1e9, "GB/step;", {k: v / 1e9 for k, v in grp.items()})


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]))
