"""DRAM traffic of the joint-stage kernel groups per step, from an ncu --set full capture of every
joint launch of a bench run (tools/gpu_session.sh 'traffic'):

  python tools/ncu_traffic.py <report.ncu-rep> <config> <n_forward_passes> <n_backward_passes> <out.json>

Forward group = k_joint_fwd_* launches; backward group = k_joint_bwd_* + k_gy_reduce. The bench run
does one target forward plus (warmup + steps) loss_grad calls, each with one forward and one backward.
"""
import csv
import json
import subprocess
import sys


def main(rep, config, nf, nb, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    ki, rd, wr, du = (h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                      h.index("gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
              "ms": 1e-3, "s": 1.0}
    g = {"joint_fwd": [0.0, 0.0, 0], "joint_bwd": [0.0, 0.0, 0]}
    for r in rows[2:]:
        name = r[ki]
        key = "joint_fwd" if "k_joint_fwd" in name else ("joint_bwd" if ("k_joint_bwd" in name or "k_gy_reduce" in name)
                                                         else None)
        if key is None:
            continue
        num = lambda x: float(x.replace(",", ""))
        b = num(r[rd]) * scale.get(units[rd], 1.0) + num(r[wr]) * scale.get(units[wr], 1.0)
        g[key][0] += b
        g[key][1] += num(r[du]) * tscale.get(units[du], 1e-9)
        g[key][2] += 1
    res = {"config": config, "source": rep, "method": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum"}
    for k, n in (("joint_fwd", nf), ("joint_bwd", nb)):
        res[k] = {"dram_bytes_per_step": g[k][0] / n, "launches_per_step": g[k][2] / n,
                  "ncu_serial_ms_per_step": 1e3 * g[k][1] / n}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4]), sys.argv[5])
