"""Tensor-pipe utilisation of the joint-stage launches of one step, from an ncu launch list taken with
--metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,
sm__pipe_tensor_subpipe_hmma_cycles_active...,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,
sm__mem_tensor_cycles_active...,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_joint.
usage: python tools/ncu_tensor.py tensor.csv launches_per_step > out.txt"""
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
        d = L.setdefault(int(r[iid]), {"k": r[ik].split("(")[0]})
        d[r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    ids = sorted(L)[-per_step:]
    print("# ncu --metrics sm__pipe_tensor_cycles_active, sm__pipe_tensor_subpipe_hmma_cycles_active, "
          "sm__mem_tensor_cycles_active (pct of peak sustained elapsed), sm__inst_executed_pipe_tensor_subpipe_hmma.sum, "
          f"dram bytes -k regex:k_joint, last {per_step} joint launches (cold-cache, serialised); source {path}")
    tw = tt = 0.0
    for i in ids:
        d = L[i]
        t = d["gpu__time_duration.sum"]
        pa = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        ph = d.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        pm = d.get("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        n = d.get("sm__inst_executed_pipe_tensor_subpipe_hmma.sum", 0.0)
        gb = (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / 1e9
        print(f"{d['k'][:38]:38s} {t:11.1f} us tensor {pa:5.1f}% hmma {ph:5.1f}% tmem {pm:5.1f}% UTCHMMA {n:8.3g} DRAM {gb:.3f} GB")
        tw += t * pa
        tt += t
    print(f"# time-weighted tensor-pipe active: {tw / tt:.1f}% over {tt / 1e3:.1f} ms")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
