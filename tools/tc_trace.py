"""Summarise gpurun_out/tc_trace.bin (JTFS_TC_TRACE build): per-tile event clocks of CTA (0,0)."""
import numpy as np
t = np.fromfile("gpurun_out/tc_trace.bin", dtype=np.int64).reshape(16, 512)
names = ["g1_start", "g1_issued", "g2_wait", "g2_a2full", "g2_issued", "ep_tfull", "ep_math", "ep_a2empty", "ep_arrive",
         "g2_c0_full", "g2_c0_commit", "g2_clast_full", "g2_clast_commit", "g1_tempty", "g1_c0_full", "x"]
n = int((t[4] > 0).sum())
t0 = t[0, 0]
print("tiles", n)
for g in list(range(0, 8)) + list(range(n // 2, n // 2 + 4)):
    print(g, " ".join(f"{names[e]}={t[e, g] - t0:8d}" for e in range(15)))
d = np.diff(t[4, :n])
print("period (g2_issued diff) median", np.median(d), "mean", d.mean())
for e in range(15):
    print(names[e], "minus g2_issued(g-1):", np.median(t[e, 1:n] - t[4, 0:n - 1]))
