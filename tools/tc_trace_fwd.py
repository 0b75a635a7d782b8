"""Summarise gpurun_out/tc_trace_fwd.bin (JTFS_TC_TRACE build): per-tile event clocks of the forward
tensor-core kernel, CTA (0, 0) of the block whose K = JTFS_TRACE_K."""
import numpy as np
t = np.fromfile("gpurun_out/tc_trace_fwd.bin", dtype=np.int64).reshape(16, 512)
names = {0: "mma_tempty", 1: "mma_full0", 2: "mma_issued", 5: "ep_tfull", 6: "ep_done"}
n = int((t[2] > 0).sum())
t0 = t[0, 0]
print("tiles", n)
for g in list(range(0, 4)) + list(range(n // 2, n // 2 + 4)):
    print(g, " ".join(f"{names[e]}={t[e, g] - t0:8d}" for e in names))
d = np.diff(t[2, :n])
print("period (issued diff) median", np.median(d), "mean", d.mean())
for e in names:
    print(names[e], "minus mma_issued(g-1):", np.median(t[e, 1:n] - t[2, 0:n - 1]))
