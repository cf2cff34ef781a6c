"""Debug: codebook phase times per plane from a QCSIM_CB_TRACE_FILE dump
(stamps 0..8, slot 15 = alphabet size)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16).astype(np.int64)
n = t[:, 15].copy()
st = t[:, :9]
t0 = st[:, 0].min()
rel = (st - t0) / 1e3
names = ["start", "alphabet", "compact", "sort", "merge+depth", "lengths", "codes", "publish", "dec tables"]
print("planes", len(t), "alphabet min/median/max", n.min(), int(np.median(n)), n.max())
print("kernel span us %.1f" % rel.max())
d = np.diff(rel, axis=1)
for i in range(8):
    print("  %-12s mean %6.2f  max %6.2f us" % (names[i + 1], d[:, i].mean(), d[:, i].max()))
k = np.argmax(rel[:, 8])
print("slowest plane", k, "n", n[k], " ".join("%.1f" % v for v in rel[k]))
m = t[:, 11] > 0
if m.any():
    print("merge loop only (stamp 10->11): mean %.2f us" % ((t[m, 11] - t[m, 10]) / 1e3).mean())
