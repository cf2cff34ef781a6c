"""Compress one plane where every element is an event and there are no
outliers (alternating 0, 1e-3 at eb 1e-5): isolates the FP64 chain."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_05630_b200 as q
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
kind = sys.argv[2] if len(sys.argv) > 2 else "alt"
if kind == "alt":
    x = np.where(np.arange(n) % 2 == 1, 1e-3, 0.0)
else:
    from oracle import planes
    x = planes.make_plane(kind, n, 99)
for _ in range(2):
    blk, st = q.compress_plane(x, q.CodecConfig(q.CodecMode.Absolute, 1e-5))
print(kind, "ratio", st.ratio, "bytes", st.output_bytes, "outliers", st.outlier_fraction)
