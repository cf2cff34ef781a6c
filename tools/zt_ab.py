"""A/B of the run-aware tile paths on a random U3+CZ circuit (n qubits,
slices of 2^20): per-kernel device time of G gate passes after layer 0.
python tools/zt_ab.py [n] [gates] [skip]   (QCSIM_ZERO_TILES=0 turns the paths off)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402
from paper_1811_05630_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
G = int(sys.argv[2]) if len(sys.argv) > 2 else 6
SKIP = int(sys.argv[3]) if len(sys.argv) > 3 else 2  # untimed gates after layer 0
acts = q.random_u3_circuit_actions(n, 20, seed=30)
setup = n + n // 2
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=20, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
eng.load_basis(0)
eng.run(acts[:setup])
eng.run(acts[setup:setup + SKIP])
lib = _native.lib()
lib.qcsim_profile_enable(1)
m0 = eng.metrics().wall_seconds
m = eng.run(acts[setup + SKIP:setup + SKIP + G])
prof = bench.profile_read(lib)
import hashlib
print(f"n={n} {G} gates: {(m.wall_seconds - m0) * 1e3 / G:.3f} ms/gate, ratio {m.mean_compression_ratio:.1f}, "
      f"sha {hashlib.sha256(eng.export_blocks()[0]).hexdigest()[:16]}")
for r in prof[:12]:
    print(f"  {r['kernel']:20s} {r['ms'] / G:8.3f} ms/gate")
