"""Short engine run for ncu captures: WORKLOAD setup + G gate passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "grover20"
gates = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = bench.workload(name)
eng = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"],
                              codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"])))
eng.load_basis(wl["basis"])
eng.run(wl["setup"])
acts = []
k = 0
while len(acts) < gates:
    acts += wl["steps"](k)
    k += 1
m = eng.run(acts[:gates])
print(f"{name}: {gates} gates, device {m.wall_seconds*1e3:.2f} ms, min ratio {m.min_compression_ratio:.3f}, "
      f"launches {q.kernel_launches()}")
