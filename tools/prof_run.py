"""Short engine run for ncu captures: WORKLOAD setup + SKIP untimed gate
passes + G timed gate passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "grover20"
gates = int(sys.argv[2]) if len(sys.argv) > 2 else 30
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = bench.workload(name)
eng = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"],
                              codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"])))
eng.load_basis(wl["basis"])
eng.run(wl["setup"])
acts = []
k = 0
while len(acts) < gates + skip:
    acts += wl["steps"](k)
    k += 1
if skip:
    eng.run(acts[:skip])
m0 = eng.metrics().wall_seconds
rng = os.environ.get("PROF_RANGE") == "1"  # ncu --profile-from-start off: profile only the timed gates
if rng:
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
m = eng.run(acts[skip:skip + gates])
if rng:
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print(f"{name}: {gates} gates after {skip}, device {(m.wall_seconds - m0)*1e3:.2f} ms, "
      f"min ratio {m.min_compression_ratio:.3f}, launches {q.kernel_launches()}")
