"""Per-kernel device time of G gate passes of a bench workload after its
setup + SKIP passes (qcsim_profile_* CUDA events):
python tools/kshare.py WORKLOAD G SKIP"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402
from paper_1811_05630_b200 import _native  # noqa: E402

name, G, skip = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
wl = bench.workload(name)
eng = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], norm_every=wl["norm_every"],
                              codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"])))
eng.load_basis(wl["basis"])
eng.run(wl["setup"])
acts, k = [], 0
while len(acts) < G + skip:
    acts += wl["steps"](k)
    k += 1
eng.run(acts[:skip])
lib = _native.lib()
m0 = eng.metrics().wall_seconds
lib.qcsim_profile_enable(1)
m = eng.run(acts[skip:skip + G])
ks = bench.profile_read(lib)
print(f"{name} {os.environ.get('QCSIM_IDX_BPC', '')}: {G} passes, {1e3 * (m.wall_seconds - m0) / G:.2f} ms/pass, "
      f"waves {eng.info()['waves']}, index {m.index_bytes} / blocks {m.current_compressed_bytes}")
for r in ks[:12]:
    print(f"   {r['kernel']:20s} {r['ms'] / G:8.3f} ms/pass  ({r['launches']} launches)")
