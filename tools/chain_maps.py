"""Debug: width histogram of the chain-scan thread maps over a run
(QCSIM_CHAIN_DEBUG=1 python tools/chain_maps.py [workload] [gates] [skip])."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402
from paper_1811_05630_b200 import _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "grover20"
gates = int(sys.argv[2]) if len(sys.argv) > 2 else 108
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 324
wl = bench.workload(name)
eng = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"])))
eng.load_basis(wl["basis"])
eng.run(wl["setup"])
acts = []
k = 0
while len(acts) < gates + skip:
    acts += wl["steps"](k)
    k += 1
eng.run(acts[:skip])
lib = _native.lib()
cs = (ctypes.c_uint32 * 5)()
lib.qcsim_debug_chain_stats(cs)  # reset
eng.run(acts[skip:skip + gates])
lib.qcsim_debug_chain_stats(cs)
print("resolve points", cs[0], "refuted", cs[1], "serial chunks", cs[2])
