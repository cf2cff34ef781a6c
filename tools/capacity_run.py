"""Capacity runs beyond a dense FP64 replica's reach (SURVEY.md §8(e) c5,
VERDICT r1 item 3): a state far larger than the dense working set the
engine holds, processed in waves of slices.

    python tools/capacity_run.py qft32 [GATES] [EB]  # 2^32 amplitudes, 64 GiB dense
    python tools/capacity_run.py grover38 [GATES]   # 2^38 amplitudes, 4 TiB dense

Prints one JSON line: geometry, waves, per-gate device seconds, peak device
bytes held by the library, compressed + index bytes.  A full QFT-32 is
checked at sampled slices against its closed form (the DFT column of the
basis state): decoded with the library's own QCB1 decoder.
"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05630_b200 as q  # noqa: E402

name = sys.argv[1]
ngates = sys.argv[2] if len(sys.argv) > 2 else "4"
wl = bench.workload(name, 0, float(sys.argv[3]) if len(sys.argv) > 3 else None)
n, s = wl["n"], wl["s"]
acts = wl["setup"] + [a for k in range(wl["nsteps"]) for a in wl["steps"](k)]
if ngates != "all":
    acts = acts[: int(ngates)]
q.device_memory(reset_peak=True)
t0 = time.time()
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, norm_every=wl["norm_every"],
                              codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"])))
eng.load_basis(wl["basis"])
t_load = time.time() - t0
secs = []
chunk = 8
for k in range(0, len(acts), chunk):
    m0 = eng.metrics().wall_seconds
    m = eng.run(acts[k:k + chunk])
    secs.append((m.wall_seconds - m0) / len(acts[k:k + chunk]))
m = eng.metrics()
mem = q.device_memory()
out = {"workload": name, "n_qubits": n, "slice_bits": s, "slices": 1 << (n - s), "gates": len(acts),
       "dense_bytes": m.dense_bytes, "info": eng.info(), "load_seconds": t_load,
       "device_s_per_gate": {"mean": float(np.mean(secs)) if secs else None, "max": float(np.max(secs)) if secs else None},
       "updates_per_s": (1 << n) * len(acts) / m.wall_seconds if m.wall_seconds else None,
       "peak_device_bytes": mem["peak_bytes"], "compressed_bytes": m.current_compressed_bytes,
       "peak_compressed_bytes": m.peak_compressed_bytes, "index_bytes": m.index_bytes,
       "min_ratio": m.min_compression_ratio, "mean_ratio": m.mean_compression_ratio,
       "norm": "every gate" if wl["norm_every"] else "off (degenerate config, SURVEY F9)"}
if name.startswith("qft") and ngates == "all":
    # closed form: QFT|x> = sum_k exp(2 pi i x k / N) |k> / sqrt(N)
    N = 1 << n
    x = wl["basis"]
    rng = np.random.default_rng(1)
    sl = sorted(rng.choice(1 << (n - s), size=4, replace=False).tolist())
    blob, offs = eng.export_slices(sl)
    blob = bytes(blob)
    err, fid_num, fid_den = 0.0, 0.0 + 0.0j, 0.0
    for k, j in enumerate(sl):
        seg = blob[offs[k]:offs[k + 1]]
        re = q.decompress_bytes(seg)
        # second block follows the first: its length from the first header
        plen = int.from_bytes(seg[32:40], "little")
        im = q.decompress_bytes(seg[40 + plen:])
        idx = (j << s) + np.arange(1 << s, dtype=np.int64)
        want = np.exp(2j * np.pi * ((x * idx) % N) / N) / math.sqrt(N)
        got = re + 1j * im
        err = max(err, float(np.max(np.abs(got - want))))
        fid_num += np.vdot(want, got)
        fid_den += float(np.vdot(want, want).real)
    out["closed_form_check"] = {"slices": sl, "max_abs_err": err,
                                "sampled_overlap": float(abs(fid_num) / fid_den),
                                "basis": "decoded slices vs the DFT column of |x>, eb = %g" % wl["eb"]}
print(json.dumps(out), flush=True)
