"""decompress_plane on a foreign QCB1 block (no decode index): GPU
(libqcsim_b200: validating token walk + chunk-parallel decode) vs the
reference's own decompress_plane (oracle/_ref, one core -- the reference
decodes a plane serially).  python tools/foreign_decode_bench.py [KIND] [N]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_05630_b200 as q  # noqa: E402
from oracle import planes  # noqa: E402
from oracle.oracle import CodecConfig as OCfg, RefLib  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "qft"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
out = []
for eb in (1e-3, 1e-5, 1e-7):
    x = planes.make_plane(kind, n, 7)
    ref = RefLib()
    blk = ref.compress(x, OCfg.make(1, eb, 16, 0)).data
    # reference decode (one core): one ref_decompress_plane call per decode
    import ctypes as C
    b = np.frombuffer(blk, dtype=np.uint8).copy()
    d_ref = np.empty(n, dtype=np.float64)
    nn = C.c_uint64()
    t0 = time.perf_counter()
    reps = 0
    while True:
        rc = ref.lib.ref_decompress_plane(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.size,
                                          d_ref.ctypes.data_as(C.POINTER(C.c_double)), n, C.byref(nn), None)
        assert rc == 0
        reps += 1
        if time.perf_counter() - t0 > 1.0:
            break
    t_ref = (time.perf_counter() - t0) / reps
    d = q.decompress_bytes(blk)  # warm-up
    assert d.tobytes() == np.asarray(d_ref).tobytes()
    t0 = time.perf_counter()
    reps = 0
    while True:
        d = q.decompress_bytes(blk)
        reps += 1
        if time.perf_counter() - t0 > 1.0:
            break
    t_gpu = (time.perf_counter() - t0) / reps
    out.append({"kind": kind, "n": n, "eb": eb, "block_bytes": len(blk), "ref_ms": 1e3 * t_ref,
                "gpu_ms_incl_h2d_d2h": 1e3 * t_gpu, "speedup": t_ref / t_gpu, "bit_exact": True})
print(json.dumps(out))
