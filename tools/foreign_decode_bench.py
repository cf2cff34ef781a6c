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
    from paper_1811_05630_b200 import _native
    import bench
    lib = _native.lib()
    lib.qcsim_profile_enable(1)
    q.decompress_bytes(blk)
    ks = {r["kernel"]: round(r["ms"], 3) for r in bench.profile_read(lib)}
    # a batch of planes through the device API (imports / checkpoint restore):
    # planes decode concurrently
    import torch
    P = 64
    dev = torch.tensor(np.frombuffer(blk * P, dtype=np.uint8), device="cuda")
    offs = (C.c_uint64 * (P + 1))(*[k * len(blk) for k in range(P + 1)])
    outs = torch.empty((P, n), dtype=torch.float64, device="cuda")
    ptrs = (C.c_void_p * P)(*[outs[k].data_ptr() for k in range(P)])
    caps = (C.c_uint64 * P)(*([n] * P))
    fn = lib.qcsim_decompress_planes_device
    fn.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p]
    assert fn(dev.data_ptr(), offs, P, ptrs, caps, None) == 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert fn(dev.data_ptr(), offs, P, ptrs, caps, None) == 0
    torch.cuda.synchronize()
    t_batch = (time.perf_counter() - t0) / P
    assert outs[P - 1].cpu().numpy().tobytes() == d_ref.tobytes()
    out.append({"kind": kind, "n": n, "eb": eb, "block_bytes": len(blk), "ref_ms": 1e3 * t_ref,
                "gpu_batch64_ms_per_plane": 1e3 * t_batch, "batch_speedup_vs_ref_16_cores": t_ref / 16 / t_batch,
                "gpu_ms_incl_h2d_d2h": 1e3 * t_gpu, "speedup": t_ref / t_gpu, "bit_exact": True, "kernels_ms": ks})
print(json.dumps(out))
