"""Stage-by-stage GPU encoder diagnosis against the oracle (run on the GPU box).

    python tools/debug_encode.py [kind n eb qb pred mode] ...
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1811_05630_b200 as q  # noqa: E402
from paper_1811_05630_b200 import _native  # noqa: E402
from oracle import planes  # noqa: E402
from oracle.oracle import CodecConfig as OCfg, Oracle  # noqa: E402


def run_case(o, kind, n, eb, qb=16, pred=0, mode=1, seed=7, verbose=True):
    L = _native.lib()
    fn = L.qcsim_debug_encode
    fn.restype = C.c_int
    x = planes.make_plane(kind, n, seed)
    cfg = _native.CodecConfigC(mode, pred, 0, qb, eb)
    sym = np.zeros(n, np.uint32)
    tsym = np.zeros(n + 1, np.uint32)
    trep = np.zeros(n + 1, np.uint32)
    ntok = C.c_uint64()
    flags = C.c_uint32()
    idx = np.zeros((n // 64 + 2) * 5, np.uint64)
    log2C = C.c_int32()
    rc = fn(x.ctypes.data_as(C.c_void_p), C.c_uint64(n), C.byref(cfg), sym.ctypes.data_as(C.c_void_p),
            tsym.ctypes.data_as(C.c_void_p), trep.ctypes.data_as(C.c_void_p), C.byref(ntok), C.byref(flags),
            idx.ctypes.data_as(C.c_void_p), C.byref(log2C))
    tag = f"{kind}/{n}/eb={eb}/qb={qb}/pred={pred}/mode={mode}"
    if rc:
        print(tag, "ERROR", L.qcsim_last_error().decode())
        return False
    osym = np.zeros(n, np.uint32)
    otsym = np.zeros(n + 1, np.uint32)
    otrep = np.zeros(n + 1, np.uint32)
    ontok = C.c_uint64()
    dec = np.zeros(n)
    ocfg = OCfg.make(mode, eb, qb, pred)
    o.lib.oracle_encode_debug(x.ctypes.data_as(C.c_void_p), C.c_uint64(n), C.byref(ocfg),
                              osym.ctypes.data_as(C.c_void_p), otsym.ctypes.data_as(C.c_void_p),
                              otrep.ctypes.data_as(C.c_void_p), C.byref(ontok), dec.ctypes.data_as(C.c_void_p))
    ok = True
    msgs = [f"flags={flags.value} log2C={log2C.value} ntok gpu={ntok.value} ref={ontok.value}"]
    bad = np.nonzero(sym != osym)[0]
    if bad.size:
        i = bad[0]
        msgs.append(f"SYM mismatch count={bad.size} first={i} gpu={sym[max(0,i-3):i+4]} ref={osym[max(0,i-3):i+4]}")
        ok = False
    else:
        nt = ontok.value
        if ntok.value != nt:
            msgs.append("NTOK mismatch")
            ok = False
        tb = np.nonzero((tsym[:nt] != otsym[:nt]) | (trep[:nt] != otrep[:nt]))[0]
        if tb.size:
            i = tb[0]
            msgs.append(f"TOK mismatch first={i} gpu={list(zip(tsym[i:i+4], trep[i:i+4]))} "
                        f"ref={list(zip(otsym[i:i+4], otrep[i:i+4]))}")
            ok = False
    blk, _ = q.compress_plane(x, q.CodecConfig(q.CodecMode(mode), eb, qb, q.Predictor(pred)))
    data = blk.to_bytes()
    ref = o.compress(x, ocfg).data
    if data != ref:
        ok = False
        m = min(len(data), len(ref))
        d = next((k for k in range(m) if data[k] != ref[k]), m)
        nsym = int.from_bytes(ref[40:44], "little")
        region = "header" if d < 40 else ("table" if d < 44 + 5 * nsym else "stream/outliers")
        msgs.append(f"BYTES differ len gpu={len(data)} ref={len(ref)} first diff @{d} ({region}) nsym={nsym} "
                    f"gpu={data[d:d+8].hex()} ref={ref[d:d+8].hex()}")
    else:
        try:
            dd = q.decompress_plane(blk)
            if dd.tobytes() != o.decompress(ref).tobytes():
                msgs.append("DECODE differs")
                ok = False
        except Exception as e:  # noqa: BLE001
            msgs.append(f"DECODE error {e}")
            ok = False
    if verbose or not ok:
        print(("OK  " if ok else "BAD ") + tag + " | " + " | ".join(msgs), flush=True)
    return ok


if __name__ == "__main__":
    o = Oracle()
    cases = []
    for kind in ["constant", "basis", "grover", "spike", "walk", "qft", "smooth", "gauss", "outliers", "neartie",
                 "negzero", "uniform"]:
        for n in [16, 100, 1024, 1025, 3000, 4096, 65536]:
            cases.append((kind, n, 1e-5))
    good = 0
    for c in cases:
        good += run_case(o, *c, verbose=False)
    print(f"{good}/{len(cases)} cases ok")
