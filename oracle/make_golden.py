"""TEST INFRASTRUCTURE ONLY -- generate tests/golden/ from the REFERENCE itself.

Runs the reference's own codec (oracle/_ref/libqcsim_ref.so, built by
oracle/Makefile from /root/reference/proj/src) on seeded planes and records
SHA-256 of the input, the QCB1 block and the decoded plane.  The oracle
restatement and the GPU path are then pinned against these fixtures on any
machine, without /root/reference.

    python oracle/make_golden.py          # rewrites tests/golden/*.json
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import planes  # noqa: E402
from oracle.oracle import (MODE_ABSOLUTE, MODE_LOSSLESS, MODE_RANGE_RELATIVE, PRED_LINEAR,  # noqa: E402
                           PRED_PREVIOUS, CodecConfig, EngineConfig, OracleError, RefLib)

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

CONFIGS = [
    ("abs1e-5", MODE_ABSOLUTE, 1e-5, 16, PRED_PREVIOUS),
    ("abs1e-3", MODE_ABSOLUTE, 1e-3, 16, PRED_PREVIOUS),
    ("abs1e-7", MODE_ABSOLUTE, 1e-7, 16, PRED_PREVIOUS),
    ("abs1e-5lin", MODE_ABSOLUTE, 1e-5, 16, PRED_LINEAR),
    ("rel1e-2", MODE_RANGE_RELATIVE, 1e-2, 16, PRED_PREVIOUS),
    ("rel1e-4q8lin", MODE_RANGE_RELATIVE, 1e-4, 8, PRED_LINEAR),
    ("lossless", MODE_LOSSLESS, 0.0, 16, PRED_PREVIOUS),
    ("lossless4lin", MODE_LOSSLESS, 0.0, 4, PRED_LINEAR),
    ("absdy_q4", MODE_ABSOLUTE, 2.0**-11, 4, PRED_PREVIOUS),
    ("absdy_q24", MODE_ABSOLUTE, 2.0**-11, 24, PRED_PREVIOUS),
    ("abs1e-4q8", MODE_ABSOLUTE, 1e-4, 8, PRED_PREVIOUS),
]
SIZES = [16, 64, 1024, 65536]


def codec_cases(ref: RefLib):
    cases = []
    for ci, (cname, mode, bound, qb, pred) in enumerate(CONFIGS):
        cfg = CodecConfig.make(mode, bound, qb, pred)
        for ki, kind in enumerate(planes.KINDS):
            for si, n in enumerate(SIZES):
                seed = 1000 * ci + 37 * ki + si + 1
                x = planes.make_plane(kind, n, seed)
                blk = ref.compress(x, cfg)
                dec = ref.decompress(blk.data)
                case = dict(config=cname, mode=mode, bound=bound, qb=qb, pred=pred, kind=kind, n=n,
                            seed=seed, input_sha=planes.sha(x), block_sha=planes.sha(blk.data),
                            block_len=len(blk.data), decoded_sha=planes.sha(dec),
                            ratio=blk.stats.ratio, outlier_fraction=blk.stats.outlier_fraction)
                if n == 16:
                    case["block_hex"] = blk.data.hex()
                cases.append(case)
    return cases


def fuzz_cases(ref: RefLib):
    """Corrupted blocks and the reference's verdict (message or decoded hash)."""
    rng = np.random.Generator(np.random.PCG64(4242))
    out = []
    sources = [("qft", 64, 11, CONFIGS[0]), ("outliers", 64, 12, CONFIGS[0]), ("grover", 256, 13, CONFIGS[0]),
               ("neartie", 64, 14, CONFIGS[8]), ("walk", 128, 15, CONFIGS[3]), ("negzero", 32, 16, CONFIGS[6])]
    for kind, n, seed, (cname, mode, bound, qb, pred) in sources:
        x = planes.make_plane(kind, n, seed)
        blk = bytearray(ref.compress(x, CodecConfig.make(mode, bound, qb, pred)).data)
        for t in range(60):
            b = bytearray(blk)
            op = t % 6
            if op == 0:  # bit flip anywhere
                pos = int(rng.integers(0, len(b) * 8))
                b[pos // 8] ^= 1 << (pos % 8)
            elif op == 1:  # truncate
                b = b[: int(rng.integers(0, len(b)))]
            elif op == 2:  # flip inside the code stream / table region
                lo = 40
                pos = int(rng.integers(lo * 8, len(b) * 8))
                b[pos // 8] ^= 1 << (pos % 8)
            elif op == 3:  # header field edit
                field = int(rng.integers(0, 8))
                b[field] = int(rng.integers(0, 256))
            elif op == 4:  # counts
                off = [8, 24, 32][int(rng.integers(0, 3))]
                b[off] = (b[off] + int(rng.integers(1, 4))) & 0xFF
            else:  # append garbage (trailing bytes are allowed by from_bytes)
                b = b + bytes(int(v) for v in rng.integers(0, 256, size=int(rng.integers(1, 9))))
            rec = dict(source=f"{kind}/{n}/{seed}/{cname}", op=op, block_hex=bytes(b).hex())
            try:
                dec = ref.decompress(bytes(b))
                rec["ok"] = True
                rec["decoded_sha"] = planes.sha(dec)
                rec["n"] = int(dec.size)
            except OracleError as e:
                rec["ok"] = False
                rec["status"] = e.status
                rec["message"] = e.msg
            out.append(rec)
    return out


def engine_cases(ref: RefLib):
    """Reference codec + the pinned engine semantics on small
    circuits: final block bytes and metrics."""
    cases = []
    specs = [
        ("qft8_s4", "qft", (8, 1), 8, 4, 1e-5, 1, 37),
        ("qft10_s6_1e-3", "qft", (10, 1), 10, 6, 1e-3, 1, 5),
        ("qft9_s9", "qft", (9, 1), 9, 9, 1e-5, 1, 300),
        ("qft8_s2_noswap", "qft", (8, 0), 8, 2, 1e-7, 1, 201),
        ("grover6_s3", "grover", (6, 45, 2), 6, 3, 1e-5, 1, 0),
        ("grover8_s4_k3", "grover", (8, 17, 3), 8, 4, 1e-5, 3, 0),
        ("grover7_s7_off", "grover", (7, 100, 2), 7, 7, 1e-5, 0, 0),
    ]
    for name, which, args, n, s, eb, norm_every, basis in specs:
        acts = ref.circuit(which, *args)
        cfg = EngineConfig.make(n, s, CodecConfig.make(MODE_ABSOLUTE, eb, 16, PRED_PREVIOUS), True, norm_every)
        eng = ref.engine(cfg, workers=4)
        if which == "grover":
            eng.load_basis(0)
        else:
            eng.load_basis(basis)
        prefix_sha = []
        for k, a in enumerate(acts):
            eng.gate(a)
            if k % max(1, len(acts) // 8) == 0:
                prefix_sha.append([k + 1, planes.sha(eng.export_blocks())])
        m = eng.metrics()
        cases.append(dict(name=name, circuit=which, args=list(args), n=n, s=s, eb=eb, norm_every=norm_every,
                          basis=basis, gates=len(acts), final_sha=planes.sha(eng.export_blocks()),
                          prefix_sha=prefix_sha, min_ratio=m.min_compression_ratio,
                          mean_ratio=m.mean_compression_ratio, final_norm=m.final_norm,
                          calls=m.compress_calls,
                          actions=[[a.kind, a.target, a.a, a.b, a.mask, list(a.factor), list(a.u)] for a in acts]))
    return cases


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    # A.4 known-answer block
    kat = ref.compress(np.array([0, 0, 0, 0, 0, 0, 6e-5, 1.0]), CodecConfig.make(MODE_ABSOLUTE, 1e-5, 16))
    data = dict(generator="oracle/make_golden.py (reference codec, oracle/_ref/libqcsim_ref.so)",
                kat_a4=dict(block_hex=kat.data.hex(), ratio=kat.stats.ratio),
                codec=codec_cases(ref), fuzz=fuzz_cases(ref), engine=engine_cases(ref))
    with open(os.path.join(OUT, "codec_golden.json"), "w") as f:
        json.dump(data, f, indent=0, sort_keys=True)
    print(f"codec cases {len(data['codec'])}, fuzz {len(data['fuzz'])}, engine {len(data['engine'])}")


if __name__ == "__main__":
    main()
