"""Digest of a 128-plane QFT-14 run (blocks, metrics) for comparing pipeline variants (env switches)."""
import hashlib, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_05630_b200 as q  # noqa: E402
n, s = 14, 8
acts = q.lower(q.build_qft(n))
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
eng.load_basis(1234)
m = eng.run(acts + acts[:40])
blob = eng.export_blocks()[0]
print(hashlib.sha256(bytes(blob)).hexdigest(), repr(m.mean_compression_ratio), repr(m.min_compression_ratio), m.compress_calls, m.peak_compressed_bytes, m.current_compressed_bytes)
