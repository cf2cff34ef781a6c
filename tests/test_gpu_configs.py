"""GPU engine parity at the benchmarked configurations (BASELINE.json
configs[1..3]) and for the engine's batching variants.

Every case hashes the GPU engine's QCB1 arena and compares it with the
reference engine loop over the reference's own codec (oracle/_ref, compiled
from /root/reference; the C restatement when _ref is absent) replaying the
identical gate prefix.  Bit-exact blocks imply bit-exact decoded amplitudes,
ratios and norms."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import Action, CodecConfig as OCfg, EngineConfig as OEng, REF_SO, Oracle, RefLib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    import paper_1811_05630_b200 as q
    return q


def _ref_engine(n, s, eb, norm_every=1):
    cfg = OEng.make(n, s, OCfg.make(1, eb, 16, 0), True, norm_every)
    if os.path.exists(REF_SO):
        eng = RefLib().engine(cfg, workers=os.cpu_count() or 1)
        return eng, lambda a: eng.gate(Action.from_buffer_copy(bytes(a)))
    eng = Oracle().engine(cfg)
    return eng, lambda a: eng.run([a])


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def _parity(q, n, s, eb, basis, acts, checkpoints=(), norm_every=1):
    """GPU engine vs the reference engine over `acts`; SHA-256 of the whole
    arena compared after every gate count in `checkpoints` and at the end."""
    eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, eb),
                                  norm_every=norm_every))
    ref, gate = _ref_engine(n, s, eb, norm_every)
    eng.load_basis(basis)
    ref.load_basis(basis)
    marks = sorted(set(list(checkpoints) + [len(acts)]))
    done = 0
    for mk in marks:
        eng.run(acts[done:mk])
        for a in acts[done:mk]:
            gate(a)
        done = mk
        assert _sha(eng.export_blocks_array()[0]) == _sha(ref.export_blocks()), f"blocks differ after {mk} gates"
    m = eng.metrics()
    rm = ref.metrics()
    assert m.min_compression_ratio == rm.min_compression_ratio
    assert m.compress_calls == rm.compress_calls
    assert m.final_norm == rm.final_norm
    return eng, m


def test_grover20_s14_two_iterations(q):
    """configs[1] geometry: 64 slices x 2^14 (128 planes: per-plane
    hand-offs, multi-chunk chain scan, fixed slots, deferred loop), the H
    layer plus two full Grover iterations (236 gate passes)."""
    n, s = 20, 14
    marked = q.seeded_index(n, 20)
    acts = ([q.to_action_c(q.gate_action(q.Gate.h(k))) for k in range(n)]
            + q.lower(q.build_grover(n, marked, 2))[n:])
    eng, m = _parity(q, n, s, 1e-5, 0, acts, checkpoints=(n, n + 108))
    rows = eng.gate_metrics()
    assert len(rows) == len(acts) + 1
    assert min(r["min_ratio"] for r in rows) == m.min_compression_ratio
    assert rows[-1]["bytes"] == m.current_compressed_bytes


@pytest.mark.parametrize("eb", [1e-3, 1e-5, 1e-7])
def test_qft28_prefix(q, eb):
    """configs[2] geometry (256 slices x 2^20: 512 planes, serial warp chain,
    host-synchronous loop) at each error bound of the sweep: the first 40
    gates of QFT-28 on its seeded basis state (H + controlled phases on the
    top qubits, cross-slice butterflies)."""
    n, s = 28, 20
    acts = q.lower(q.build_qft(n))[:40]
    _parity(q, n, s, eb, q.seeded_index(n, n), acts, checkpoints=(1, 20))


def test_random30_layer(q):
    """configs[3] (1024 slices x 2^20, 2048 planes): the U3 half of the
    depth-20 random circuit's first layer plus its first CZs, which turn |0>
    into the dense low-compressibility state the benchmark times (bench.py
    pins the full 58-gate prefix of its timed window the same way)."""
    n, s = 30, 20
    acts = q.random_u3_circuit_actions(n, 20, seed=30)[:33]
    eng, m = _parity(q, n, s, 1e-5, 0, acts, checkpoints=(21, 30))
    assert m.index_bytes <= 0.1 * m.current_compressed_bytes


_WAVES_SCRIPT = r"""
import hashlib, sys
import numpy as np
import paper_1811_05630_b200 as q
case = sys.argv[1]
G = q.Gate
if case == "qft":
    n, s = 16, 8
    acts = q.lower(q.build_qft(n))
    eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    eng.load_basis(4321)
else:
    n, s = 10, 4
    gates = [G.h(k) for k in range(n)] + [G.cnot(7, 2), G.cnot(1, 8), G.swap(3, 6), G.swap(5, 8), G.swap(6, 9),
             G.swap(0, 1), G.y(6), G.t(8), G.cphase(0.3, 2, 7), G.mcz([0, 5, 8]), G.x(4), G.phase(1.1, 5)]
    acts = [q.to_action_c(q.gate_action(g)) for g in gates] + q.random_u3_circuit_actions(n, 2, seed=9)
    rng = np.random.default_rng(3)
    amps = rng.standard_normal(2 << n)
    amps /= np.linalg.norm(amps)
    eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    eng.load_amplitudes(amps)
m = eng.run(acts)
info = eng.info()
rows = eng.gate_metrics()
blob = eng.export_blocks()[0]
amps = eng.gather()
print(info["waves"], hashlib.sha256(blob).hexdigest(), hashlib.sha256(amps.tobytes()).hexdigest(),
      repr(m.mean_compression_ratio), repr(m.min_compression_ratio), m.index_bytes,
      repr([(r["min_ratio"], r["bytes"], r["index_bytes"]) for r in rows]))
"""


def _run_script(script, args, env_extra):
    e = dict(os.environ)
    for k in ("QCSIM_WAVE_SLICES", "QCSIM_SYNC_GATES", "QCSIM_FOREIGN_SERIAL", "QCSIM_FUSE_GL", "QCSIM_ZERO_TILES",
              "QCSIM_ENCX_VEC", "QCSIM_PACK_COUNT", "QCSIM_CHAIN_PIPE"):
        e.pop(k, None)
    e.update(env_extra)
    r = subprocess.run([sys.executable, "-c", script] + args, cwd=ROOT, env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout.strip().splitlines()[-1].split(" ", 1)


@pytest.mark.parametrize("case", ["qft", "cross"])
@pytest.mark.parametrize("wave", ["4", "8"])
def test_waves_bit_identical(case, wave):
    """A gate pass in waves (each wave closed under the gate's partner mask,
    decode tables parsed from the blocks, blocks appended wave by wave)
    produces the same blocks, amplitudes, per-gate metrics and index as one
    batch -- including swaps with both qubits in the slice index."""
    w_many, rest_many = _run_script(_WAVES_SCRIPT, [case], {"QCSIM_WAVE_SLICES": wave})
    w_one, rest_one = _run_script(_WAVES_SCRIPT, [case], {"QCSIM_SYNC_GATES": "1"})
    assert int(w_many) > 1 and int(w_one) == 1
    assert rest_many == rest_one


def test_waves_vs_oracle(q, oracle):
    """Waves against the C oracle directly (QFT-14, 64 slices in waves of 4)."""
    script = r"""
import sys
import paper_1811_05630_b200 as q
n, s = 14, 8
acts = q.lower(q.build_qft(n))
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
eng.load_basis(999)
eng.run(acts)
sys.stdout.write(str(eng.info()["waves"]) + " " + eng.export_blocks()[0].hex() + "\n")
"""
    waves, hexblob = _run_script(script, [], {"QCSIM_WAVE_SLICES": "4"})
    assert int(waves) == 16
    oe = oracle.engine(OEng.make(14, 8, OCfg.make(1, 1e-5, 16, 0)))
    oe.load_basis(999)
    oe.run(q.lower(q.build_qft(14)))
    assert bytes.fromhex(hexblob) == oe.export_blocks()[0]


def _block_sizes(blob):
    out, pos = [], 0
    while pos < len(blob):
        payload = int.from_bytes(blob[pos + 32:pos + 40], "little")
        out.append(40 + payload)
        pos += 40 + payload
    return out


@pytest.mark.parametrize("waves", [False, True])
def test_gate_metrics_vs_oracle(q, oracle, waves):
    """Per-gate rows (SPEC.md:310 per_gate_min_ratio, :383 CSV fields) equal
    the oracle's per-gate block sizes, on the deferred loop and on the
    host-synchronous wave loop."""
    n, s = 12, 6
    acts = q.lower(q.build_grover(n, q.seeded_index(n, 5), 1))
    eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5),
                                  wave_bytes=1 if waves else 0))
    assert (eng.info()["waves"] > 1) == waves
    oe = oracle.engine(OEng.make(n, s, OCfg.make(1, 1e-5, 16, 0)))
    eng.load_basis(0)
    oe.load_basis(0)
    want = []
    want.append(_block_sizes(oe.export_blocks()[0]))
    for a in acts:
        oe.run([a])
        want.append(_block_sizes(oe.export_blocks()[0]))
    eng.run(acts)
    rows = eng.gate_metrics()
    assert len(rows) == len(want)
    L = 1 << s
    for k, (r, sz) in enumerate(zip(rows, want)):
        ratios = [8.0 * L / b for b in sz]
        assert r["min_ratio"] == min(ratios), k
        assert r["mean_ratio"] == pytest.approx(sum(ratios) / len(ratios), rel=1e-14), k
        assert r["bytes"] == sum(sz), k
        assert r["calls"] == len(sz)
        if k:
            assert r["seconds"] > 0.0
    m = eng.metrics()
    assert m.min_compression_ratio == min(r["min_ratio"] for r in rows)


def test_index_bounded_by_block_bytes(q):
    """The decode index lives next to each block and is <= 7.8% of it
    (one 40-byte record per 512 block bytes), on sparse and dense states."""
    for n, s, acts, basis in [(16, 12, q.lower(q.build_qft(16)), 77),
                              (12, 8, q.random_u3_circuit_actions(12, 3, seed=4), 0),
                              (14, 10, q.lower(q.build_grover(14, 5, 3)), 0)]:
        eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
        eng.load_basis(basis)
        m = eng.run(acts)
        assert m.index_bytes <= 0.078 * m.current_compressed_bytes + 1, (n, m.index_bytes)
        for r in eng.gate_metrics():
            assert r["index_bytes"] <= 0.078 * r["bytes"] + 1


def test_device_memory_bounded_by_waves(q):
    """wave_bytes bounds the dense working set: the same circuit with a
    budget of ~1/8 of the one-batch working set allocates less and produces
    identical blocks."""
    n, s = 22, 16
    acts = q.random_u3_circuit_actions(n, 1, seed=2)[:12]
    res = []
    for wb in (0, 48 << 20):
        q.device_memory(reset_peak=True)
        base = q.device_memory()["current_bytes"]
        eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5),
                                      wave_bytes=wb))
        eng.load_basis(0)
        eng.run(acts)
        res.append((eng.info()["waves"], q.device_memory()["peak_bytes"] - base,
                    hashlib.sha256(eng.export_blocks_array()[0]).hexdigest()))
        eng.close()
    (w0, p0, h0), (w1, p1, h1) = res
    assert w0 == 1 and w1 > 1
    assert h0 == h1
    assert p1 < p0 / 2, (p0, p1)


def test_compare_dense_in_waves(q):
    """On-device accuracy check wave by wave (compressed engine in waves vs
    the compression-off engine) equals the one-batch comparison."""
    n, s = 14, 8
    acts = q.lower(q.build_qft(n))
    out = []
    for wb in (0, 2 << 20):
        comp = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5),
                                       wave_bytes=wb))
        dense = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, compression_enabled=False))
        for e in (comp, dense):
            e.load_basis(4242)
            e.run(acts)
        out.append((comp.info()["waves"], comp.compare(dense)))
    assert out[0][0] == 1 and out[1][0] > 1
    assert out[0][1] == out[1][1]
    assert out[0][1]["fidelity"] > 0.999


class _InProcessRanks:
    """`world` CUDA engines (ranks) on one device driven like
    distributed.ShardedEngine, with the exchange done in-process: per gate,
    every rank imports the compressed partner slices it needs (X1) and gets
    the all-gathered sq_norm table (X2)."""

    def __init__(self, q, cfg_kw, world):
        self.engs = [q.Engine(q.EngineConfig(rank=r, world=world, **cfg_kw)) for r in range(world)]

    def _norms(self):
        allsq = np.concatenate([e.slice_norms() for e in self.engs])
        for e in self.engs:
            e.set_global_norms(allsq)

    def load_basis(self, x):
        for e in self.engs:
            e.load_basis(x)
        self._norms()

    def run(self, acts, device=False):
        import torch
        ns = self.engs[0].local_slices
        for a in acts:
            keep = []
            for e in self.engs:
                need = e.partner_slices_needed(a)
                if not need:
                    continue
                if device:  # device-direct: peer gathers into a device buffer, e decodes from it
                    owner = self.engs[need[0] // ns]
                    total, offs = owner.export_slices_device(need)
                    buf = torch.empty(max(1, total), dtype=torch.uint8, device="cuda")
                    owner.export_slices_device(need, buf.data_ptr(), buf.numel())
                    e.import_partners_device(need, buf.data_ptr(), offs)
                    keep.append(buf)
                else:
                    for pj in need:
                        e.import_partner(pj, self.engs[pj // ns].export_slice(pj))
            for e in self.engs:
                e.run([a])
            self._norms()

    def blocks(self):
        return b"".join(e.export_blocks()[0] for e in self.engs)


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("world", [2, 4])
def test_ranks_on_one_gpu_vs_single(q, world, device):
    """The multi-rank CUDA path (export_slice / import_partner, or the
    device-direct export_slices_device / import_partners_device; validating
    decode of imported partners with on-device header checks;
    set_global_norms; remote slot layout) with `world` engines as logical
    ranks on one GPU: byte-identical to one engine, including butterflies and
    swaps on the rank bits."""
    n, s = 12, 6
    G = q.Gate
    gates = [G.h(k) for k in range(n)] + [G.cnot(11, 2), G.swap(3, 11), G.swap(10, 11), G.swap(7, 10), G.y(11),
                                          G.cphase(0.4, 1, 11), G.mcz([0, 6, 11]), G.x(10)]
    acts = [q.to_action_c(q.gate_action(g)) for g in gates] + q.random_u3_circuit_actions(n, 1, seed=7)
    kw = dict(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5))
    one = q.Engine(q.EngineConfig(**kw))
    one.load_basis(1234)
    one.run(acts)
    ranks = _InProcessRanks(q, kw, world)
    ranks.load_basis(1234)
    ranks.run(acts, device=device)
    assert ranks.blocks() == one.export_blocks()[0]
    m1 = one.metrics()
    assert sum(e.metrics().compress_calls for e in ranks.engs) == m1.compress_calls


def test_measure_overhead_and_report(q, tmp_path):
    """SPEC.md:353-361 overhead factor (compressed vs compression-off wall on
    the same GPU) and the JSON / CSV metrics report."""
    import json
    n, s = 14, 8
    acts = q.lower(q.build_qft(n))
    cfg = q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5))
    m = q.measure_overhead(acts, cfg, basis=77)
    assert m.baseline_wall_seconds > 0 and m.overhead_factor > 1.0
    assert len(m.per_gate_min_ratio) == len(acts)
    assert min(m.per_gate_min_ratio) >= m.min_compression_ratio
    eng = q.Engine(cfg)
    eng.load_basis(77)
    eng.run(acts)
    d = eng.write_report(tmp_path / "m.json", tmp_path / "m.csv")
    assert json.loads((tmp_path / "m.json").read_text())["gates"] == len(acts)
    assert len(d["per_gate"]) == len(acts) + 1 and d["per_gate"][0]["gate_index"] == -1
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "gate_index,min_ratio,mean_ratio,seconds" and len(lines) == len(acts) + 2


def test_device_import_rejects_corrupt(q):
    """A corrupt device-resident partner block fails with the reference's
    from_bytes message (header checks on the device)."""
    import torch
    kw = dict(num_qubits=8, slice_bits=4, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5))
    a = q.Engine(q.EngineConfig(rank=0, world=2, **kw))
    b = q.Engine(q.EngineConfig(rank=1, world=2, **kw))
    for e in (a, b):
        e.load_basis(3)
    act = q.to_action_c(q.gate_action(q.Gate.h(7)))
    need = a.partner_slices_needed(act)
    total, offs = b.export_slices_device(need)
    buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    b.export_slices_device(need, buf.data_ptr(), total)
    buf[0] = ord("X")  # first block's magic
    a.import_partners_device(need, buf.data_ptr(), offs)
    with pytest.raises(q.CodecError, match="bad block magic"):
        a.run([act])


_FOREIGN_SCRIPT = r"""
import hashlib, sys
import numpy as np
import paper_1811_05630_b200 as q
from oracle import planes
h = hashlib.sha256()
for kind in ("qft", "gauss", "walk", "outliers", "grover", "smooth", "uniform"):
    for n in (1000, 1 << 16, 1 << 20):
        for eb in (1e-3, 1e-5, 1e-7):
            x = planes.make_plane(kind, n, 11)
            blk, _ = q.compress_plane(x, q.CodecConfig(q.CodecMode.Absolute, eb))
            h.update(q.decompress_plane(blk).tobytes())
print(h.hexdigest())
"""


def test_foreign_decode_parallel_vs_serial():
    """decompress_plane of index-less blocks: the parallel path (speculative
    segments, resync, event chain, chunk-parallel decode) gives the same bytes
    as the serial validating walk, on dense and sparse planes of every size
    (the fuzz verdicts of test_gpu_codec cover the error paths)."""
    fast = _run_script(_FOREIGN_SCRIPT, [], {})
    slow = _run_script(_FOREIGN_SCRIPT, [], {"QCSIM_FOREIGN_SERIAL": "1"})
    assert fast == slow


_FUSE_SCRIPT = r"""
import hashlib, sys
import paper_1811_05630_b200 as q
n, s = 19, 17  # 4 slices of 2^17: 128 tiles per plane (the fused gate + lattice grid)
acts = q.lower(q.build_qft(n))[:60] + q.random_u3_circuit_actions(n, 1, seed=3)
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
eng.load_basis(12345)
m = eng.run(acts)
print(hashlib.sha256(eng.export_blocks()[0]).hexdigest(), repr(m.mean_compression_ratio), m.fallback_planes)
"""


def test_fused_gate_lattice_bit_identical(oracle):
    """The fused gate + lattice grid (planes of > 64 tiles; planes holding a
    speculative outlier are redone by the lattice grid -- the basis state's
    1.0 is one) produces the same blocks as the two separate grids, with and
    without the run-aware tile paths, and as the C oracle."""
    fused = _run_script(_FUSE_SCRIPT, [], {})
    split = _run_script(_FUSE_SCRIPT, [], {"QCSIM_FUSE_GL": "0"})
    plain = _run_script(_FUSE_SCRIPT, [], {"QCSIM_FUSE_GL": "0", "QCSIM_ZERO_TILES": "0", "QCSIM_ENCX_VEC": "0",
                                           "QCSIM_PACK_COUNT": "1", "QCSIM_CHAIN_PIPE": "0"})
    pipe = _run_script(_FUSE_SCRIPT, [], {"QCSIM_CHAIN_PIPE": "0", "QCSIM_PACK_COUNT": "1"})
    assert fused == split == plain == pipe
    import paper_1811_05630_b200 as q
    n, s = 19, 17
    acts = q.lower(q.build_qft(n))[:60] + q.random_u3_circuit_actions(n, 1, seed=3)
    oe = oracle.engine(OEng.make(n, s, OCfg.make(1, 1e-5, 16, 0)))
    oe.load_basis(12345)
    oe.run(acts)
    assert fused[0] == hashlib.sha256(oe.export_blocks()[0]).hexdigest()


_RESUME_SCRIPT = r"""
import sys
import numpy as np
import paper_1811_05630_b200 as q
n, s = 14, 8
acts = q.lower(q.build_qft(n))
cut = 60
cfg = q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5))
a = q.Engine(cfg)
a.load_basis(777)
a.run(acts[:cut])
blob, offs = a.export_blocks()
norms = a.slice_norms()
b = q.Engine(cfg)
b.load_blocks(blob, offs, norms, gates_done=cut)
same_ckpt = b.export_blocks()[0] == blob
mb = b.run(acts[cut:])
ma = a.run(acts[cut:])
ok = same_ckpt and b.export_blocks()[0] == a.export_blocks()[0] and np.array_equal(a.slice_norms(), b.slice_norms())
ok = ok and ma.final_norm == mb.final_norm and mb.gates == len(acts)
bad = bytearray(blob)
bad[offs[3] + 1] ^= 0xFF                     # magic of block 3
try:
    q.Engine(cfg).load_blocks(bytes(bad), offs, norms)
    ok = False
except q.CodecError as e:
    ok = ok and "bad block magic" in str(e)
sys.stdout.write(str(b.info()["waves"]) + " " + str(ok) + " " + a.export_blocks()[0].hex() + "\n")
"""


@pytest.mark.parametrize("wave", [None, "4"])
def test_resume_from_checkpoint(oracle, q, wave):
    """Checkpoint / resume: QCB1 blocks + the sq_norm table
    exported after 60 gates of QFT-14 are loaded into a fresh engine
    (qcsim_engine_load_blocks: from_bytes + decoder checks, decode and
    re-encode on the device), which then holds byte-identical blocks and
    finishes the circuit exactly like the uninterrupted engine and the
    oracle.  A corrupt checkpoint fails with the reference's message."""
    env = {"QCSIM_WAVE_SLICES": wave} if wave else {}
    waves, rest = _run_script(_RESUME_SCRIPT, [], env)
    ok, hexblob = rest.split(" ", 1)
    assert int(waves) == (16 if wave else 1)
    assert ok == "True"
    oe = oracle.engine(OEng.make(14, 8, OCfg.make(1, 1e-5, 16, 0)))
    oe.load_basis(777)
    oe.run(q.lower(q.build_qft(14)))
    assert bytes.fromhex(hexblob) == oe.export_blocks()[0]
