"""GPU engine parity: every gate pass (decode -> normalize -> gate ->
sq_norm -> encode) bit-exact with the CPU oracle engine and the
reference-codec golden runs; physics checks against the dense reference."""
import math

import numpy as np
import pytest

from oracle import planes
from oracle.oracle import Action, CodecConfig as OCfg, EngineConfig as OEng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1811_05630_b200 as q
    return q


def _golden_actions(rows):
    out = []
    for kind, target, a, b, mask, factor, u in rows:
        act = Action()
        act.kind, act.target, act.a, act.b, act.mask = kind, target, a, b, mask
        act.factor[0], act.factor[1] = factor
        for i in range(8):
            act.u[i] = u[i]
        out.append(act)
    return out


def _to_c(q, acts):
    out = []
    for a in acts:
        c = q._native.ActionC()
        C_bytes = bytes(a)
        import ctypes
        ctypes.memmove(ctypes.addressof(c), C_bytes, ctypes.sizeof(c))
        out.append(c)
    return out


@pytest.mark.parametrize("idx", range(7))
def test_engine_golden(q, golden, idx):
    """Reference codec + pinned engine semantics (tests/golden) == GPU."""
    e = golden["engine"][idx]
    acts = _to_c(q, _golden_actions(e["actions"]))
    cfg = q.EngineConfig(num_qubits=e["n"], slice_bits=e["s"], codec=q.CodecConfig(q.CodecMode.Absolute, e["eb"]),
                         norm_every=e["norm_every"])
    eng = q.Engine(cfg)
    eng.load_basis(e["basis"])
    prefix = dict((k, h) for k, h in e["prefix_sha"])
    for k, a in enumerate(acts):
        eng.run([a])
        if k + 1 in prefix:
            assert planes.sha(eng.export_blocks()[0]) == prefix[k + 1], f"{e['name']} gate {k + 1}"
    m = eng.metrics()
    assert planes.sha(eng.export_blocks()[0]) == e["final_sha"]
    assert m.min_compression_ratio == e["min_ratio"]
    assert m.final_norm == e["final_norm"]
    assert m.compress_calls == e["calls"]


def _run_both(q, oracle, n, s, acts, eb=1e-5, basis=0, norm_every=1, per_gate=False, amps=None):
    cfg = q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, eb),
                         norm_every=norm_every)
    eng = q.Engine(cfg)
    oe = oracle.engine(OEng.make(n, s, OCfg.make(1, eb, 16, 0), True, norm_every))
    if amps is None:
        eng.load_basis(basis)
        oe.load_basis(basis)
    else:
        eng.load_amplitudes(amps)
        oe.load_amplitudes(amps)
    if per_gate:
        for k, a in enumerate(acts):
            eng.run([a])
            oe.run([a])
            assert eng.export_blocks()[0] == oe.export_blocks()[0], f"gate {k}"
    else:
        eng.run(acts)
        oe.run(acts)
    assert eng.export_blocks()[0] == oe.export_blocks()[0]
    assert np.array_equal(eng.slice_norms(), oe.slice_norms())
    return eng, oe


@pytest.mark.parametrize("n,s", [(12, 8), (14, 10), (16, 12)])
def test_qft_vs_oracle(q, oracle, n, s):
    acts = q.lower(q.build_qft(n))
    x = q.seeded_index(n, 1234 + n)
    eng, oe = _run_both(q, oracle, n, s, acts, basis=x)
    m = eng.metrics()
    om = oe.run([])
    assert m.min_compression_ratio == om.min_compression_ratio
    assert m.mean_compression_ratio == pytest.approx(om.mean_compression_ratio, rel=1e-15)
    assert m.peak_compressed_bytes == om.peak_compressed_bytes


def test_qft16_closed_form(q):
    """Config 1 physics: QFT16|x> vs the closed-form DFT column (eb 1e-5)."""
    n, s = 16, 12
    x = q.seeded_index(n, 1)
    eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    eng.load_basis(x)
    m = eng.run(q.build_qft(n))
    z = eng.amplitudes()
    N = 1 << n
    k = np.arange(N)
    want = np.exp(2j * np.pi * ((x * k) % N) / N) / math.sqrt(N)
    err = np.max(np.abs(z - want))
    fid = abs(np.vdot(want, z)) ** 2
    assert err < 1e-3 and fid > 0.99, (err, fid)
    assert m.min_compression_ratio > 1.0


def test_grover_vs_oracle(q, oracle):
    n, s = 10, 6
    marked = q.seeded_index(n, 99)
    acts = q.lower(q.build_grover(n, marked, 3))
    _run_both(q, oracle, n, s, acts, per_gate=True)


def test_grover_many_planes_vs_oracle(q, oracle):
    """128 planes: the per-plane hand-offs (chain -> verify -> serial ->
    tok_count) and fixed-slot packing of the deferred loop are active."""
    n, s = 12, 6
    marked = q.seeded_index(n, 7)
    acts = q.lower(q.build_grover(n, marked, 2))
    eng, oe = _run_both(q, oracle, n, s, acts)
    m = eng.metrics()
    om = oe.run([])
    assert m.min_compression_ratio == om.min_compression_ratio
    assert m.mean_compression_ratio == pytest.approx(om.mean_compression_ratio, rel=1e-15)
    assert m.compress_calls == om.compress_calls


@pytest.mark.parametrize("n,s,norm_every", [(12, 6, 3), (10, 5, 1), (10, 5, 0)])
def test_deferred_variants_vs_oracle(q, oracle, n, s, norm_every):
    """Deferred-loop bookkeeping at the edges: passes without normalization
    (run metrics still accumulated by the decoder-grid block) and a batch of
    exactly 64 planes (the smallest with per-plane hand-offs)."""
    marked = q.seeded_index(n, 11)
    acts = q.lower(q.build_grover(n, marked, 2))
    eng, oe = _run_both(q, oracle, n, s, acts, norm_every=norm_every)
    m = eng.metrics()
    om = oe.run([])
    assert m.min_compression_ratio == om.min_compression_ratio
    assert m.mean_compression_ratio == pytest.approx(om.mean_compression_ratio, rel=1e-15)
    assert m.compress_calls == om.compress_calls
    assert m.peak_compressed_bytes == om.peak_compressed_bytes


def test_cross_slice_gates(q, oracle):
    """Butterflies/swaps/controls on slice-index bits (pairing)."""
    n, s = 9, 4
    G = q.Gate
    gates = [G.h(q_) for q_ in range(n)] + [G.cnot(7, 2), G.cnot(1, 8), G.swap(3, 6), G.swap(5, 8), G.swap(0, 1),
                                           G.y(6), G.t(8), G.cphase(0.3, 2, 7), G.mcz([0, 5, 8]), G.x(4),
                                           G.phase(1.1, 5), G.s(0), G.z(7), G.cz(6, 8)]
    acts = [q.to_action_c(q.gate_action(g)) for g in gates]
    rng = np.random.default_rng(3)
    amps = rng.standard_normal(2 << n)
    amps /= np.linalg.norm(amps)
    _run_both(q, oracle, n, s, acts, per_gate=True, amps=amps)


def test_random_u3_vs_oracle(q, oracle):
    """Config-4 structure (U3 layers + CZ matchings) at small scale."""
    n, s = 10, 6
    acts = q.random_u3_circuit_actions(n, 3, seed=5)
    _run_both(q, oracle, n, s, acts, basis=0, per_gate=False)


def test_lossless_engine_vs_dense(q, oracle):
    """compression off + norm off == dense reference <= 1e-12."""
    n = 10
    acts = q.lower(q.build_qft(n))
    for s in (4, 8, 10):
        eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, compression_enabled=False, norm_every=0))
        eng.load_basis(300)
        eng.run(acts)
        amps = np.zeros(2 << n)
        amps[600] = 1.0
        ref = oracle.ref_run(n, amps, acts)
        assert np.max(np.abs(eng.gather() - ref)) <= 1e-12


def test_norm_drift_error(q):
    eng = q.Engine(q.EngineConfig(num_qubits=6, slice_bits=3, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    amps = np.zeros(2 << 6)
    amps[0] = 2.0  # |psi|^2 = 4: beyond 10x tolerance
    eng.load_amplitudes(amps)
    with pytest.raises(q.NumericError):
        eng.run(q.lower(q.build_qft(6)))


def test_gather_guard(q):
    eng = q.Engine(q.EngineConfig(num_qubits=12, slice_bits=8))
    eng.load_basis(0)
    with pytest.raises(q.CapacityError):
        eng.gather(guard_qubits=10)


def test_cpp_api_smoke():
    """The reference's C++ API surface end to end on the GPU."""
    import subprocess
    from paper_1811_05630_b200 import build as b
    out = subprocess.run([b.API_SMOKE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "api_smoke ok" in out.stdout


def test_compare_against_dense_run(q):
    """On-device max error / fidelity of a compressed run against the
    compression-off FP64 run of the same circuit."""
    n, s = 16, 12
    acts = q.lower(q.build_qft(n))
    comp = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    dense = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, compression_enabled=False))
    for e in (comp, dense):
        e.load_basis(12345)
        e.run(acts)
    r = comp.compare(dense)
    ref = comp.amplitudes() - dense.amplitudes()
    assert r["max_abs_diff"] == pytest.approx(np.max(np.abs(ref)), rel=1e-12)
    assert r["fidelity"] > 0.999 and r["max_abs_diff"] < 1e-3
    assert r["norm_b"] == pytest.approx(1.0, abs=1e-9)
    same = comp.compare(comp)
    assert same["max_abs_diff"] == 0.0
    assert same["fidelity"] == pytest.approx(same["norm_a"] ** 2, rel=1e-12)
    twin = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    twin.load_basis(12345)
    twin.run(acts)
    assert comp.compare(twin)["max_abs_diff"] == 0.0  # deterministic, bit-identical


_VARIANT_SCRIPT = r"""
import hashlib, sys
import paper_1811_05630_b200 as q
n, s = 14, 8  # 128 planes: per-plane hand-offs active by default
acts = q.lower(q.build_qft(n))
eng = q.Engine(q.EngineConfig(num_qubits=n, slice_bits=s, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
eng.load_basis(1234)
m = eng.run(acts + acts[:40])
blob = eng.export_blocks()[0]
print(hashlib.sha256(bytes(blob)).hexdigest(), repr(m.mean_compression_ratio), repr(m.min_compression_ratio))
"""


@pytest.mark.parametrize("env", [{"QCSIM_CHAIN": "2"}, {"QCSIM_SYNC_GATES": "1"}, {"QCSIM_PDL": "0"},
                                 {"QCSIM_CHAIN_OVERLAP": "0"}, {"QCSIM_FIXED_SLOTS": "0"}, {"QCSIM_FINE_DECODE": "0"}])
def test_pipeline_variants_bit_identical(env):
    """The serial warp chain, the host-synchronous gate loop, plain launches,
    grid-wide waits instead of per-plane hand-offs and the packed (scanned)
    slot layout, and decoding from the stored slot records only (instead of
    the previous pass's fine checkpoints) produce the same blocks and metrics as the default pipeline
    (block-parallel chain, deferred loop, programmatic dependent launch,
    per-plane hand-offs, fixed slots)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(extra):
        e = dict(os.environ)
        for k in ("QCSIM_CHAIN", "QCSIM_SYNC_GATES", "QCSIM_PDL", "QCSIM_CHAIN_OVERLAP", "QCSIM_FIXED_SLOTS",
                  "QCSIM_FINE_DECODE"):
            e.pop(k, None)
        e.update(extra)
        r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT], cwd=root, env=e, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        return r.stdout.strip().splitlines()[-1]

    assert run(env) == run({})


def test_deferred_drift_error_unloads(q):
    """A norm-drift error latched by the deferred loop leaves the engine
    without a state (it must be reloaded)."""
    eng = q.Engine(q.EngineConfig(num_qubits=6, slice_bits=3, codec=q.CodecConfig(q.CodecMode.Absolute, 1e-5)))
    amps = np.zeros(2 << 6)
    amps[0] = 2.0
    eng.load_amplitudes(amps)
    with pytest.raises(q.NumericError):
        eng.run(q.lower(q.build_qft(6)))
    with pytest.raises((q.NumericError, ValueError)):
        eng.run(q.lower(q.build_qft(6)))
    eng.load_basis(0)
    eng.run(q.lower(q.build_qft(6)))
