"""The oracle restatement is pinned to the reference (CPU, no GPU).

Fixtures in tests/golden/codec_golden.json were produced by the reference's
own codec (oracle/make_golden.py -> oracle/_ref).  These tests need neither
/root/reference nor a GPU.
"""
import numpy as np
import pytest

from oracle import planes
from oracle.oracle import Action, CodecConfig, EngineConfig, OracleError


def _cfg(c):
    return CodecConfig.make(c["mode"], c["bound"], c["qb"], c["pred"])


def test_kat_a4(oracle, golden):
    """the 82-byte worked block."""
    blk = oracle.compress(np.array([0, 0, 0, 0, 0, 0, 6e-5, 1.0]), CodecConfig.make(1, 1e-5, 16, 0))
    assert blk.data.hex() == golden["kat_a4"]["block_hex"]
    assert len(blk.data) == 82
    assert blk.data[-18:-16].hex() == "72c0"
    dec = oracle.decompress(blk.data)
    assert dec.tolist() == [0, 0, 0, 0, 0, 0, 6.000000000000001e-05, 1.0]
    assert blk.stats.ratio == pytest.approx(64 / 82)


def test_codec_golden_all(oracle, golden):
    bad = []
    for c in golden["codec"]:
        x = planes.make_plane(c["kind"], c["n"], c["seed"])
        assert planes.sha(x) == c["input_sha"], f"plane generator drift: {c['kind']}/{c['n']}/{c['seed']}"
        blk = oracle.compress(x, _cfg(c))
        dec = oracle.decompress(blk.data)
        if (planes.sha(blk.data) != c["block_sha"] or planes.sha(dec) != c["decoded_sha"]
                or blk.stats.ratio != c["ratio"]):
            bad.append((c["config"], c["kind"], c["n"]))
        if "block_hex" in c:
            assert blk.data.hex() == c["block_hex"]
    assert not bad, bad[:10]


def test_decoder_fuzz_verdicts(oracle, golden):
    for f in golden["fuzz"]:
        b = bytes.fromhex(f["block_hex"])
        if f["ok"]:
            dec = oracle.decompress(b)
            assert planes.sha(dec) == f["decoded_sha"], f["source"]
        else:
            with pytest.raises(OracleError) as ei:
                oracle.decompress(b)
            assert ei.value.status == f["status"] and ei.value.msg == f["message"], (f["source"], f["op"])


def _actions(rows):
    out = []
    for kind, target, a, b, mask, factor, u in rows:
        act = Action()
        act.kind, act.target, act.a, act.b, act.mask = kind, target, a, b, mask
        act.factor[0], act.factor[1] = factor
        for i in range(8):
            act.u[i] = u[i]
        out.append(act)
    return out


@pytest.mark.parametrize("idx", range(7))
def test_engine_golden(oracle, golden, idx):
    """Oracle engine == reference codec under the pinned engine semantics."""
    e = golden["engine"][idx]
    acts = _actions(e["actions"])
    assert len(acts) == e["gates"]
    cfg = EngineConfig.make(e["n"], e["s"], CodecConfig.make(1, e["eb"], 16, 0), True, e["norm_every"])
    eng = oracle.engine(cfg)
    eng.load_basis(e["basis"])
    prefix = dict((k, h) for k, h in e["prefix_sha"])
    for k, a in enumerate(acts):
        eng.run([a])
        if k + 1 in prefix:
            assert planes.sha(eng.export_blocks()[0]) == prefix[k + 1], f"{e['name']} after gate {k+1}"
    m = eng.run([])
    assert planes.sha(eng.export_blocks()[0]) == e["final_sha"]
    assert m.min_compression_ratio == e["min_ratio"]
    assert m.final_norm == e["final_norm"]
    assert m.compress_calls == e["calls"]


def test_oracle_matches_reference_random(oracle, reflib):
    """Direct cross-check against the compiled reference on fresh seeds
    (only where oracle/_ref exists, i.e. in the build container)."""
    rng = np.random.default_rng(7)
    for t in range(60):
        kind = planes.KINDS[t % len(planes.KINDS)]
        n = int(rng.choice([1, 2, 3, 5, 100, 333, 4096]))
        x = planes.make_plane(kind, max(n, 1), 90000 + t)
        cfg = CodecConfig.make(int(rng.integers(0, 3)), float(rng.choice([1e-2, 1e-5, 2.0**-9])),
                               int(rng.integers(4, 25)), int(rng.integers(0, 2)))
        a = oracle.compress(x, cfg)
        b = reflib.compress(x, cfg)
        assert a.data == b.data
        assert oracle.decompress(a.data).tobytes() == reflib.decompress(b.data).tobytes()


def test_lowering_matches_reference(oracle, reflib):
    import math
    cases = [(0, [3]), (1, [0]), (2, [5]), (3, [1]), (4, [2]), (5, [7]), (6, [4]), (7, [1, 6]), (8, [2, 0]),
             (9, [0, 3]), (10, [1, 9]), (11, [0, 2, 5])]
    for kind, qs in cases:
        for theta in (0.0, 0.3, -2.0 * math.pi / 3):
            a = oracle.gate_action(kind, qs, theta)
            b = reflib.gate_action(kind, qs, theta)
            assert bytes(a) == bytes(b), (kind, qs, theta)


def test_python_lowering_matches_reference(oracle, reflib):
    """The Python mirror's gate_action / to_action_c (paper_1811_05630_b200/
    circuit.py) produces the same flattened actions as the compiled reference
    (circuit.cpp:392-427) and the C restatement, byte for byte -- including
    the Phase / CPhase factors from libm's cos / sin."""
    import math
    from paper_1811_05630_b200 import circuit as pc
    cases = [(0, [3]), (1, [0]), (2, [5]), (3, [1]), (4, [2]), (5, [7]), (6, [4]), (7, [1, 6]), (8, [2, 0]),
             (9, [0, 3]), (10, [1, 9]), (11, [0, 2, 5])]
    for kind, qs in cases:
        for theta in (0.0, 0.3, -2.0 * math.pi / 3, 2.0 * math.pi / (1 << 20)):
            mine = bytes(pc.to_action_c(pc.gate_action(pc.Gate(pc.GateKind(kind), theta, list(qs)))))
            assert mine == bytes(reflib.gate_action(kind, qs, theta)), (kind, qs, theta)
            assert mine == bytes(oracle.gate_action(kind, qs, theta)), (kind, qs, theta)
    # the QFT / Grover builders emit the reference's gate lists (circuit.cpp:88-168)
    for n in (5, 12):
        ref = reflib.circuit("qft", n, 1)
        assert [bytes(a) for a in pc.lower(pc.build_qft(n))] == [bytes(a) for a in ref]
    ref = reflib.circuit("grover", 6, 37, 3)
    assert [bytes(a) for a in pc.lower(pc.build_grover(6, 37, 3))] == [bytes(a) for a in ref]


def test_codec_errors(oracle):
    with pytest.raises(OracleError, match="cannot compress an empty plane"):
        oracle.compress(np.zeros(0), CodecConfig.make())
    with pytest.raises(OracleError, match="non-finite"):
        oracle.compress(np.array([1.0, np.nan]), CodecConfig.make())
    with pytest.raises(OracleError, match="quant_code_bits"):
        oracle.compress(np.ones(4), CodecConfig.make(qb=3))
    with pytest.raises(OracleError, match="error bound must be positive"):
        oracle.compress(np.ones(4), CodecConfig.make(bound=0.0))
    with pytest.raises(OracleError, match="must not exceed 1"):
        oracle.compress(np.ones(4), CodecConfig.make(mode=0, bound=2.0))


def test_edge_behaviours(oracle):
    """SURVEY.md Appendix A.5."""
    cfg = CodecConfig.make(1, 1e-5, 16, 0)
    d = oracle.decompress(oracle.compress(np.array([1e-5]), cfg).data)
    assert d[0] == 2e-5
    d = oracle.decompress(oracle.compress(np.array([-0.0, -0.0]), cfg).data)
    assert not np.signbit(d).any()
    ll = CodecConfig.make(2, 0.0, 16, 0)
    d = oracle.decompress(oracle.compress(np.array([-0.0, -0.0, 1.5, 1.5]), ll).data)
    assert d.tobytes() == np.array([-0.0, -0.0, 1.5, 1.5]).tobytes()


def test_dense_reference_qft_closed_form(oracle):
    """QFT|k> equals the DFT column (qubit 0 = LSB, with the
    final reversal swaps)."""
    import math
    n = 6
    gates = oracle.build_qft(n)
    acts = [oracle.gate_action(k, qs, th) for k, th, qs in gates]
    N = 1 << n
    for k in (0, 1, 5, 37):
        amps = np.zeros(2 * N)
        amps[2 * k] = 1.0
        out = oracle.ref_run(n, amps, acts)
        z = out[0::2] + 1j * out[1::2]
        want = np.array([np.exp(2j * math.pi * k * j / N) for j in range(N)]) / math.sqrt(N)
        assert np.max(np.abs(z - want)) < 1e-10


def test_lossless_engine_matches_dense(oracle):
    """SPEC.md:329 / acceptance 1: compression off + norm off == ref_run."""
    n = 8
    gates = oracle.build_qft(n)
    acts = [oracle.gate_action(k, qs, th) for k, th, qs in gates]
    for s in (4, 8, 2):
        eng = oracle.engine(EngineConfig.make(n, s, compression=False, norm_every=0))
        eng.load_basis(77)
        eng.run(acts)
        amps = np.zeros(2 << n)
        amps[2 * 77] = 1.0
        ref = oracle.ref_run(n, amps, acts)
        assert np.max(np.abs(eng.gather() - ref)) <= 1e-12


def test_tree_norm_shape(oracle):
    v = np.random.default_rng(1).standard_normal(1 << 10)
    z = np.zeros_like(v)
    # S(lo,len) = S(lo,len/2) + S(lo+len/2,len/2)
    def tree(a):
        return a[0] if a.size == 1 else tree(a[: a.size // 2]) + tree(a[a.size // 2:])
    assert oracle.tree_sq_norm(v, z) == tree(v * v)
    assert oracle.tree_sum(v) == tree(v)
