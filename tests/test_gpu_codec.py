"""GPU codec parity: QCB1 streams and decoded values bit-exact vs the
reference (golden fixtures made by the reference's own codec) and the
oracle, through the C-ABI (libqcsim_b200.so)."""
import numpy as np
import pytest

from oracle import planes
from oracle.oracle import CodecConfig as OCfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1811_05630_b200 as q
    return q


def _cfg(q, c):
    return q.CodecConfig(q.CodecMode(c["mode"]), c["bound"], c["qb"], q.Predictor(c["pred"]))


def test_kat_a4(q, golden):
    blk, st = q.compress_plane(np.array([0, 0, 0, 0, 0, 0, 6e-5, 1.0]), q.CodecConfig(q.CodecMode.Absolute, 1e-5))
    assert blk.to_bytes().hex() == golden["kat_a4"]["block_hex"]
    assert st.ratio == golden["kat_a4"]["ratio"]
    d = q.decompress_plane(blk)
    assert d.tolist() == [0, 0, 0, 0, 0, 0, 6.000000000000001e-05, 1.0]


def test_golden_all(q, golden):
    """Every reference-generated case: stream bytes, decoded bytes, ratio."""
    bad = []
    for c in golden["codec"]:
        x = planes.make_plane(c["kind"], c["n"], c["seed"])
        assert planes.sha(x) == c["input_sha"]
        blk, st = q.compress_plane(x, _cfg(q, c))
        data = blk.to_bytes()
        dec = q.decompress_plane(blk)
        if planes.sha(data) != c["block_sha"] or planes.sha(dec) != c["decoded_sha"] or st.ratio != c["ratio"]:
            bad.append((c["config"], c["kind"], c["n"]))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:8]}"


def test_fuzz_verdicts(q, golden):
    """Corrupt blocks: same error message (or same decode) as the reference."""
    for f in golden["fuzz"]:
        b = bytes.fromhex(f["block_hex"])
        if f["ok"]:
            assert planes.sha(q.decompress_bytes(b)) == f["decoded_sha"], f["source"]
        else:
            exc = q.CodecError if f["status"] == 2 else ValueError
            with pytest.raises(exc) as ei:
                q.decompress_bytes(b)
            assert str(ei.value) == f["message"], (f["source"], f["op"])


@pytest.mark.parametrize("kind", ["qft", "gauss", "walk", "outliers", "grover", "basis", "uniform", "smooth"])
@pytest.mark.parametrize("n", [1 << 16, (1 << 20)])
def test_large_planes_vs_oracle(q, oracle, kind, n):
    """Full plane sizes of configs 3/4 (2^20) and beyond the fixtures."""
    x = planes.make_plane(kind, n, 4321 + n % 97)
    for eb in (1e-3, 1e-5, 1e-7):
        cfg = q.CodecConfig(q.CodecMode.Absolute, eb)
        blk, st = q.compress_plane(x, cfg)
        ref = oracle.compress(x, OCfg.make(1, eb, 16, 0))
        assert blk.to_bytes() == ref.data, (kind, n, eb)
        dec = q.decompress_plane(blk)
        assert dec.tobytes() == oracle.decompress(ref.data).tobytes()
        assert np.max(np.abs(dec - x)) <= eb  # error-bound soundness (SPEC acceptance 2)


def test_edge_cases(q, oracle):
    cases = [np.array([1e-5]), np.array([-0.0, -0.0, 0.0]), np.array([1.0]), np.zeros(5), np.zeros(1025),
             np.array([1e300, -1e300, 5.0]), np.full(3000, 2.0**-10), np.arange(10000) * 2e-5]
    for mode, bound, qb, pred in [(1, 1e-5, 16, 0), (2, 0.0, 16, 0), (0, 1e-2, 8, 0), (1, 2.0**-11, 4, 0),
                                  (1, 1e-5, 16, 1), (0, 0.5, 24, 1)]:
        for x in cases:
            cfg = q.CodecConfig(q.CodecMode(mode), bound, qb, q.Predictor(pred))
            blk, _ = q.compress_plane(x, cfg)
            ref = oracle.compress(x, OCfg.make(mode, bound, qb, pred))
            assert blk.to_bytes() == ref.data, (mode, bound, qb, pred, x[:4])
            assert q.decompress_plane(blk).tobytes() == oracle.decompress(ref.data).tobytes()


def test_errors(q):
    with pytest.raises(ValueError, match="cannot compress an empty plane"):
        q.compress_plane(np.zeros(0), q.CodecConfig())
    with pytest.raises(ValueError, match="non-finite"):
        q.compress_plane(np.array([0.0, np.inf]), q.CodecConfig())
    with pytest.raises(ValueError, match="quant_code_bits"):
        q.compress_plane(np.ones(3), q.CodecConfig(quant_code_bits=25))


def test_random_property(q, oracle):
    """Seeded random planes / configs (SPEC acceptance 2 style)."""
    rng = np.random.default_rng(11)
    for t in range(40):
        kind = planes.KINDS[t % len(planes.KINDS)]
        n = int(rng.choice([7, 100, 1023, 1024, 1025, 5000, 40000]))
        x = planes.make_plane(kind, n, 777 + t)
        mode = int(rng.integers(0, 3))
        bound = float(rng.choice([1e-1, 1e-2, 1e-4, 1e-6, 2.0**-9]))
        qb = int(rng.choice([4, 8, 12, 16]))
        pred = int(rng.integers(0, 2))
        blk, _ = q.compress_plane(x, q.CodecConfig(q.CodecMode(mode), bound, qb, q.Predictor(pred)))
        ref = oracle.compress(x, OCfg.make(mode, bound, qb, pred))
        assert blk.to_bytes() == ref.data, (kind, n, mode, bound, qb, pred)
