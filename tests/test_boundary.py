"""The C-ABI boundary (CPU-only checks, no compute): the CUDA library loads
and exports every symbol include/qcsim_c.h declares, the ctypes layouts
match the header, and the product fails loudly without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "qcsim_c.h")).read()
    return sorted(set(re.findall(r"\b(qcsim_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported():
    from paper_1811_05630_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in _native.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_struct_layouts():
    from paper_1811_05630_b200 import _native
    assert ctypes.sizeof(_native.CodecConfigC) == 16
    assert ctypes.sizeof(_native.ActionC) == 24 + 8 + 16 + 64
    assert ctypes.sizeof(_native.RunMetricsC) == 4 * 8 + 8 * 8
    from oracle import oracle as o
    for a, b in [(_native.CodecConfigC, o.CodecConfig), (_native.ActionC, o.Action),
                 (_native.EngineConfigC, o.EngineConfig), (_native.RunMetricsC, o.RunMetrics)]:
        assert ctypes.sizeof(a) == ctypes.sizeof(b)


def test_version_and_no_cpu_fallback():
    import torch
    from paper_1811_05630_b200 import _native
    lib = _native.lib()
    assert b"sm_100a" in lib.qcsim_version()
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1811_05630_b200 as q
    with pytest.raises(q.CudaError):
        q.compress_plane(np.ones(8), q.CodecConfig(q.CodecMode.Absolute, 1e-5))
    with pytest.raises(q.CudaError):
        q.Engine(q.EngineConfig(num_qubits=4, slice_bits=2))


def test_block_bound_is_upper_bound(oracle):
    import numpy as np
    from oracle import planes
    from oracle.oracle import CodecConfig
    from paper_1811_05630_b200 import _native
    lib = _native.lib()
    for kind in ("uniform", "outliers", "negzero"):
        for qb in (4, 16, 24):
            x = planes.make_plane(kind, 3000, 5)
            blk = oracle.compress(x, CodecConfig.make(1, 1e-9, qb, 0))
            assert len(blk.data) <= lib.qcsim_block_bound(3000, qb)


def test_cpp_api_shim_links():
    """The C++ drop-in (include/qcsim/*.hpp -> libqcsim.so -> C-ABI) builds
    and links; the GPU leg runs it (tests/test_gpu_engine.py)."""
    from paper_1811_05630_b200 import build as b
    b.build(verbose=False)
    assert os.path.exists(b.API_LIB) and os.path.exists(b.API_SMOKE)
    lib = ctypes.CDLL(b.API_LIB)
    assert lib is not None
