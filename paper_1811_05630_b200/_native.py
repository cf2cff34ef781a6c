"""ctypes binding of libqcsim_b200.so (the C-ABI in include/qcsim_c.h).

The shared library is built in-tree by ``paper_1811_05630_b200.build``.  If it
is missing this module raises at import: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqcsim_b200.so")


class CodecConfigC(C.Structure):
    _fields_ = [("mode", C.c_uint8), ("predictor", C.c_uint8), ("reserved", C.c_uint16),
                ("quant_code_bits", C.c_int32), ("bound", C.c_double)]


class CodecStatsC(C.Structure):
    _fields_ = [("input_bytes", C.c_uint64), ("output_bytes", C.c_uint64),
                ("ratio", C.c_double), ("outlier_fraction", C.c_double)]


class ActionC(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("target", C.c_int32), ("a", C.c_int32), ("b", C.c_int32),
                ("reserved", C.c_uint32), ("mask", C.c_uint64), ("factor", C.c_double * 2),
                ("u", C.c_double * 8)]


class EngineConfigC(C.Structure):
    _fields_ = [("num_qubits", C.c_int32), ("slice_bits", C.c_int32), ("codec", CodecConfigC),
                ("compression_enabled", C.c_int32), ("norm_every", C.c_int32),
                ("norm_drift_tolerance", C.c_double), ("device", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("checkpoint_bits", C.c_int32), ("wave_bytes", C.c_uint64)]


class CompareC(C.Structure):
    _fields_ = [("max_abs_diff", C.c_double), ("inner_re", C.c_double), ("inner_im", C.c_double),
                ("norm_a", C.c_double), ("norm_b", C.c_double), ("fidelity", C.c_double)]


class RunMetricsC(C.Structure):
    _fields_ = [("min_compression_ratio", C.c_double), ("mean_compression_ratio", C.c_double),
                ("wall_seconds", C.c_double), ("final_norm", C.c_double),
                ("compress_calls", C.c_uint64), ("gates", C.c_uint64),
                ("peak_compressed_bytes", C.c_uint64), ("dense_bytes", C.c_uint64),
                ("current_compressed_bytes", C.c_uint64), ("index_bytes", C.c_uint64),
                ("fallback_planes", C.c_uint64), ("kernel_launches", C.c_uint64)]


class GateMetricsC(C.Structure):
    _fields_ = [("min_ratio", C.c_double), ("mean_ratio", C.c_double), ("seconds", C.c_double),
                ("compressed_bytes", C.c_uint64), ("index_bytes", C.c_uint64), ("compress_calls", C.c_uint64)]


class EngineInfoC(C.Structure):
    _fields_ = [("local_slices", C.c_uint64), ("wave_slices", C.c_uint64), ("waves", C.c_uint64),
                ("checkpoint_bits", C.c_int32), ("reserved", C.c_int32)]


P = C.POINTER
u8p, dp, u64p = P(C.c_uint8), P(C.c_double), P(C.c_uint64)

# (name, restype, argtypes) -- every symbol include/qcsim_c.h declares
SIGNATURES = [
    ("qcsim_last_error", C.c_char_p, []),
    ("qcsim_version", C.c_char_p, []),
    ("qcsim_codec_validate", C.c_int, [P(CodecConfigC)]),
    ("qcsim_block_bound", C.c_uint64, [C.c_uint64, C.c_int32]),
    ("qcsim_compress_plane", C.c_int, [dp, C.c_uint64, P(CodecConfigC), u8p, C.c_uint64, u64p, P(CodecStatsC)]),
    ("qcsim_decompress_plane", C.c_int, [u8p, C.c_uint64, dp, C.c_uint64, u64p, u64p]),
    ("qcsim_compress_planes_device", C.c_int, [P(C.c_void_p), u64p, C.c_uint32, P(CodecConfigC), C.c_void_p,
                                               C.c_uint64, u64p, P(CodecStatsC), C.c_void_p]),
    ("qcsim_decompress_planes_device", C.c_int, [C.c_void_p, u64p, C.c_uint32, P(C.c_void_p), u64p,
                                                 C.c_void_p]),
    ("qcsim_engine_create", C.c_int, [P(EngineConfigC), P(C.c_void_p)]),
    ("qcsim_engine_destroy", C.c_int, [C.c_void_p]),
    ("qcsim_engine_load_basis", C.c_int, [C.c_void_p, C.c_uint64]),
    ("qcsim_engine_load_amplitudes", C.c_int, [C.c_void_p, dp, C.c_uint64]),
    ("qcsim_engine_load_blocks", C.c_int, [C.c_void_p, u8p, C.c_uint64, u64p, C.c_uint64, dp, C.c_uint64, C.c_uint64]),
    ("qcsim_engine_run", C.c_int, [C.c_void_p, P(ActionC), C.c_uint64, P(RunMetricsC)]),
    ("qcsim_engine_gather", C.c_int, [C.c_void_p, dp, C.c_uint64, C.c_int32]),
    ("qcsim_engine_slice_norms", C.c_int, [C.c_void_p, dp, C.c_uint64]),
    ("qcsim_engine_compare", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("qcsim_engine_export_blocks", C.c_int, [C.c_void_p, u8p, C.c_uint64, u64p, u64p, C.c_uint64]),
    ("qcsim_engine_partner_blocks_needed", C.c_int, [C.c_void_p, P(ActionC), u64p, C.c_uint64, u64p]),
    ("qcsim_engine_export_slice", C.c_int, [C.c_void_p, C.c_uint64, u8p, C.c_uint64, u64p]),
    ("qcsim_engine_import_partner", C.c_int, [C.c_void_p, C.c_uint64, u8p, C.c_uint64]),
    ("qcsim_engine_export_slices", C.c_int, [C.c_void_p, u64p, C.c_uint64, u8p, C.c_uint64, u64p, u64p]),
    ("qcsim_engine_export_slices_device", C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_void_p, C.c_uint64, u64p,
                                                    u64p]),
    ("qcsim_engine_import_partners_device", C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_void_p, u64p]),
    ("qcsim_engine_set_global_norms", C.c_int, [C.c_void_p, dp, C.c_uint64]),
    ("qcsim_engine_gate_metrics", C.c_int, [C.c_void_p, P(GateMetricsC), C.c_uint64, u64p]),
    ("qcsim_engine_info", C.c_int, [C.c_void_p, P(EngineInfoC)]),
    ("qcsim_device_memory", C.c_int, [u64p, u64p, C.c_int32]),
    ("qcsim_engine_trim", C.c_int, [C.c_void_p]),
]
EXTRA = [("qcsim_kernel_launches", C.c_uint64, [])]

_lib = None


def lib():
    """Load the CUDA library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (qcsim-b200 has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES + EXTRA:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
