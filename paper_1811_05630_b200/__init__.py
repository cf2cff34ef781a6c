"""qcsim-b200: B200-native compressed state-vector update path of
arXiv:1811.05630 (per gate, per slice: decompress -> normalize -> apply gate
-> recompress with the QCB1 error-bounded codec).

The compute path is libqcsim_b200.so (hand-written sm_100a CUDA behind the
C-ABI in include/qcsim_c.h).  This package mirrors the reference API of
proj/include/qcsim/ (codec.hpp, circuit.hpp, the SPEC engine) for Python
callers, tests and bench.py.
"""
from .circuit import (Amplitude, ButterflyOp, Circuit, DiagonalOp, Gate, GateKind, Mat2, SwapOp,  # noqa: F401
                      build_grover, build_grover_oracle, build_qft, gate_action, grover_optimal_iterations,
                      lower, random_u3_circuit_actions, seeded_index, to_action_c, u3_matrix, unitary2,
                      validate_circuit)
from .codec import (CodecConfig, CodecMode, CodecStats, CompressedBlock, Predictor, compress_plane,  # noqa: F401
                    compress_plane_bytes, compression_ratio, decompress_bytes, decompress_plane)
from .engine import (Engine, EngineConfig, RunMetrics, device_memory, kernel_launches,  # noqa: F401
                     measure_overhead)
from .errors import CapacityError, CodecError, CudaError, NumericError, ParseError, QcsimError  # noqa: F401

__version__ = "0.1.0"
