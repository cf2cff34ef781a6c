"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, the C restatement (qcsim_oracle.c).
* ``RefLib``  -> oracle/_ref/libqcsim_ref.so, the reference's own TUs compiled
  unmodified (oracle/Makefile) + ref_glue.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqcsim_ref.so")

MODE_RANGE_RELATIVE, MODE_ABSOLUTE, MODE_LOSSLESS = 0, 1, 2
PRED_PREVIOUS, PRED_LINEAR = 0, 1
ACTION_DIAGONAL, ACTION_BUTTERFLY, ACTION_SWAP = 0, 1, 2
# GateKind order, circuit.hpp:36-49
H, X, Y, Z, S, T, PHASE, CPHASE, CNOT, CZ, SWAP, MCZ = range(12)

STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "CODEC", 3: "CAPACITY", 4: "PARSE",
                5: "NUMERIC", 6: "CUDA", 7: "NOMEM", 8: "RUNTIME"}


class CodecConfig(C.Structure):
    _fields_ = [("mode", C.c_uint8), ("predictor", C.c_uint8), ("reserved", C.c_uint16),
                ("quant_code_bits", C.c_int32), ("bound", C.c_double)]

    @classmethod
    def make(cls, mode=MODE_ABSOLUTE, bound=1e-5, qb=16, pred=PRED_PREVIOUS):
        return cls(mode, pred, 0, qb, bound)


class CodecStats(C.Structure):
    _fields_ = [("input_bytes", C.c_uint64), ("output_bytes", C.c_uint64),
                ("ratio", C.c_double), ("outlier_fraction", C.c_double)]


class Action(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("target", C.c_int32), ("a", C.c_int32), ("b", C.c_int32),
                ("reserved", C.c_uint32), ("mask", C.c_uint64), ("factor", C.c_double * 2),
                ("u", C.c_double * 8)]


class EngineConfig(C.Structure):
    _fields_ = [("num_qubits", C.c_int32), ("slice_bits", C.c_int32), ("codec", CodecConfig),
                ("compression_enabled", C.c_int32), ("norm_every", C.c_int32),
                ("norm_drift_tolerance", C.c_double), ("device", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("checkpoint_bits", C.c_int32), ("wave_bytes", C.c_uint64)]

    @classmethod
    def make(cls, n, s, codec=None, compression=True, norm_every=1, tol=0.02, device=0,
             rank=0, world=1, checkpoint_bits=0, wave_bytes=0):
        return cls(n, s, codec or CodecConfig.make(), int(compression), norm_every, tol, device,
                   rank, world, checkpoint_bits, wave_bytes)


class RunMetrics(C.Structure):
    _fields_ = [("min_compression_ratio", C.c_double), ("mean_compression_ratio", C.c_double),
                ("wall_seconds", C.c_double), ("final_norm", C.c_double),
                ("compress_calls", C.c_uint64), ("gates", C.c_uint64),
                ("peak_compressed_bytes", C.c_uint64), ("dense_bytes", C.c_uint64),
                ("current_compressed_bytes", C.c_uint64), ("index_bytes", C.c_uint64),
                ("fallback_planes", C.c_uint64), ("kernel_launches", C.c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def actions_array(actions):
    arr = (Action * max(1, len(actions)))()
    for i, a in enumerate(actions):
        # accept any struct with the qcsim_action layout (e.g. the product's)
        arr[i] = a if isinstance(a, Action) else Action.from_buffer_copy(bytes(a))
    return arr


@dataclass
class Block:
    data: bytes
    stats: CodecStats


def partner_slice(a, s, j):
    """the other slice whose old values slice j needs."""
    if a.kind == ACTION_BUTTERFLY and a.target >= s:
        return j ^ (1 << (a.target - s))
    if a.kind == ACTION_SWAP:
        hm = (1 << (a.a - s) if a.a >= s else 0) | (1 << (a.b - s) if a.b >= s else 0)
        return j ^ hm
    return j


class Oracle:
    """The C restatement."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -f oracle/Makefile`")
        L = self.lib = C.CDLL(path)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_block_bound.restype = C.c_uint64
        L.oracle_block_bound.argtypes = [C.c_uint64, C.c_int32]
        L.oracle_compress_plane.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(CodecConfig),
                                            C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint64),
                                            C.POINTER(CodecStats)]
        L.oracle_decompress_plane.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_double),
                                              C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_gate_action.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_int32), C.c_int,
                                         C.POINTER(Action)]
        L.oracle_ref_run.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(Action), C.c_uint64, C.c_int]
        L.oracle_tree_sum.restype = C.c_double
        L.oracle_tree_sum.argtypes = [C.POINTER(C.c_double), C.c_uint64]
        L.oracle_tree_sq_norm.restype = C.c_double
        L.oracle_tree_sq_norm.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint64]
        L.oracle_planes_sq_norm.restype = C.c_double
        L.oracle_planes_sq_norm.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint64]
        L.oracle_engine_create.argtypes = [C.POINTER(EngineConfig), C.POINTER(C.c_void_p)]
        L.oracle_engine_destroy.argtypes = [C.c_void_p]
        L.oracle_engine_load_basis.argtypes = [C.c_void_p, C.c_uint64]
        L.oracle_engine_load_amplitudes.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint64]
        L.oracle_engine_run.argtypes = [C.c_void_p, C.POINTER(Action), C.c_uint64, C.POINTER(RunMetrics)]
        L.oracle_engine_gather.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint64]
        L.oracle_engine_slice_norms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint64]
        L.oracle_engine_export_blocks.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.c_uint64,
                                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_uint64]
        L.oracle_engine_export_slice.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8), C.c_uint64,
                                                 C.POINTER(C.c_uint64)]
        L.oracle_engine_import_partner.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8), C.c_uint64]
        L.oracle_engine_set_global_norms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint64]
        L.oracle_build_qft.restype = C.c_int64
        L.oracle_build_qft.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.oracle_grover_optimal_iterations.argtypes = [C.c_int]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.oracle_last_error().decode())

    # codec -------------------------------------------------------------
    def compress(self, values, cfg) -> Block:
        v = np.ascontiguousarray(values, dtype=np.float64)
        ln = C.c_uint64()
        st = CodecStats()
        self._check(self.lib.oracle_compress_plane(_dptr(v), v.size, C.byref(cfg), None, 0, C.byref(ln),
                                                   C.byref(st)))
        out = np.empty(ln.value, dtype=np.uint8)
        self._check(self.lib.oracle_compress_plane(_dptr(v), v.size, C.byref(cfg), _u8ptr(out), out.size,
                                                   C.byref(ln), C.byref(st)))
        return Block(out.tobytes(), st)

    def decompress(self, block: bytes):
        b = np.frombuffer(block, dtype=np.uint8).copy()
        n = C.c_uint64()
        cons = C.c_uint64()
        self._check(self.lib.oracle_decompress_plane(_u8ptr(b), b.size, None, 0, C.byref(n), C.byref(cons)))
        out = np.empty(n.value, dtype=np.float64)
        self._check(self.lib.oracle_decompress_plane(_u8ptr(b), b.size, _dptr(out), out.size, C.byref(n),
                                                     C.byref(cons)))
        return out

    # lowering / dense ----------------------------------------------------
    def gate_action(self, kind, qubits, theta=0.0) -> Action:
        qs = (C.c_int32 * len(qubits))(*qubits)
        a = Action()
        self._check(self.lib.oracle_gate_action(kind, theta, qs, len(qubits), C.byref(a)))
        return a

    def ref_run(self, n, amps, actions, guard=24):
        a = np.ascontiguousarray(amps, dtype=np.float64).copy()
        arr = actions_array(actions)
        self._check(self.lib.oracle_ref_run(n, _dptr(a), arr, len(actions), guard))
        return a

    def tree_sq_norm(self, re, im):
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        return self.lib.oracle_tree_sq_norm(_dptr(re), _dptr(im), re.size)

    def tree_sum(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.lib.oracle_tree_sum(_dptr(v), v.size)

    def planes_sq_norm(self, re, im):
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        return self.lib.oracle_planes_sq_norm(_dptr(re), _dptr(im), re.size)

    def build_qft(self, n, swaps=True):
        cnt = self.lib.oracle_build_qft(n, int(swaps), None, None, None, None)
        kind = (C.c_int32 * cnt)()
        theta = (C.c_double * cnt)()
        q0 = (C.c_int32 * cnt)()
        q1 = (C.c_int32 * cnt)()
        self.lib.oracle_build_qft(n, int(swaps), kind, theta, q0, q1)
        gates = []
        for k in range(cnt):
            qs = [q0[k]] if q1[k] < 0 else [q0[k], q1[k]]
            gates.append((kind[k], theta[k], qs))
        return gates

    def engine(self, cfg):
        return OracleEngine(self, cfg)


class OracleEngine:
    def __init__(self, o: Oracle, cfg: EngineConfig):
        self.o = o
        self.cfg = cfg
        h = C.c_void_p()
        o._check(o.lib.oracle_engine_create(C.byref(cfg), C.byref(h)))
        self.h = h
        n = cfg.num_qubits
        self.n = n
        self.s = cfg.slice_bits if cfg.slice_bits >= 0 else min(n, 20)
        self.world = max(1, cfg.world)
        self.local_slices = (1 << (n - self.s)) // self.world

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.oracle_engine_destroy(self.h)
            self.h = None

    def load_basis(self, x):
        self.o._check(self.o.lib.oracle_engine_load_basis(self.h, x))

    def load_amplitudes(self, amps):
        a = np.ascontiguousarray(amps, dtype=np.float64)
        self.o._check(self.o.lib.oracle_engine_load_amplitudes(self.h, _dptr(a), a.size // 2))

    def run(self, actions):
        arr = actions_array(actions)
        m = RunMetrics()
        self.o._check(self.o.lib.oracle_engine_run(self.h, arr, len(actions), C.byref(m)))
        return m

    def gather(self):
        out = np.empty(2 << self.n, dtype=np.float64)
        self.o._check(self.o.lib.oracle_engine_gather(self.h, _dptr(out), out.size))
        return out

    def slice_norms(self):
        out = np.empty(self.local_slices, dtype=np.float64)
        self.o._check(self.o.lib.oracle_engine_slice_norms(self.h, _dptr(out), out.size))
        return out

    def metrics(self):
        return self.run([])

    # ---- multi-rank hooks (same surface as paper_1811_05630_b200.Engine)
    def partner_slices_needed(self, action):
        s0 = self.cfg.rank * self.local_slices
        out = []
        for j in range(s0, s0 + self.local_slices):
            pj = partner_slice(action, self.s, j)
            if not (s0 <= pj < s0 + self.local_slices):
                out.append(pj)
        return out

    def export_slice(self, j):
        ln = C.c_uint64()
        self.o._check(self.o.lib.oracle_engine_export_slice(self.h, j, None, 0, C.byref(ln)))
        out = np.empty(ln.value, dtype=np.uint8)
        self.o._check(self.o.lib.oracle_engine_export_slice(self.h, j, _u8ptr(out), out.size, C.byref(ln)))
        return out.tobytes()

    def import_partner(self, j, data):
        b = np.frombuffer(data, dtype=np.uint8).copy()
        self.o._check(self.o.lib.oracle_engine_import_partner(self.h, j, _u8ptr(b), b.size))

    def set_global_norms(self, norms):
        v = np.ascontiguousarray(norms, dtype=np.float64)
        self.o._check(self.o.lib.oracle_engine_set_global_norms(self.h, _dptr(v), v.size))

    def export_blocks(self):
        ln = C.c_uint64()
        nplanes = 2 * self.local_slices
        offs = (C.c_uint64 * (nplanes + 1))()
        self.o._check(self.o.lib.oracle_engine_export_blocks(self.h, None, 0, C.byref(ln), offs, nplanes + 1))
        out = np.empty(ln.value, dtype=np.uint8)
        self.o._check(self.o.lib.oracle_engine_export_blocks(self.h, _u8ptr(out), out.size, C.byref(ln),
                                                             offs, nplanes + 1))
        return out.tobytes(), list(offs)


class RefLib:
    """The reference's own codec/statevec/circuit TUs (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_compress_plane.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(CodecConfig),
                                         C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint64),
                                         C.POINTER(CodecStats)]
        L.ref_decompress_plane.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_double),
                                           C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_planes_sq_norm.restype = C.c_double
        L.ref_planes_sq_norm.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint64]
        L.ref_gate_action.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_int32), C.c_int, C.POINTER(Action)]
        L.ref_build_qft.argtypes = [C.c_int, C.c_int, C.POINTER(Action), C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_build_grover.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(Action), C.c_uint64,
                                       C.POINTER(C.c_uint64)]
        L.ref_grover_optimal_iterations.argtypes = [C.c_int]
        L.ref_engine_create.argtypes = [C.POINTER(EngineConfig), C.c_int, C.POINTER(C.c_void_p)]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_load_basis.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_engine_gate.argtypes = [C.c_void_p, C.POINTER(Action), C.c_uint64, C.c_uint64]
        L.ref_engine_export_blocks.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.c_uint64,
                                               C.POINTER(C.c_uint64)]
        L.ref_engine_metrics.argtypes = [C.c_void_p, C.POINTER(RunMetrics)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def compress(self, values, cfg) -> Block:
        v = np.ascontiguousarray(values, dtype=np.float64)
        ln = C.c_uint64()
        st = CodecStats()
        self._check(self.lib.ref_compress_plane(_dptr(v), v.size, C.byref(cfg), None, 0, C.byref(ln),
                                                C.byref(st)))
        out = np.empty(ln.value, dtype=np.uint8)
        self._check(self.lib.ref_compress_plane(_dptr(v), v.size, C.byref(cfg), _u8ptr(out), out.size,
                                                C.byref(ln), C.byref(st)))
        return Block(out.tobytes(), st)

    def decompress(self, block: bytes):
        b = np.frombuffer(block, dtype=np.uint8).copy()
        n = C.c_uint64()
        self._check(self.lib.ref_decompress_plane(_u8ptr(b), b.size, None, 0, C.byref(n), None))
        out = np.empty(n.value, dtype=np.float64)
        self._check(self.lib.ref_decompress_plane(_u8ptr(b), b.size, _dptr(out), out.size, C.byref(n), None))
        return out

    def gate_action(self, kind, qubits, theta=0.0) -> Action:
        qs = (C.c_int32 * len(qubits))(*qubits)
        a = Action()
        self._check(self.lib.ref_gate_action(kind, theta, qs, len(qubits), C.byref(a)))
        return a

    def circuit(self, which, *args):
        cnt = C.c_uint64()
        fn = self.lib.ref_build_qft if which == "qft" else self.lib.ref_build_grover
        self._check(fn(*args, None, 0, C.byref(cnt)))
        arr = (Action * cnt.value)()
        self._check(fn(*args, arr, cnt.value, C.byref(cnt)))
        return list(arr)

    def engine(self, cfg, workers=0):
        return RefEngine(self, cfg, workers)


class RefEngine:
    def __init__(self, r: RefLib, cfg: EngineConfig, workers=0):
        self.r = r
        h = C.c_void_p()
        r._check(r.lib.ref_engine_create(C.byref(cfg), workers, C.byref(h)))
        self.h = h
        self.n = cfg.num_qubits
        self.s = cfg.slice_bits if cfg.slice_bits >= 0 else min(self.n, 20)

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_engine_destroy(self.h)
            self.h = None

    def load_basis(self, x):
        self.r._check(self.r.lib.ref_engine_load_basis(self.h, x))

    def gate(self, action, first=0, count=None):
        if count is None:
            count = 1 << (self.n - self.s)
        self.r._check(self.r.lib.ref_engine_gate(self.h, C.byref(action), first, count))

    def run(self, actions):
        for a in actions:
            self.gate(a)

    def export_blocks(self):
        ln = C.c_uint64()
        self.r._check(self.r.lib.ref_engine_export_blocks(self.h, None, 0, C.byref(ln)))
        out = np.empty(ln.value, dtype=np.uint8)
        self.r._check(self.r.lib.ref_engine_export_blocks(self.h, _u8ptr(out), out.size, C.byref(ln)))
        return out.tobytes()

    def metrics(self):
        m = RunMetrics()
        self.r.lib.ref_engine_metrics(self.h, C.byref(m))
        return m
