"""Engine API -- Algorithm 1 as specified by SPEC.md:297-392
(the reference ships no engine source; semantics pinned in DESIGN.md §3).

    eng = Engine(EngineConfig(num_qubits=16, slice_bits=12,
                              codec=CodecConfig(CodecMode.Absolute, 1e-5)))
    eng.load_basis(x)
    metrics = eng.run(build_qft(16))      # gate passes on the GPU
    amps = eng.gather()

Every gate pass runs on the device (libqcsim_b200.so): decode -> normalize
-> gate -> sq_norm -> encode, bit-exact with the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .circuit import Circuit, lower
from .codec import CodecConfig, CodecMode
from .errors import raise_status


@dataclass
class EngineConfig:
    """EngineConfig.  norm_every: 0 off, 1 every gate,
    k every k-th gate.  workers is accepted for API parity; the device
    processes all slices of a pass concurrently."""
    num_qubits: int = 1
    slice_bits: int = -1
    codec: CodecConfig = field(default_factory=lambda: CodecConfig(CodecMode.Absolute, 1e-5))
    compression_enabled: bool = True
    workers: int = 1
    norm_every: int = 1
    norm_drift_tolerance: float = 0.02
    device: int = 0
    rank: int = 0
    world: int = 1
    checkpoint_bits: int = 0
    wave_bytes: int = 0  # dense working-set budget of a gate pass (0 = 45% of the device)

    def to_c(self) -> _native.EngineConfigC:
        return _native.EngineConfigC(self.num_qubits, self.slice_bits, self.codec.to_c(),
                                     int(self.compression_enabled), self.norm_every, self.norm_drift_tolerance,
                                     self.device, self.rank, self.world, self.checkpoint_bits, self.wave_bytes)


@dataclass
class RunMetrics:
    """RunMetrics."""
    min_compression_ratio: float
    mean_compression_ratio: float
    wall_seconds: float
    final_norm: float
    compress_calls: int
    gates: int
    peak_compressed_bytes: int
    dense_bytes: int
    current_compressed_bytes: int
    index_bytes: int
    fallback_planes: int
    kernel_launches: int
    per_gate_min_ratio: list = field(default_factory=list)  # filled by Engine.metrics()/run()
    baseline_wall_seconds: float | None = None             # measure_overhead
    overhead_factor: float | None = None                   # measure_overhead: wall / baseline wall

    @classmethod
    def from_c(cls, m: _native.RunMetricsC):
        return cls(*[getattr(m, f) for f, _ in _native.RunMetricsC._fields_])

    def to_json(self, rows=None) -> dict:
        """Metrics report: every RunMetrics field plus the
        per-gate rows."""
        d = {f: getattr(self, f) for f in self.__dataclass_fields__}
        if rows is not None:
            d["per_gate"] = [dict(gate_index=k - 1, **r) for k, r in enumerate(rows)]
        return d


def _actions(actions):
    if isinstance(actions, C.Array) and actions._type_ is _native.ActionC:
        return actions, len(actions)  # already the C layout: no copy
    if isinstance(actions, Circuit):
        actions = lower(actions)
    arr = (_native.ActionC * max(1, len(actions)))()
    for i, a in enumerate(actions):
        arr[i] = a if isinstance(a, _native.ActionC) else _native.ActionC.from_buffer_copy(bytes(a))
    return arr, len(actions)


class Engine:
    def __init__(self, config: EngineConfig):
        self.L = _native.lib()
        self.config = config
        c = config.to_c()
        h = C.c_void_p()
        raise_status(self.L.qcsim_engine_create(C.byref(c), C.byref(h)), self.L)
        self.h = h
        self.n = config.num_qubits
        self.s = config.slice_bits if config.slice_bits >= 0 else min(self.n, 20)
        self.world = max(1, config.world)
        self.local_slices = (1 << (self.n - self.s)) // self.world

    def close(self):
        if getattr(self, "h", None):
            self.L.qcsim_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _ck(self, rc):
        raise_status(rc, self.L)

    def load_basis(self, x: int):
        self._ck(self.L.qcsim_engine_load_basis(self.h, x))

    def load_amplitudes(self, amps):
        a = np.ascontiguousarray(amps)
        if np.iscomplexobj(a):
            a = a.view(np.float64)
        a = np.ascontiguousarray(a, dtype=np.float64)
        self._ck(self.L.qcsim_engine_load_amplitudes(self.h, a.ctypes.data_as(_native.dp), a.size // 2))

    def load_blocks(self, blocks, offsets, sq_norms, gates_done: int = 0):
        """Resume from a checkpoint: this rank's QCB1 blocks in
        export_blocks order, their offsets, and the global per-slice sq_norm
        table (qcsim_engine_load_blocks)."""
        b = np.frombuffer(bytes(blocks), dtype=np.uint8) if not isinstance(blocks, np.ndarray) else blocks
        b = np.ascontiguousarray(b, dtype=np.uint8)
        offs = (C.c_uint64 * len(offsets))(*offsets)
        v = np.ascontiguousarray(sq_norms, dtype=np.float64)
        self._ck(self.L.qcsim_engine_load_blocks(self.h, b.ctypes.data_as(_native.u8p), b.size, offs,
                                                 len(offsets) - 1, v.ctypes.data_as(_native.dp), v.size, gates_done))

    def run(self, actions=()) -> RunMetrics:
        arr, n = _actions(actions)
        m = _native.RunMetricsC()
        self._ck(self.L.qcsim_engine_run(self.h, arr, n, C.byref(m)))
        return RunMetrics.from_c(m)

    def full_metrics(self) -> RunMetrics:
        """metrics() plus per_gate_min_ratio (one entry per gate pass since
        the load)."""
        m = self.metrics()
        m.per_gate_min_ratio = [r["min_ratio"] for r in self.gate_metrics()[1:]]
        return m

    def write_report(self, json_path=None, csv_path=None, metrics: RunMetrics | None = None) -> dict:
        """JSON with every RunMetrics field plus the per-gate
        rows; CSV of (gate_index, min_ratio, mean_ratio, seconds)."""
        import json
        rows = self.gate_metrics()
        m = metrics or self.full_metrics()
        d = m.to_json(rows)
        if json_path:
            with open(json_path, "w") as f:
                json.dump(d, f, indent=1)
        if csv_path:
            with open(csv_path, "w") as f:
                f.write("gate_index,min_ratio,mean_ratio,seconds\n")
                for k, r in enumerate(rows):
                    f.write(f"{k - 1},{r['min_ratio']!r},{r['mean_ratio']!r},{r['seconds']!r}\n")
        return d

    def metrics(self) -> RunMetrics:
        return self.run(())

    def gather(self, guard_qubits: int = 28) -> np.ndarray:
        """Interleaved (re, im) amplitudes of this rank's slices."""
        out = np.empty(2 * self.local_slices << self.s, dtype=np.float64)
        self._ck(self.L.qcsim_engine_gather(self.h, out.ctypes.data_as(_native.dp), out.size, guard_qubits))
        return out

    def amplitudes(self, guard_qubits: int = 28) -> np.ndarray:
        g = self.gather(guard_qubits)
        return g[0::2] + 1j * g[1::2]

    def compare(self, other: "Engine") -> dict:
        """On-device comparison with another engine's current state (same
        qubits and slicing): max |a - b|, <a|b>, both squared norms and
        fidelity |<a|b>|^2 (statevec.hpp:83-84)."""
        r = _native.CompareC()
        self._ck(self.L.qcsim_engine_compare(self.h, other.h, C.byref(r)))
        return {"max_abs_diff": r.max_abs_diff, "inner": complex(r.inner_re, r.inner_im), "norm_a": r.norm_a,
                "norm_b": r.norm_b, "fidelity": r.fidelity}

    def gate_metrics(self) -> list:
        """Per-pass rows since the last load (row 0: the initial
        compression; row k: after gate k-1): min / mean ratio, device
        seconds, compressed and decode-index bytes."""
        cnt = C.c_uint64()
        self._ck(self.L.qcsim_engine_gate_metrics(self.h, None, 0, C.byref(cnt)))
        buf = (_native.GateMetricsC * max(1, cnt.value))()
        self._ck(self.L.qcsim_engine_gate_metrics(self.h, buf, cnt.value, C.byref(cnt)))
        return [{"min_ratio": r.min_ratio, "mean_ratio": r.mean_ratio, "seconds": r.seconds,
                 "bytes": r.compressed_bytes, "index_bytes": r.index_bytes, "calls": r.compress_calls}
                for r in buf[: cnt.value]]

    def trim(self):
        """Release the gate-pass scratch (the compressed state stays)."""
        self._ck(self.L.qcsim_engine_trim(self.h))

    def info(self) -> dict:
        """Wave layout of a gate pass (qcsim_engine_info)."""
        i = _native.EngineInfoC()
        self._ck(self.L.qcsim_engine_info(self.h, C.byref(i)))
        return {"local_slices": i.local_slices, "wave_slices": i.wave_slices, "waves": i.waves,
                "checkpoint_bits": i.checkpoint_bits}

    def slice_norms(self) -> np.ndarray:
        out = np.empty(self.local_slices, dtype=np.float64)
        self._ck(self.L.qcsim_engine_slice_norms(self.h, out.ctypes.data_as(_native.dp), out.size))
        return out

    def export_blocks(self):
        """QCB1 blocks of this rank's planes (slice-major, re then im) as
        bytes, plus the plane offsets."""
        out, offs = self.export_blocks_array()
        return out.tobytes(), offs

    def export_blocks_array(self):
        """export_blocks without the bytes copy (a uint8 numpy array)."""
        ln = C.c_uint64()
        P = 2 * self.local_slices
        offs = (C.c_uint64 * (P + 1))()
        self._ck(self.L.qcsim_engine_export_blocks(self.h, None, 0, C.byref(ln), offs, P + 1))
        out = np.empty(ln.value, dtype=np.uint8)
        self._ck(self.L.qcsim_engine_export_blocks(self.h, out.ctypes.data_as(_native.u8p), out.size,
                                                   C.byref(ln), offs, P + 1))
        return out, list(offs)

    # ---- multi-rank hooks (paper_1811_05630_b200/distributed.py drives them)
    def partner_slices_needed(self, action) -> list:
        cnt = C.c_uint64()
        a = action
        self._ck(self.L.qcsim_engine_partner_blocks_needed(self.h, C.byref(a), None, 0, C.byref(cnt)))
        buf = (C.c_uint64 * max(1, cnt.value))()
        self._ck(self.L.qcsim_engine_partner_blocks_needed(self.h, C.byref(a), buf, cnt.value, C.byref(cnt)))
        return list(buf[: cnt.value])

    def export_slice(self, slice_index: int) -> bytes:
        ln = C.c_uint64()
        self._ck(self.L.qcsim_engine_export_slice(self.h, slice_index, None, 0, C.byref(ln)))
        out = np.empty(ln.value, dtype=np.uint8)
        self._ck(self.L.qcsim_engine_export_slice(self.h, slice_index, out.ctypes.data_as(_native.u8p), out.size,
                                                  C.byref(ln)))
        return out.tobytes()

    def export_slices(self, slices) -> tuple:
        """Blocks of several owned slices in one device gather + one copy:
        (bytes, offsets) with offsets[k] the start of slices[k]."""
        arr = (C.c_uint64 * max(1, len(slices)))(*slices)
        ln = C.c_uint64()
        offs = (C.c_uint64 * (len(slices) + 1))()
        self._ck(self.L.qcsim_engine_export_slices(self.h, arr, len(slices), None, 0, C.byref(ln), offs))
        out = np.empty(ln.value, dtype=np.uint8)
        self._ck(self.L.qcsim_engine_export_slices(self.h, arr, len(slices), out.ctypes.data_as(_native.u8p),
                                                   out.size, C.byref(ln), offs))
        return out, list(offs)

    def export_slices_device(self, slices, out_ptr=None, capacity=0):
        """Device-direct export: gathers the slices' blocks into the device
        buffer at `out_ptr` (None: size query).  Returns (total bytes,
        per-plane offsets)."""
        arr = (C.c_uint64 * max(1, len(slices)))(*slices)
        ln = C.c_uint64()
        offs = (C.c_uint64 * (2 * len(slices) + 1))()
        self._ck(self.L.qcsim_engine_export_slices_device(self.h, arr, len(slices), out_ptr, capacity, C.byref(ln),
                                                          offs))
        return ln.value, list(offs)

    def import_partners_device(self, slices, ptr, plane_offsets):
        """Registers partner slices whose blocks sit in a device buffer
        (kept alive by the caller until the next run returns)."""
        arr = (C.c_uint64 * max(1, len(slices)))(*slices)
        offs = (C.c_uint64 * max(1, len(plane_offsets)))(*plane_offsets)
        self._ck(self.L.qcsim_engine_import_partners_device(self.h, arr, len(slices), ptr, offs))

    def import_partner(self, slice_index: int, data: bytes):
        b = np.frombuffer(data, dtype=np.uint8).copy()
        self._ck(self.L.qcsim_engine_import_partner(self.h, slice_index, b.ctypes.data_as(_native.u8p), b.size))

    def set_global_norms(self, norms):
        v = np.ascontiguousarray(norms, dtype=np.float64)
        self._ck(self.L.qcsim_engine_set_global_norms(self.h, v.ctypes.data_as(_native.dp), v.size))


def measure_overhead(actions, config: EngineConfig, basis: int = 0) -> RunMetrics:
    """SPEC.md:353-361 (Fig. 2: "24x, 21x and 19x"): the
    circuit twice on the same device, compression on (`config`) and off;
    returns the compressed run's metrics with baseline_wall_seconds and
    overhead_factor = wall_on / wall_off filled (device time of the gate
    passes)."""
    import dataclasses
    on = Engine(config)
    on.load_basis(basis)
    on.run(actions)
    m = on.full_metrics()
    off = Engine(dataclasses.replace(config, compression_enabled=False))
    off.load_basis(basis)
    moff = off.run(actions)
    on.close()
    off.close()
    m.baseline_wall_seconds = moff.wall_seconds
    m.overhead_factor = m.wall_seconds / moff.wall_seconds if moff.wall_seconds > 0 else None
    return m


def device_memory(reset_peak: bool = False) -> dict:
    """Device bytes held by libqcsim_b200.so: current and high-water mark."""
    cur, peak = C.c_uint64(), C.c_uint64()
    raise_status(_native.lib().qcsim_device_memory(C.byref(cur), C.byref(peak), int(reset_peak)), _native.lib())
    return {"current_bytes": cur.value, "peak_bytes": peak.value}


def kernel_launches() -> int:
    """Kernels launched by libqcsim_b200.so in this process."""
    return int(_native.lib().qcsim_kernel_launches())
