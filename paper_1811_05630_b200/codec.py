"""Codec API -- Python mirror of proj/include/qcsim/codec.hpp over the C-ABI.

Names, defaults, argument meaning and error behaviour follow the reference:
``CodecConfig`` (codec.hpp:52-60), ``CompressedBlock`` (codec.hpp:64-87),
``CodecStats`` (codec.hpp:89-94), ``compress_plane`` / ``decompress_plane``
(codec.hpp:98-103).  Exceptions: ``ValueError`` where the reference throws
std::invalid_argument, ``CodecError`` where it throws qcsim::CodecError.
The arithmetic runs on the GPU (libqcsim_b200.so); nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import raise_status


class CodecMode(enum.IntEnum):
    RangeRelative = 0
    Absolute = 1
    Lossless = 2


class Predictor(enum.IntEnum):
    PreviousValue = 0
    LinearExtrapolation = 1


@dataclass
class CodecConfig:
    mode: CodecMode = CodecMode.RangeRelative
    bound: float = 0.01
    quant_code_bits: int = 16
    predictor: Predictor = Predictor.PreviousValue

    def to_c(self) -> _native.CodecConfigC:
        return _native.CodecConfigC(int(self.mode), int(self.predictor), 0, int(self.quant_code_bits),
                                    float(self.bound))

    def validate(self) -> None:
        """CodecConfig::validate (codec.cpp:331-341)."""
        L = _native.lib()
        c = self.to_c()
        raise_status(L.qcsim_codec_validate(C.byref(c)), L)


@dataclass
class CodecStats:
    input_bytes: int = 0
    output_bytes: int = 0
    ratio: float = 0.0
    outlier_fraction: float = 0.0


def compression_ratio(stats: CodecStats) -> float:
    return float(stats.input_bytes) / float(stats.output_bytes)


@dataclass
class CompressedBlock:
    mode: CodecMode = CodecMode.RangeRelative
    predictor: Predictor = Predictor.PreviousValue
    quant_code_bits: int = 16
    element_count: int = 0
    effective_abs_bound: float = 0.0
    outlier_count: int = 0
    payload: bytes = field(default=b"", repr=False)

    kHeaderBytes = 40
    kFormatVersion = 1

    def byte_size(self) -> int:
        return self.kHeaderBytes + len(self.payload)

    def to_bytes(self) -> bytes:
        """Wire format "QCB1" (codec.cpp:343-364)."""
        hdr = b"QCB1" + struct.pack("<BBBBQdQQ", self.kFormatVersion, int(self.mode), int(self.predictor),
                                    self.quant_code_bits, self.element_count, self.effective_abs_bound,
                                    self.outlier_count, len(self.payload))
        return hdr + bytes(self.payload)

    @classmethod
    def from_bytes(cls, data: bytes):
        """CompressedBlock::from_bytes (codec.cpp:366-408); returns
        (block, consumed)."""
        from .errors import CodecError
        b = bytes(data)
        if len(b) < 40:
            raise CodecError("block header truncated")
        if b[:4] != b"QCB1":
            raise CodecError("bad block magic")
        if b[4] != 1:
            raise CodecError(f"unsupported block version {b[4]}")
        if b[5] > 2:
            raise CodecError("bad codec mode byte")
        if b[6] > 1:
            raise CodecError("bad predictor byte")
        qb = b[7]
        if qb < 4 or qb > 24:
            raise CodecError("quant_code_bits out of range")
        n, eb, outl, plen = struct.unpack_from("<QdQQ", b, 8)
        if n == 0:
            raise CodecError("element_count must be at least 1")
        if outl > n:
            raise CodecError("outlier_count exceeds element_count")
        if not (eb >= 0.0) or not np.isfinite(eb):
            raise CodecError("bad effective_abs_bound")
        if plen > len(b) - 40:
            raise CodecError("block payload truncated")
        blk = cls(CodecMode(b[5]), Predictor(b[6]), qb, n, eb, outl, b[40:40 + plen])
        return blk, 40 + plen


def compress_plane(values, config: CodecConfig):
    """compress_plane (codec.hpp:98-99) on the GPU -> (CompressedBlock, CodecStats)."""
    L = _native.lib()
    v = np.ascontiguousarray(values, dtype=np.float64)
    cfg = config.to_c()
    n = v.size
    cap = int(L.qcsim_block_bound(max(n, 1), int(config.quant_code_bits)))
    out = np.empty(cap, dtype=np.uint8)
    ln = C.c_uint64()
    st = _native.CodecStatsC()
    rc = L.qcsim_compress_plane(v.ctypes.data_as(_native.dp), n, C.byref(cfg),
                                out.ctypes.data_as(_native.u8p), cap, C.byref(ln), C.byref(st))
    raise_status(rc, L)
    data = out[: ln.value].tobytes()
    blk, _ = CompressedBlock.from_bytes(data)
    return blk, CodecStats(st.input_bytes, st.output_bytes, st.ratio, st.outlier_fraction)


def compress_plane_bytes(values, config: CodecConfig) -> bytes:
    blk, _ = compress_plane(values, config)
    return blk.to_bytes()


def decompress_bytes(data: bytes) -> np.ndarray:
    """from_bytes + decompress_plane on the GPU."""
    L = _native.lib()
    b = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    n = C.c_uint64()
    cons = C.c_uint64()
    raise_status(L.qcsim_decompress_plane(b.ctypes.data_as(_native.u8p), b.size, None, 0, C.byref(n),
                                          C.byref(cons)), L)
    out = np.empty(n.value, dtype=np.float64)
    raise_status(L.qcsim_decompress_plane(b.ctypes.data_as(_native.u8p), b.size, out.ctypes.data_as(_native.dp),
                                          out.size, C.byref(n), C.byref(cons)), L)
    return out


def decompress_plane(block: CompressedBlock) -> np.ndarray:
    """decompress_plane (codec.hpp:103) on the GPU."""
    return decompress_bytes(block.to_bytes())
