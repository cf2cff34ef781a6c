"""Circuit IR, workload builders and gate lowering -- Python mirror of
proj/include/qcsim/circuit.hpp (host-side; not accelerated).

Conventions (circuit.hpp:20-21): qubit 0 is the least-significant bit of a
basis index; CPhase(theta) multiplies |11> by exp(i*theta).

Lowering (gate_action, circuit.cpp:392-427) is bit-identical to the
reference: same 1/sqrt(2) literal, same std::cos/std::sin (glibc via
math.cos/math.sin) -- tests/test_oracle_golden.py::
test_python_lowering_matches_reference pins it against the compiled reference.  Extension: U3 enters as a pre-lowered
ButterflyOp; its matrix convention is stated in ``u3_matrix``.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Union

from ._native import ActionC


class GateKind(enum.IntEnum):
    H = 0
    X = 1
    Y = 2
    Z = 3
    S = 4
    T = 5
    Phase = 6
    CPhase = 7
    CNOT = 8
    CZ = 9
    Swap = 10
    MCZ = 11


@dataclass
class Gate:
    kind: GateKind
    theta: float = 0.0
    qubits: List[int] = field(default_factory=list)

    def target(self) -> int:
        return self.qubits[-1]

    def control(self) -> int:
        return self.qubits[0]

    @staticmethod
    def h(q): return Gate(GateKind.H, 0.0, [q])
    @staticmethod
    def x(q): return Gate(GateKind.X, 0.0, [q])
    @staticmethod
    def y(q): return Gate(GateKind.Y, 0.0, [q])
    @staticmethod
    def z(q): return Gate(GateKind.Z, 0.0, [q])
    @staticmethod
    def s(q): return Gate(GateKind.S, 0.0, [q])
    @staticmethod
    def t(q): return Gate(GateKind.T, 0.0, [q])
    @staticmethod
    def phase(theta, q): return Gate(GateKind.Phase, theta, [q])
    @staticmethod
    def cphase(theta, c, t): return Gate(GateKind.CPhase, theta, [c, t])
    @staticmethod
    def cnot(c, t): return Gate(GateKind.CNOT, 0.0, [c, t])
    @staticmethod
    def cz(c, t): return Gate(GateKind.CZ, 0.0, [c, t])
    @staticmethod
    def swap(a, b): return Gate(GateKind.Swap, 0.0, [a, b])
    @staticmethod
    def mcz(qs): return Gate(GateKind.MCZ, 0.0, list(qs))


@dataclass
class Circuit:
    num_qubits: int = 0
    name: str = ""
    gates: List[Gate] = field(default_factory=list)

    def gate_count(self) -> int:
        return len(self.gates)


_ARITY = {GateKind.H: 1, GateKind.X: 1, GateKind.Y: 1, GateKind.Z: 1, GateKind.S: 1, GateKind.T: 1,
          GateKind.Phase: 1, GateKind.CPhase: 2, GateKind.CNOT: 2, GateKind.CZ: 2, GateKind.Swap: 2}


def validate_gate(g: Gate, n: int) -> None:
    """circuit.cpp:51-69."""
    if g.kind == GateKind.MCZ:
        if not g.qubits:
            raise ValueError("mcz needs at least one qubit")
    elif len(g.qubits) != _ARITY[g.kind]:
        raise ValueError("wrong qubit count for gate")
    seen = set()
    for q in g.qubits:
        if q < 0 or q >= n:
            raise ValueError(f"qubit index {q} out of range")
        if q in seen:
            raise ValueError("duplicate qubit index in gate")
        seen.add(q)
    if not math.isfinite(g.theta):
        raise ValueError("gate angle must be finite")


def validate_circuit(c: Circuit) -> None:
    if c.num_qubits < 1:
        raise ValueError("circuit needs at least one qubit")
    for g in c.gates:
        validate_gate(g, c.num_qubits)


def build_qft(n: int, include_swaps: bool = True) -> Circuit:
    """circuit.cpp:88-104."""
    if n < 1:
        raise ValueError("QFT needs at least one qubit")
    c = Circuit(n, f"qft{n}")
    for i in range(n - 1, -1, -1):
        c.gates.append(Gate.h(i))
        for j in range(i - 1, -1, -1):
            c.gates.append(Gate.cphase(math.pi / math.ldexp(1.0, i - j), j, i))
    if include_swaps:
        for i in range(n // 2):
            c.gates.append(Gate.swap(i, n - 1 - i))
    return c


def build_grover_oracle(n: int, marked: int) -> Circuit:
    """circuit.cpp:106-125."""
    if n < 2:
        raise ValueError("Grover search needs at least two qubits")
    if marked >= (1 << n):
        raise ValueError("marked state out of range")
    c = Circuit(n, "grover_oracle")
    flips = [Gate.x(q) for q in range(n) if not (marked >> q) & 1]
    c.gates = flips + [Gate.mcz(range(n))] + [Gate.x(q) for q in range(n) if not (marked >> q) & 1]
    return c


def build_grover(n: int, marked: int, iterations: int) -> Circuit:
    """circuit.cpp:127-160."""
    if n < 2:
        raise ValueError("Grover search needs at least two qubits")
    if marked >= (1 << n):
        raise ValueError("marked state out of range")
    if iterations < 1:
        raise ValueError("iterations must be at least 1")
    c = Circuit(n, f"grover{n}")
    c.gates = [Gate.h(q) for q in range(n)]
    oracle = build_grover_oracle(n, marked).gates
    for _ in range(iterations):
        c.gates += oracle
        c.gates += [Gate.h(q) for q in range(n)]
        c.gates += [Gate.x(q) for q in range(n)]
        c.gates.append(Gate.mcz(range(n)))
        c.gates += [Gate.x(q) for q in range(n)]
        c.gates += [Gate.h(q) for q in range(n)]
    return c


def grover_optimal_iterations(n: int) -> int:
    """circuit.cpp:162-168."""
    if n < 2:
        raise ValueError("Grover search needs at least two qubits")
    r = math.floor(math.pi / 4.0 * math.sqrt(math.ldexp(1.0, n)))
    return 1 if r < 1.0 else int(r)


# ------------------------------------------------------------ gate algebra
INV_SQRT2 = 0.7071067811865475244

Amplitude = complex


@dataclass
class Mat2:
    u00: complex
    u01: complex
    u10: complex
    u11: complex


@dataclass
class DiagonalOp:
    mask: int
    factor: complex


@dataclass
class ButterflyOp:
    u: Mat2
    target: int
    control_mask: int


@dataclass
class SwapOp:
    a: int
    b: int


GateAction = Union[DiagonalOp, ButterflyOp, SwapOp]


def unitary2(kind: GateKind, theta: float = 0.0) -> Mat2:
    """circuit.cpp:366-390."""
    r = INV_SQRT2
    if kind == GateKind.H:
        return Mat2(complex(r, 0), complex(r, 0), complex(r, 0), complex(-r, 0))
    if kind == GateKind.X:
        return Mat2(0j, 1 + 0j, 1 + 0j, 0j)
    if kind == GateKind.Y:
        return Mat2(0j, complex(0, -1), complex(0, 1), 0j)
    if kind == GateKind.Z:
        return Mat2(1 + 0j, 0j, 0j, -1 + 0j)
    if kind == GateKind.S:
        return Mat2(1 + 0j, 0j, 0j, 1j)
    if kind == GateKind.T:
        return Mat2(1 + 0j, 0j, 0j, complex(r, r))
    if kind == GateKind.Phase:
        return Mat2(1 + 0j, 0j, 0j, complex(math.cos(theta), math.sin(theta)))
    raise ValueError("gate kind has no single-qubit matrix")


def gate_action(g: Gate) -> GateAction:
    """circuit.cpp:392-427."""
    k = g.kind
    if k in (GateKind.H, GateKind.X, GateKind.Y):
        return ButterflyOp(unitary2(k), g.target(), 0)
    if k == GateKind.Z:
        return DiagonalOp(1 << g.target(), complex(-1.0, 0.0))
    if k == GateKind.S:
        return DiagonalOp(1 << g.target(), complex(0.0, 1.0))
    if k == GateKind.T:
        return DiagonalOp(1 << g.target(), complex(INV_SQRT2, INV_SQRT2))
    if k == GateKind.Phase:
        return DiagonalOp(1 << g.target(), complex(math.cos(g.theta), math.sin(g.theta)))
    if k == GateKind.CPhase:
        return DiagonalOp((1 << g.control()) | (1 << g.target()), complex(math.cos(g.theta), math.sin(g.theta)))
    if k == GateKind.CNOT:
        return ButterflyOp(unitary2(GateKind.X), g.target(), 1 << g.control())
    if k == GateKind.CZ:
        return DiagonalOp((1 << g.control()) | (1 << g.target()), complex(-1.0, 0.0))
    if k == GateKind.Swap:
        return SwapOp(g.qubits[0], g.qubits[1])
    if k == GateKind.MCZ:
        m = 0
        for q in g.qubits:
            m |= 1 << q
        return DiagonalOp(m, complex(-1.0, 0.0))
    raise ValueError("unknown gate kind")


def to_action_c(op: GateAction) -> ActionC:
    """Flatten a GateAction into the C-ABI POD (include/qcsim_c.h)."""
    a = ActionC()
    if isinstance(op, DiagonalOp):
        a.kind, a.mask = 0, op.mask
        a.factor[0], a.factor[1] = op.factor.real, op.factor.imag
    elif isinstance(op, ButterflyOp):
        a.kind, a.target, a.mask = 1, op.target, op.control_mask
        for i, z in enumerate((op.u.u00, op.u.u01, op.u.u10, op.u.u11)):
            a.u[2 * i], a.u[2 * i + 1] = z.real, z.imag
    else:
        a.kind, a.a, a.b = 2, op.a, op.b
    return a


def lower(c: Circuit):
    """Circuit -> list of C-ABI actions."""
    return [to_action_c(gate_action(g)) for g in c.gates]


# ------------------------------------------------- U3 / random circuits (c4)
def u3_matrix(theta: float, phi: float, lam: float) -> Mat2:
    """U3 convention:
    [[cos(t/2), -e^{i lam} sin(t/2)], [e^{i phi} sin(t/2), e^{i(phi+lam)} cos(t/2)]],
    entries computed once on the host with libm."""
    c, s = math.cos(theta / 2.0), math.sin(theta / 2.0)
    e_l = complex(math.cos(lam), math.sin(lam))
    e_p = complex(math.cos(phi), math.sin(phi))
    e_pl = complex(math.cos(phi + lam), math.sin(phi + lam))
    return Mat2(complex(c, 0.0), complex(-e_l.real * s, -e_l.imag * s), complex(e_p.real * s, e_p.imag * s),
                complex(e_pl.real * c, e_pl.imag * c))


def mt19937_64(seed: int):
    """std::mt19937_64 raw outputs (sequence fixed by the C++ standard)."""
    NN, MM = 312, 156
    A, UM, LM = 0xB5026F5AA96619E9, 0xFFFFFFFF80000000, 0x7FFFFFFF
    mask = (1 << 64) - 1
    mt = [0] * NN
    mt[0] = seed & mask
    for i in range(1, NN):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & mask
    idx = NN
    while True:
        if idx >= NN:
            for i in range(NN):
                x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM)
                xa = (x >> 1) ^ (A if x & 1 else 0)
                mt[i] = mt[(i + MM) % NN] ^ xa
            idx = 0
        x = mt[idx]
        idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        yield x & mask


def random_u3_circuit_actions(n: int, depth: int, seed: int):
    """Config 4 (BASELINE.json configs[3]): per layer U3(theta,phi,lambda)
    on every qubit with angles uniform in [0, 2pi), then CZ on a seeded
    random perfect matching.  Angles = (rng() >> 11) * 2^-53 * 2pi;
    matching = Fisher-Yates with rng() % (i+1), paired consecutively."""
    rng = mt19937_64(seed)
    acts = []
    for _ in range(depth):
        for q in range(n):
            th, ph, la = [((next(rng) >> 11) * 2.0**-53) * (2.0 * math.pi) for _ in range(3)]
            acts.append(to_action_c(ButterflyOp(u3_matrix(th, ph, la), q, 0)))
        perm = list(range(n))
        for i in range(n - 1, 0, -1):
            j = next(rng) % (i + 1)
            perm[i], perm[j] = perm[j], perm[i]
        for k in range(0, n - 1, 2):
            acts.append(to_action_c(DiagonalOp((1 << perm[k]) | (1 << perm[k + 1]), complex(-1.0, 0.0))))
    return acts


def seeded_index(n: int, seed: int) -> int:
    """Basis / marked index drawn from the seed: rng() & (2^n - 1)."""
    return next(mt19937_64(seed)) & ((1 << n) - 1)
