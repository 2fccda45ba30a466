"""Gate-list IR and the OpenQASM 2.0 subset frontend.

Same IR as the reference (``GateKind``/``GateOp``/``Circuit``,
/root/reference/pkg/src/hisim/qasm.py:26-100): 19 gate kinds, controls first
and target last, angles in radians evaluated at parse time. The engine only
consumes ``GateKind`` + qubits + params; the parser and serializer exist so
circuits round-trip through the same text the reference reads
(``parse_qasm`` ~ qasm.py:263-355, ``to_qasm`` ~ qasm.py:358-375).
"""

from __future__ import annotations

import enum
import math
import re
from dataclasses import dataclass, field

from .errors import (
    DuplicateQubitError,
    InvalidQubitCountError,
    QasmSyntaxError,
    QubitOutOfRangeError,
    UnsupportedGateError,
)


class GateKind(enum.Enum):
    """The supported gates; the value is the OpenQASM mnemonic."""

    H = "h"
    X = "x"
    Y = "y"
    Z = "z"
    S = "s"
    T = "t"
    SDG = "sdg"
    TDG = "tdg"
    RX = "rx"
    RY = "ry"
    RZ = "rz"
    U1 = "u1"
    U3 = "u3"
    CX = "cx"
    CZ = "cz"
    CRZ = "crz"
    CRY = "cry"
    SWAP = "swap"
    CCX = "ccx"

    @property
    def arity(self) -> int:
        return _SIGNATURE[self][0]

    @property
    def num_params(self) -> int:
        return _SIGNATURE[self][1]


# (arity, number of angle parameters) per kind
_SIGNATURE: dict[GateKind, tuple[int, int]] = {}
for _k in GateKind:
    _SIGNATURE[_k] = (1, 0)
for _k in (GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.U1):
    _SIGNATURE[_k] = (1, 1)
_SIGNATURE[GateKind.U3] = (1, 3)
for _k in (GateKind.CX, GateKind.CZ, GateKind.SWAP):
    _SIGNATURE[_k] = (2, 0)
for _k in (GateKind.CRZ, GateKind.CRY):
    _SIGNATURE[_k] = (2, 1)
_SIGNATURE[GateKind.CCX] = (3, 0)

_KIND_BY_MNEMONIC = {k.value: k for k in GateKind}


@dataclass(frozen=True)
class GateOp:
    """One gate application; ``qubits`` lists controls first, target last."""

    kind: GateKind
    qubits: tuple[int, ...]
    params: tuple[float, ...] = ()


@dataclass(frozen=True)
class Circuit:
    """Register width plus the gate list in program order."""

    num_qubits: int
    ops: tuple[GateOp, ...] = field(default_factory=tuple)

    @property
    def num_ops(self) -> int:
        return len(self.ops)


def _check_op(i: int, op: GateOp, n: int, where: str) -> None:
    arity, nparams = _SIGNATURE[op.kind]
    if len(op.qubits) != arity:
        raise InvalidQubitCountError(
            f"{where}{op.kind.value} takes {arity} qubits, got {len(op.qubits)}"
        )
    if len(op.params) != nparams:
        raise InvalidQubitCountError(
            f"{where}{op.kind.value} takes {nparams} params, got {len(op.params)}"
        )
    if len(set(op.qubits)) != arity:
        raise DuplicateQubitError(f"{where}repeated qubit in {op.qubits}")
    for q in op.qubits:
        if q < 0 or q >= n:
            raise QubitOutOfRangeError(f"{where}qubit {q} outside [0, {n})")


def validate(circuit: Circuit) -> None:
    """Raise the matching ``QasmError`` subclass if ``circuit`` breaks an IR
    invariant (reference: qasm.py:103-130)."""
    if circuit.num_qubits < 1:
        raise InvalidQubitCountError(
            f"circuit needs at least one qubit, got {circuit.num_qubits}"
        )
    for i, op in enumerate(circuit.ops):
        _check_op(i, op, circuit.num_qubits, f"op {i}: ")


# --- angle expressions ------------------------------------------------------

_ANGLE_TOKEN = re.compile(
    r"\s*(?:(?P<num>\d+\.\d*(?:[eE][+-]?\d+)?|\.?\d+(?:[eE][+-]?\d+)?)"
    r"|(?P<pi>pi)|(?P<sym>[-+*/^()]))"
)
_BINARY = {"+": 1, "-": 1, "*": 2, "/": 2, "^": 3}


class _AngleParser:
    """Precedence-climbing evaluator for ``pi``-expressions."""

    def __init__(self, text: str, line: int, col: int):
        self.text, self.line, self.col = text, line, col
        self.toks: list = []
        pos = 0
        while pos < len(text):
            m = _ANGLE_TOKEN.match(text, pos)
            if m is None:
                if text[pos:].strip():
                    self.fail("bad angle expression")
                break
            if m.group("num") is not None:
                self.toks.append(float(m.group("num")))
            elif m.group("pi") is not None:
                self.toks.append(math.pi)
            else:
                self.toks.append(m.group("sym"))
            pos = m.end()
        self.i = 0

    def fail(self, what: str):
        raise QasmSyntaxError(f"{what} {self.text!r}", self.line, self.col)

    def peek(self):
        return self.toks[self.i] if self.i < len(self.toks) else None

    def atom(self) -> float:
        tok = self.peek()
        if tok is None:
            self.fail("bad angle expression")
        self.i += 1
        if isinstance(tok, float):
            return tok
        if tok == "-":
            return -self.atom()
        if tok == "+":
            return self.atom()
        if tok == "(":
            val = self.expr(0)
            if self.peek() != ")":
                self.fail("unbalanced parens in")
            self.i += 1
            return val
        self.fail("bad angle expression")

    def expr(self, min_prec: int) -> float:
        val = self.atom()
        while True:
            tok = self.peek()
            if not isinstance(tok, str) or tok not in _BINARY:
                return val
            prec = _BINARY[tok]
            if prec < min_prec:
                return val
            self.i += 1
            rhs = self.expr(prec if tok == "^" else prec + 1)
            if tok == "+":
                val += rhs
            elif tok == "-":
                val -= rhs
            elif tok == "*":
                val *= rhs
            elif tok == "/":
                val /= rhs
            else:
                val **= rhs

    def evaluate(self) -> float:
        if not self.toks:
            raise QasmSyntaxError("empty angle expression", self.line, self.col)
        try:
            val = self.expr(0)
        except ZeroDivisionError:
            self.fail("division by zero in")
        if self.i != len(self.toks):
            self.fail("trailing junk in angle")
        return val


def eval_angle(text: str, line: int = 1, col: int = 1) -> float:
    """Evaluate an angle expression (numbers, ``pi``, ``+ - * / ^``, parens)."""
    return _AngleParser(text, line, col).evaluate()


# --- statements -------------------------------------------------------------

def _split_statements(src: str):
    """Yield ``(statement, line, col)`` for each ';'-terminated statement,
    with ``//`` comments removed and newlines folded to spaces."""
    stmt: list[str] = []
    anchor = None
    line = col = 1
    i = 0
    n = len(src)
    while i < n:
        ch = src[i]
        if ch == "/" and src.startswith("//", i):
            j = src.find("\n", i)
            i = n if j < 0 else j
            continue
        if ch == "\n":
            if stmt:
                stmt.append(" ")
            line += 1
            col = 1
            i += 1
            continue
        if ch == ";":
            text = "".join(stmt).strip()
            if anchor is not None and text:
                yield text, anchor[0], anchor[1]
            stmt, anchor = [], None
        elif anchor is None:
            if not ch.isspace():
                anchor = (line, col)
                stmt.append(ch)
        else:
            stmt.append(ch)
        col += 1
        i += 1
    if anchor is not None and "".join(stmt).strip():
        raise QasmSyntaxError("statement missing ';'", anchor[0], anchor[1])


_QREG = re.compile(r"qreg\s+([A-Za-z_]\w*)\s*\[\s*(\d+)\s*\]$")
_OPERAND = re.compile(r"([A-Za-z_]\w*)\s*\[\s*(\d+)\s*\]$")
_APPLY = re.compile(r"([A-Za-z_]\w*)\s*(\(([^)]*)\))?\s*(.*)$")
_IGNORED = {"OPENQASM", "include", "barrier"}
_REFUSED = {
    "measure": "measurement is not supported (simulation is pure-state)",
    "reset": "reset is not supported",
    "creg": "classical registers are not supported",
    "if": "classical control is not supported",
    "gate": "custom gate definitions are not supported",
    "opaque": "opaque gates are not supported",
}


def parse_qasm(text: str) -> Circuit:
    """Parse OpenQASM 2.0 subset text into a validated ``Circuit``."""
    reg: str | None = None
    width = 0
    ops: list[GateOp] = []
    for stmt, line, col in _split_statements(text):
        words = stmt.split(None, 1)
        head = words[0] if words else stmt
        if head in _IGNORED:
            continue
        if head in _REFUSED:
            raise UnsupportedGateError(f"line {line}: {_REFUSED[head]}")
        if head == "qreg":
            m = _QREG.match(stmt)
            if m is None:
                raise QasmSyntaxError("malformed qreg", line, col)
            if reg is not None:
                raise UnsupportedGateError(
                    f"line {line}: only one quantum register is supported"
                )
            reg, width = m.group(1), int(m.group(2))
            if width < 1:
                raise InvalidQubitCountError(
                    f"line {line}: register must hold at least one qubit"
                )
            continue
        m = _APPLY.match(stmt)
        if m is None:
            raise QasmSyntaxError("unrecognized statement", line, col)
        name, paren, ptext, otext = m.groups()
        kind = _KIND_BY_MNEMONIC.get(name)
        if kind is None:
            raise UnsupportedGateError(f"line {line}: unsupported gate {name!r}")
        if reg is None:
            raise QasmSyntaxError("gate application before qreg", line, col)
        params: tuple[float, ...] = ()
        if paren is not None:
            params = tuple(
                eval_angle(p, line, col) for p in ptext.split(",") if p.strip()
            )
        if len(params) != kind.num_params:
            raise InvalidQubitCountError(
                f"line {line}: {name} takes {kind.num_params} params, "
                f"got {len(params)}"
            )
        qubits = []
        for o in (s.strip() for s in otext.split(",")):
            if not o:
                continue
            om = _OPERAND.match(o)
            if om is None:
                raise QasmSyntaxError(f"bad operand {o!r}", line, col)
            if om.group(1) != reg:
                raise QasmSyntaxError(f"unknown register {om.group(1)!r}", line, col)
            q = int(om.group(2))
            if q >= width:
                raise QubitOutOfRangeError(
                    f"line {line}: qubit {q} outside [0, {width})"
                )
            qubits.append(q)
        op = GateOp(kind, tuple(qubits), params)
        _check_op(len(ops), op, width, f"line {line}: ")
        ops.append(op)
    if reg is None:
        raise QasmSyntaxError("no qreg declaration", 1, 1)
    circuit = Circuit(width, tuple(ops))
    validate(circuit)
    return circuit


def to_qasm(circuit: Circuit) -> str:
    """Canonical text, register ``q``, angles at repr precision so that
    ``parse_qasm(to_qasm(c)) == c``."""
    out = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{circuit.num_qubits}];"]
    for op in circuit.ops:
        head = op.kind.value
        if op.params:
            head += "(" + ",".join(repr(float(p)) for p in op.params) + ")"
        out.append(head + " " + ",".join(f"q[{q}]" for q in op.qubits) + ";")
    return "\n".join(out) + "\n"
