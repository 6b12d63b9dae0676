"""Operator expressions and permutation-invariant (PIT) axes.

Host-side analysis that feeds plan construction; it performs no per-step arithmetic. Same
grammar and classification rules as ``pittile.expr`` (reference pkg/src/pittile/expr.py:194-344):

    OUT[ax,...] (+= | =) IN1[ax,...] ((* | +) IN2[ax,...])?     ax := sym | sym+sym (inputs only)

An axis is PIT iff it is not inside a compound subscript and is spatial (in the output) or an
additive reduction. An axis present in every operand is *prevalent*: each slice along it may carry
its own permutation (``simplify``), which is how batched / per-expert / per-head operators get one
independent micro-tile index per slice.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field, replace
from typing import Mapping, Optional

SPATIAL, REDUCTION = "spatial", "reduction"
SPORADIC, PREVALENT, COMPOUND = "sporadic", "prevalent", "compound-member"


class ExprError(ValueError):
    def __init__(self, message: str, position: Optional[int] = None):
        super().__init__(message if position is None else f"{message} (at position {position})")
        self.position = position


@dataclass(frozen=True)
class Axis:
    syms: tuple[str, ...]

    @property
    def is_compound(self) -> bool:
        return len(self.syms) == 2

    def __str__(self) -> str:
        return "+".join(self.syms)


@dataclass(frozen=True)
class Operand:
    name: str
    axes: tuple[Axis, ...]

    def symbols(self) -> tuple[str, ...]:
        return tuple(s for ax in self.axes for s in ax.syms)

    def __str__(self) -> str:
        return f"{self.name}[{','.join(map(str, self.axes))}]"


@dataclass(frozen=True)
class TensorExpr:
    output: Operand
    inputs: tuple[Operand, ...]
    elementwise_op: str = "identity"
    reduction_op: str = "sum"
    accumulate: bool = True
    extents: Mapping[str, int] = field(default_factory=dict)

    def operands(self) -> tuple[Operand, ...]:
        return (self.output, *self.inputs)

    def symbols(self) -> tuple[str, ...]:
        seen: dict[str, None] = {}
        for op in self.operands():
            for s in op.symbols():
                seen.setdefault(s, None)
        return tuple(seen)

    def extent(self, sym: str) -> int:
        if sym not in self.extents:
            raise ExprError(f"axis {sym!r} has no bound extent")
        return self.extents[sym]

    def text(self) -> str:
        sep = {"multiply": " * ", "add": " + ", "identity": ""}[self.elementwise_op]
        return f"{self.output} {'+=' if self.accumulate else '='} {sep.join(map(str, self.inputs))}"


@dataclass(frozen=True)
class AxisInfo:
    name: str
    kind: str
    category: str
    is_pit: bool
    extent: Optional[int] = None


_TOK = re.compile(r"\s*(?:(?P<name>[A-Za-z_]\w*)|(?P<op>\+=|[=,\[\]+*]))")
_NAME = re.compile(r"[A-Za-z_]\w*")


def _tokens(text: str) -> list[tuple[str, int]]:
    out, pos = [], 0
    while pos < len(text):
        if text[pos:].strip() == "":
            break
        m = _TOK.match(text, pos)
        if m is None:
            bad = pos + len(text[pos:]) - len(text[pos:].lstrip())
            raise ExprError(f"unexpected character {text[bad]!r}", position=bad)
        kind = "name" if m.group("name") else "op"
        out.append((m.group(kind), m.start(kind)))
        pos = m.end()
    return out


def parse_expr(text: str) -> TensorExpr:
    if not text.isascii():
        raise ExprError("expression must be ASCII")
    toks = _tokens(text)
    i = 0

    def peek():
        return toks[i][0] if i < len(toks) else None

    def take(want=None):
        nonlocal i
        if i >= len(toks):
            raise ExprError(f"unexpected end of expression, expected {want or 'token'}", position=len(text))
        tok, pos = toks[i]
        if want is not None and tok != want:
            raise ExprError(f"expected {want!r}, got {tok!r}", position=pos)
        i += 1
        return tok

    def name():
        tok = take()
        if not _NAME.fullmatch(tok):
            raise ExprError(f"expected name, got {tok!r}", position=toks[i - 1][1])
        return tok

    def operand(compound_ok: bool) -> Operand:
        nm = name()
        take("[")
        axes = []
        while peek() != "]":
            first = name()
            if peek() == "+":
                take("+")
                second = name()
                if not compound_ok:
                    raise ExprError(f"compound term {first}+{second} not allowed in output", position=toks[i - 1][1])
                axes.append(Axis((first, second)))
            else:
                axes.append(Axis((first,)))
            if peek() == ",":
                take(",")
            elif peek() != "]":
                take("]")
        take("]")
        return Operand(nm, tuple(axes))

    out = operand(False)
    assign = take()
    if assign not in ("+=", "="):
        raise ExprError(f"expected '+=' or '=', got {assign!r}", position=toks[i - 1][1])
    ins = [operand(True)]
    ew = "identity"
    if peek() in ("*", "+"):
        ew = "multiply" if take() == "*" else "add"
        ins.append(operand(True))
    if peek() is not None:
        raise ExprError(f"trailing input after expression: {peek()!r}", position=toks[i][1])
    expr = TensorExpr(out, tuple(ins), ew, accumulate=assign == "+=")
    seen: dict[str, tuple[Axis, ...]] = {}
    for op in expr.operands():
        if seen.setdefault(op.name, op.axes) != op.axes:
            raise ExprError(f"operand {op.name!r} repeated with different subscripts")
    in_syms = {s for op in expr.inputs for s in op.symbols()}
    for s in out.symbols():
        if s not in in_syms:
            raise ExprError(f"output axis {s!r} appears in no input")
    return expr


def classify_axes(expr: TensorExpr) -> tuple[AxisInfo, ...]:
    out_syms = set(expr.output.symbols())
    compound = {s for op in expr.operands() for ax in op.axes if ax.is_compound for s in ax.syms}
    per_op = [set(op.symbols()) for op in expr.operands()]
    infos = []
    for s in expr.symbols():
        kind = SPATIAL if s in out_syms else REDUCTION
        cat = COMPOUND if s in compound else PREVALENT if all(s in p for p in per_op) else SPORADIC
        pit = cat != COMPOUND and (kind == SPATIAL or expr.reduction_op == "sum")
        infos.append(AxisInfo(s, kind, cat, pit, expr.extents.get(s)))
    return tuple(infos)


def pit_axes(expr: TensorExpr) -> frozenset:
    return frozenset(a.name for a in classify_axes(expr) if a.is_pit)


def simplify(expr: TensorExpr):
    prevalent = {a.name for a in classify_axes(expr) if a.category == PREVALENT}
    if not prevalent:
        return expr, {}

    def strip(op: Operand) -> Operand:
        return Operand(op.name, tuple(ax for ax in op.axes if ax.is_compound or ax.syms[0] not in prevalent))

    reduced = replace(
        expr,
        output=strip(expr.output),
        inputs=tuple(strip(op) for op in expr.inputs),
        extents={k: v for k, v in expr.extents.items() if k not in prevalent},
    )
    return reduced, {s: "independent-per-slice" for s in sorted(prevalent)}


def bind_extents(expr: TensorExpr, extents: Mapping[str, int]) -> TensorExpr:
    for s in expr.symbols():
        if s not in extents:
            raise ExprError(f"no extent bound for axis {s!r}")
        if int(extents[s]) <= 0:
            raise ExprError(f"extent for axis {s!r} must be positive")
    return replace(expr, extents={s: int(extents[s]) for s in expr.symbols()})


def operator_kind(expr: TensorExpr) -> str:
    if any(ax.is_compound for op in expr.operands() for ax in op.axes):
        return "convolution"
    core, removed = simplify(expr)
    out = [a.syms[0] for a in core.output.axes]
    ins = [[a.syms[0] for a in op.axes] for op in core.inputs]
    if core.elementwise_op == "multiply" and len(ins) == 2 and len(out) == 2 and core.accumulate:
        red = ins[0][-1] if ins[0] else None
        if ins[0] == [out[0], red] and ins[1] == [red, out[1]]:
            return "batch_matmul" if removed else "matmul"
    if core.elementwise_op == "identity" and len(ins) == 1 and core.accumulate:
        extra = set(ins[0]) - set(out)
        if set(out) <= set(ins[0]) and extra:
            return "reduce_sum"
        if not extra and removed:
            return "reduce_sum"
    if core.elementwise_op == "add" and len(ins) == 2 and ins[0] == ins[1] == out:
        return "vec_add"
    return "custom"
