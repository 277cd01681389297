"""Coefficient fields as postfix "field programs".

The reference passes coefficients as `ScalarField` callbacks evaluated on whole
arrays of physical quadrature points (proj/include/hdg/coefficient.hpp:13-14).
A C ABI cannot carry a callback into a GPU kernel, so the engine accepts either
sampled arrays (Nq x Nelt, the callback already evaluated by the caller) or a
small postfix program over (x, y, z) that the kernels evaluate at each node.
This module compiles a Python expression string into that program.

Opcodes (keep in sync with include/hdg_b200.h HDG_OP_*):
  0 X  1 Y  2 Z  3 CONST  4 ADD  5 SUB  6 MUL  7 DIV  8 NEG
  9 SIN 10 COS 11 EXP 12 SQRT 13 ABS 14 LT(a,b)=a<b 15 POW
"""
from __future__ import annotations

import ast
import math
from dataclasses import dataclass, field
from typing import List

OP = dict(X=0, Y=1, Z=2, CONST=3, ADD=4, SUB=5, MUL=6, DIV=7, NEG=8, SIN=9, COS=10,
          EXP=11, SQRT=12, ABS=13, LT=14, POW=15)
MAX_STACK = 16
MAX_OPS = 256

_BIN = {ast.Add: OP["ADD"], ast.Sub: OP["SUB"], ast.Mult: OP["MUL"], ast.Div: OP["DIV"],
        ast.Pow: OP["POW"]}
_FUN1 = {"sin": OP["SIN"], "cos": OP["COS"], "exp": OP["EXP"], "sqrt": OP["SQRT"],
         "abs": OP["ABS"]}


@dataclass
class FieldProgram:
    """A compiled scalar field f(x, y, z)."""
    expr: str
    ops: List[int] = field(default_factory=list)
    consts: List[float] = field(default_factory=list)

    def __call__(self, x, y, z):
        """Evaluate with numpy (host-side helper for samples/tests)."""
        import numpy as np
        st = []
        ci = 0
        for op in self.ops:
            if op == 0: st.append(np.asarray(x, dtype=float))
            elif op == 1: st.append(np.asarray(y, dtype=float))
            elif op == 2: st.append(np.asarray(z, dtype=float))
            elif op == 3: st.append(np.float64(self.consts[ci])); ci += 1
            elif op in (4, 5, 6, 7, 14, 15):
                b = st.pop(); a = st.pop()
                st.append({4: lambda: a + b, 5: lambda: a - b, 6: lambda: a * b,
                           7: lambda: a / b, 14: lambda: (a < b) * 1.0,
                           15: lambda: a ** b}[op]())
            elif op == 8: st.append(-st.pop())
            else:
                a = st.pop()
                st.append({9: np.sin, 10: np.cos, 11: np.exp, 12: np.sqrt, 13: np.abs}[op](a))
        return st[0] + 0.0 * np.asarray(x, dtype=float)


def compile_field(expr: str | float) -> FieldProgram:
    """Compile e.g. "1 + 0.5*sin(2*pi*x)*cos(2*pi*y)" into a FieldProgram."""
    if isinstance(expr, (int, float)):
        expr = repr(float(expr))
    prog = FieldProgram(expr)
    depth = [0, 0]

    def push(n=1):
        depth[0] += n
        depth[1] = max(depth[1], depth[0])

    def emit(node):
        if isinstance(node, ast.Expression):
            return emit(node.body)
        if isinstance(node, ast.Constant):
            prog.ops.append(OP["CONST"]); prog.consts.append(float(node.value)); push(); return
        if isinstance(node, ast.Name):
            if node.id in ("x", "y", "z"):
                prog.ops.append(OP[node.id.upper()]); push(); return
            if node.id == "pi":
                prog.ops.append(OP["CONST"]); prog.consts.append(math.pi); push(); return
            raise ValueError(f"unknown name {node.id!r} in field {expr!r}")
        if isinstance(node, ast.BinOp) and type(node.op) in _BIN:
            emit(node.left); emit(node.right)
            prog.ops.append(_BIN[type(node.op)]); depth[0] -= 1; return
        if isinstance(node, ast.UnaryOp) and isinstance(node.op, (ast.USub, ast.UAdd)):
            emit(node.operand)
            if isinstance(node.op, ast.USub):
                prog.ops.append(OP["NEG"])
            return
        if isinstance(node, ast.Call) and isinstance(node.func, ast.Name):
            name = node.func.id
            if name in _FUN1 and len(node.args) == 1:
                emit(node.args[0]); prog.ops.append(_FUN1[name]); return
            if name == "lt" and len(node.args) == 2:
                emit(node.args[0]); emit(node.args[1]); prog.ops.append(OP["LT"]); depth[0] -= 1
                return
            if name == "pow" and len(node.args) == 2:
                emit(node.args[0]); emit(node.args[1]); prog.ops.append(OP["POW"]); depth[0] -= 1
                return
        raise ValueError(f"unsupported construct in field {expr!r}: {ast.dump(node)}")

    emit(ast.parse(str(expr), mode="eval"))
    if depth[1] > MAX_STACK or len(prog.ops) > MAX_OPS:
        raise ValueError(f"field {expr!r} too large for the device VM")
    return prog
