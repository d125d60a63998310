"""CUDA code generation for fused elementwise programs.

An ``EwProgram`` (the canonical Composite payload, reference
``ops/elemwise.py:646-673``) becomes one translation unit: the hand-written
template ``csrc/ew_template.cuh`` plus generated macros holding the
straight-line scalar body.  ``tx_ew_compile`` builds it with NVRTC for
sm_100a; modules are cached per program key for the life of the process.

Floating-point contract: operands are converted to each kernel's declared
compute dtype, and the module is compiled with ``-fmad=false`` so
``a*b+c`` rounds twice exactly like NumPy's separate ufunc passes.
"""
from __future__ import annotations

import os
import struct
import threading

from .dtypes import C_TYPE, FLOAT32, FLOAT64, is_float
from .elemwise import EwProgram, kernel_compute_dtype

_TEMPLATE_PATH = os.path.join(os.path.dirname(__file__), "csrc", "ew_template.cuh")
_template_text = None


def template_text() -> str:
    global _template_text
    if _template_text is None:
        with open(_TEMPLATE_PATH) as f:
            _template_text = f.read()
    return _template_text


def literal(dtype: str, value) -> str:
    """Exact C spelling of a constant in ``dtype``."""
    if dtype == FLOAT32:
        bits = struct.unpack("<I", struct.pack("<f", float(value)))[0]
        return f"__int_as_float(0x{bits:08x})"
    if dtype == FLOAT64:
        bits = struct.unpack("<q", struct.pack("<d", float(value)))[0]
        return f"__longlong_as_double({bits}LL)"
    if dtype == "bool":
        return "((u8)1)" if bool(value) else "((u8)0)"
    if dtype == "int32":
        return f"((int){int(value)})"
    return f"((i64){int(value)}LL)"


def _cast(expr: str, src: str, dst: str) -> str:
    if src == dst:
        return expr
    if dst == "bool":
        return f"((u8)(({expr}) != 0))"
    return f"(({C_TYPE[dst]})({expr}))"


def scalar_expr(kernel: str, args: list, arg_dtypes: list, out_dtype: str) -> str:
    """C expression for one scalar kernel; args already C expressions."""
    cd = kernel_compute_dtype(kernel, arg_dtypes)
    if kernel == "switch":
        c = f"(({args[0]}) != 0)"
        a = _cast(args[1], arg_dtypes[1], cd)
        b = _cast(args[2], arg_dtypes[2], cd)
        return _cast(f"({c} ? {a} : {b})", cd, out_dtype)
    if kernel == "second":
        return _cast(args[1], arg_dtypes[1], out_dtype)
    xs = [_cast(a, d, cd) for a, d in zip(args, arg_dtypes)]
    ct = C_TYPE[cd]
    if kernel in ("add", "sub", "mul"):
        op = {"add": "+", "sub": "-", "mul": "*"}[kernel]
        if cd == "bool":  # numpy bool add/mul are logical or/and
            e = f"((int){xs[0]} {op} (int){xs[1]})"
            return _cast(e, "int32", out_dtype)
        return _cast(f"({xs[0]} {op} {xs[1]})", cd, out_dtype)
    if kernel == "div":
        return _cast(f"tx_div<{ct}>({xs[0]}, {xs[1]}, err)" if not is_float(cd)
                     else f"tx_div({xs[0]}, {xs[1]}, err)", cd, out_dtype)
    if kernel == "neg":
        return _cast(f"(-{xs[0]})", cd, out_dtype)
    if kernel == "sqr":
        return _cast(f"({xs[0]} * {xs[0]})", cd, out_dtype)
    if kernel in ("exp", "log", "log1p", "sqrt", "tanh", "sigmoid"):
        fn = f"tx_{kernel}"
        return _cast(f"{fn}({xs[0]})" if is_float(cd) else f"{fn}<{ct}>({xs[0]})", cd, out_dtype)
    if kernel == "pow":
        return _cast(f"tx_pow({xs[0]}, {xs[1]})" if is_float(cd) else f"tx_pow<{ct}>({xs[0]}, {xs[1]})",
                     cd, out_dtype)
    if kernel == "maximum":
        return _cast(f"tx_maximum({xs[0]}, {xs[1]})" if is_float(cd)
                     else f"tx_maximum<{ct}>({xs[0]}, {xs[1]})", cd, out_dtype)
    if kernel in ("lt", "gt", "le", "ge", "eq", "neq"):
        op = {"lt": "<", "gt": ">", "le": "<=", "ge": ">=", "eq": "==", "neq": "!="}[kernel]
        return f"((u8)({xs[0]} {op} {xs[1]}))"
    if kernel == "isnan":
        return f"tx_isnan({xs[0]})" if is_float(cd) else "((u8)0)"
    raise ValueError(f"no CUDA spelling for kernel {kernel!r}")


def program_body(p: EwProgram) -> str:
    lines = []
    for j, (k, refs, dt) in enumerate(p.nodes):
        args, dts = [], []
        for kind, i in refs:
            if kind == "in":
                args.append(f"(({C_TYPE[p.in_dtypes[i]]})IN({i}))")
            elif kind == "const":
                args.append(literal(*p.consts[i]))
            else:
                args.append(f"t{i}")
            dts.append(p.ref_dtype((kind, i)))
        lines.append(f"const {C_TYPE[dt]} t{j} = {scalar_expr(k, args, dts, dt)};")
    for o, ref in enumerate(p.outputs):
        kind, i = ref
        src = f"t{i}" if kind == "node" else (f"(({C_TYPE[p.in_dtypes[i]]})IN({i}))" if kind == "in"
                                               else literal(*p.consts[i]))
        lines.append(f"OUT({o}, ({C_TYPE[p.out_dtypes[o]]})({src}));")
    return "{ " + " ".join(lines) + " }"


def generate_source(p: EwProgram) -> str:
    n_out, n_in = len(p.outputs), len(p.in_dtypes)
    if n_out + n_in > 24:
        raise ValueError("program has more than 24 operands")
    out_dt = p.out_dtypes
    ptrs = []
    for k, d in enumerate(out_dt):
        ptrs.append(f"{C_TYPE[d]}* q{k} = ({C_TYPE[d]}*)a.ptr[{k}];")
    for k, d in enumerate(p.in_dtypes):
        ptrs.append(f"const {C_TYPE[d]}* p{k} = (const {C_TYPE[d]}*)a.ptr[{n_out + k}];")
    vdecl = " ".join(f"V4<{C_TYPE[d]}> vout{k};" for k, d in enumerate(out_dt))
    vload = " ".join(f"const V4<{C_TYPE[d]}> vin{k} = tx_ld4(p{k} + (o_));" for k, d in enumerate(p.in_dtypes))
    vstore = " ".join(f"tx_st4(q{k} + (o_), vout{k});" for k in range(n_out))
    vload2d = " ".join(f"const V4<{C_TYPE[d]}> vin{k} = tx_ld4b(p{k} + OFF({n_out + k}), a.strides[{n_out + k}][1]);"
                       for k, d in enumerate(p.in_dtypes))
    vstore2d = " ".join(f"tx_st4(q{k} + OFF({k}), vout{k});" for k in range(n_out))
    body = program_body(p)
    return "\n".join([
        "#define TX_KERNELS 1",
        f"#define TX_NOPS {n_out + n_in}",
        f"#define TX_IN_SLOT(k) ((k) + {n_out})",
        f"#define TX_PTRS {' '.join(ptrs)}",
        f"#define TX_VDECL {vdecl}",
        f"#define TX_VLOAD(o_) {vload}",
        f"#define TX_VSTORE(o_) {vstore}",
        f"#define TX_VLOAD2D {vload2d}",
        f"#define TX_VSTORE2D {vstore2d}",
        f"#define TX_BODY {body}",
        template_text(),
    ])


def has_int_div(p: EwProgram) -> bool:
    return any(k == "div" and not is_float(kernel_compute_dtype(k, [p.ref_dtype(r) for r in refs]))
               for k, refs, _ in p.nodes)


class KernelCache:
    """NVRTC modules keyed by program; shared by all compiled functions."""

    def __init__(self):
        self._lock = threading.Lock()
        self._mods: dict = {}

    def get(self, lib, p: EwProgram):
        key = p.key()
        with self._lock:
            h = self._mods.get(key)
            if h is None:
                h = lib.ew_compile(generate_source(p), f"ew{len(self._mods)}")
                self._mods[key] = h
            return h


CACHE = KernelCache()


def lower_elementwise(node, plan, program: EwProgram) -> None:
    """Append the launch of ``program`` over ``node``'s operands to a plan."""
    plan.emit_elementwise(node, program)
