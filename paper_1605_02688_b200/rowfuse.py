"""Plan-time row fusion: softmax / cross-entropy regions as one kernel.

The reference has no softmax or cross-entropy op; the configs compose them
from max, exp, sum, div, log, mul and DimShuffle, and ``grad`` adds ~25 more
nodes.  On [B, 10] tensors every one of those nodes is
pure launch latency.  With concrete shapes known (step-plan time), this
module finds maximal convex groups of nodes that live in one *row space*
(N rows x K <= 10240 columns) and emits ONE generated kernel per group:

  * one warp per row (K <= 256) or one 1024-thread CTA per row (wider rows:
    a vocabulary-sized softmax); a row vector lives in registers (thread c of
    the row holds columns c, c+T, ...), row scalars are uniform over the row;
  * elementwise nodes and inlined Composite programs run per element
    (same scalar spellings and rounding as ``codegen``);
  * ``sum``/``max``/``argmax``/``argmax_onehot`` over the row are warp-shuffle
    trees, then a fixed-order combine of the warp partials for wide rows
    (max/argmax NaN- and tie-exact);
  * reductions over the batch (``sum[0]`` -> bias gradient, ``sum[0,1]`` ->
    cost) are group sinks: per-CTA partials in fixed order, then the last CTA
    (ticket counter) combines the partials in block order — deterministic, no
    float atomics;
  * only values consumed outside the group are stored.

Value classes inside a group: V row vector [N,K], S row scalar [N]/[N,1],
C column vector [K]/[1,K] (broadcast over rows), U scalar.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import codegen
from .dtypes import C_TYPE, ITEMSIZE, is_float
from .elemwise import Composite, Elemwise, kernel_compute_dtype
from .reduce import Argmax, ArgmaxOnehot, Max, Sum

MAX_K = 256          # warp-per-row form
MAX_WIDE = 10240     # block-per-row form (<= 1024 threads, <= 10 columns per thread)
WIDE_T_ENV = __import__('os').environ.get('TX_ROW_WIDE_T')
MAX_OPS = 48
V, S, C, U = "V", "S", "C", "U"


# every generated kernel waits for its stream predecessor first: the launch is
# programmatic (tx_nvrtc.cu launch_drv; tx_common.h TX_GRID_WAIT)
_GRID_WAIT = 'asm volatile("griddepcontrol.wait;\\n\\tgriddepcontrol.launch_dependents;" ::: "memory");'


def wide_threads(K):
    """Threads per row of the block-per-row form: about 8 columns per thread
    (register-resident rows; measured on softmax-xent fwd+bwd: K=1000 best at
    256, K=4096 at 512, K=10000 at 1024)."""
    if WIDE_T_ENV:
        return int(WIDE_T_ENV)
    t = 256
    while t < 1024 and t * 8 < K:
        t *= 2
    return t


def classify(shape, lead, K):
    """Class of a value in the row space lead + (K,): lead is (N,) for a
    matrix of rows or (A, B) for a rank-3 tensor whose A*B rows are flattened."""
    shape = tuple(shape)
    if isinstance(lead, int):
        lead = (lead,)
    r = len(lead)
    if shape == lead + (K,):
        return V
    if shape in (lead, lead + (1,)):
        return S
    if len(shape) <= r + 1 and shape[-1:] == (K,) and all(d == 1 for d in shape[:-1]):
        return C
    if all(d == 1 for d in shape):
        return U
    return None


def _rows_flat(shape, strides, lead):
    """Can a V / S value of a rank-3 row space be addressed with one row stride?"""
    if len(lead) == 1:
        return True
    return len(shape) >= 2 and (shape[0] <= 1 or strides[0] == shape[1] * strides[1])


def _combine(classes):
    cs = set(classes)
    if V in cs or (S in cs and C in cs):
        return V
    if S in cs:
        return S
    if C in cs:
        return C
    return U


class RowArgs(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("K", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("ptr", ctypes.c_void_p * MAX_OPS), ("rs", ctypes.c_int64 * MAX_OPS),
                ("cs", ctypes.c_int64 * MAX_OPS), ("ws", ctypes.c_void_p), ("counter", ctypes.c_void_p)]


class RowGroup:
    def __init__(self, lead, K):
        self.lead = tuple(lead)
        self.N, self.K = int(np.prod(self.lead)), K
        self.row_axis = len(self.lead)
        self.members = []          # nodes (views included), schedule order
        self.member_ids = set()
        self.values = {}           # var id -> class, for every group-produced value
        self.sink_vars = set()     # var ids produced by sinks (not usable inside)
        self.last_pos = -1
        self.deferred = []         # non-members moved after the launch

    def launchable(self):
        return [n for n in self.members if not getattr(n.op, "view_capable", False)]


# ---------------------------------------------------------------- grouping

def _is_sink(n, shapes, lead):
    """A sum over the batch: all leading (row) axes of a row vector (-> a
    column vector) or every axis (-> a scalar); of a row scalar, its row axes."""
    if not isinstance(n.op, Sum):
        return False
    shp, lead = tuple(shapes(n.inputs[0])), tuple(lead)
    r = len(lead)
    rows, every = tuple(range(r)), tuple(range(len(shp)))
    if len(shp) == r + 1 and shp[:r] == lead:
        return n.op.axes in (rows, every)
    if shp in (lead, lead + (1,)):
        return n.op.axes in (rows, every)
    return False


def _flat_ok(plan, v, grp):
    """Rank-3 row spaces read every V / S operand through one row stride."""
    if len(grp.lead) == 1 or v.id not in plan.lay:
        return True
    lay = plan.lay[v.id]
    if classify(lay.shape, grp.lead, grp.K) not in (V, S):
        return True
    return _rows_flat(lay.shape, lay.strides, grp.lead)


def _node_fits(n, grp, shapes, allowed_in, plan=None):
    """Can node n join group grp (given the values the group already has)?"""
    op = n.op
    lead, K = grp.lead, grp.K
    ins = [classify(shapes(x), lead, K) for x in n.inputs]
    outs = [classify(shapes(o), lead, K) for o in n.outputs]
    if any(c is None for c in ins + outs):
        return False
    if any(x.id in grp.sink_vars for x in n.inputs):
        return False
    if plan is not None and not all(_flat_ok(plan, x, grp) for x in n.inputs):
        return False
    # (not necessarily connected: any row-space node whose inputs are ready
    # can run inside the group — fewer launches)
    if not all(allowed_in(x) for x in n.inputs):
        return False
    if getattr(op, "view_capable", False):
        return outs[0] == ins[0] or {outs[0], ins[0]} <= {U}
    if isinstance(op, (Elemwise, Composite)):
        prog_has_int_div = codegen.has_int_div(op.program) if isinstance(op, Composite) else (
            op.kernel == "div" and not is_float(kernel_compute_dtype("div", [x.type.dtype for x in n.inputs])))
        return not prog_has_int_div
    if isinstance(op, (Sum, Max, ArgmaxOnehot, Argmax)):
        if op.axes == (grp.row_axis,) and ins[0] == V:
            return is_float(n.inputs[0].type.dtype)
        if isinstance(op, Sum) and _is_sink(n, shapes, lead) and ins[0] in (V, S):
            # a wide row's column sums ([N, K] -> [K]) would be combined by a
            # single CTA; they stay a separate (parallel) column reduction
            return not (grp.K > MAX_K and ins[0] == V and op.axes == tuple(range(len(lead))))
        return False
    return False


def _seed(n, shapes, exclude_ids, plan=None):
    """A node that can open a group: a reduction over the last axis of an
    [N, K] or [A, B, K] tensor, or an elementwise node producing one (the
    logits' bias add), 2 <= K <= MAX_WIDE."""
    if n.id in exclude_ids:
        return None
    op = n.op
    if isinstance(op, (Sum, Max, ArgmaxOnehot, Argmax)):
        shp = tuple(shapes(n.inputs[0]))
        if op.axes != (len(shp) - 1,) or not is_float(n.inputs[0].type.dtype):
            return None
    elif isinstance(op, (Elemwise, Composite)):
        shp = tuple(shapes(n.outputs[0]))
        if any(tuple(shapes(o)) != tuple(shp) for o in n.outputs):
            return None
        if isinstance(op, Composite) and codegen.has_int_div(op.program):
            return None
    else:
        return None
    if len(shp) not in (2, 3):
        return None
    lead, K = shp[:-1], shp[-1]
    N = int(np.prod(lead))
    if not (2 <= K <= MAX_WIDE) or N < 2 or N >= (1 << 31) or K in lead or (len(lead) == 2 and N == K):
        return None
    grp = RowGroup(lead, K)
    for x in n.inputs:
        if classify(shapes(x), lead, K) is None or (plan is not None and not _flat_ok(plan, x, grp)):
            return None
    return grp


def find_groups(plan, order, fgraph, exclude_ids=()):
    """Greedy convex grouping over the schedule.

    The group launches at its last member.  A non-member that reads a group
    value (e.g. the scalar cost composite reading the batch-sum sink) is
    *deferred* to run right after the launch, together with everything that
    depends on it; a would-be member that needs a deferred value closes the
    group instead.  Nodes in ``exclude_ids`` (data-parallel partial sums,
    whose allreduce is positioned by the schedule) are never deferred: reading
    a group value closes the group.  Groups with fewer than two launching
    members are dropped (their deferred nodes stay in place).
    """
    shapes = lambda v: plan.lay[v.id].shape if v.id in plan.lay else tuple(v.value.shape)  # noqa: E731
    groups, cur = [], None
    deferred_out = set()

    def close():
        nonlocal cur
        # a wide-row (block-per-row) group pays only where it fuses row
        # reductions; pure elementwise work on wide rows stays on the
        # 128-bit elementwise kernels
        if cur is not None and len(cur.launchable()) >= 2 and (cur.K <= MAX_K or any(
                isinstance(n.op, (Sum, Max, ArgmaxOnehot, Argmax)) and n.op.axes == (cur.row_axis,)
                for n in cur.members)):
            groups.append(cur)
        cur = None
        deferred_out.clear()

    def add(grp, n, i):
        grp.members.append(n)
        grp.member_ids.add(n.id)
        grp.last_pos = i
        sink = _is_sink(n, shapes, grp.lead)
        for o in n.outputs:
            grp.values[o.id] = classify(shapes(o), grp.lead, grp.K)
            if sink:
                grp.sink_vars.add(o.id)

    for i, n in enumerate(order):
        reads_group = cur is not None and any(x.id in cur.values for x in n.inputs)
        reads_deferred = any(x.id in deferred_out for x in n.inputs)
        if cur is not None and not reads_deferred and n.id not in exclude_ids \
                and _node_fits(n, cur, shapes, lambda x: True, plan):
            add(cur, n, i)
            continue
        if (reads_group or reads_deferred) and cur is not None and len(cur.launchable()) < 2:
            # a one-kernel group would only drag everything downstream into
            # its deferred list (blocking later groups): drop it here
            close()
            reads_group = reads_deferred = False
        if (reads_group or reads_deferred) and n.id not in exclude_ids:
            cur.deferred.append(n)
            for o in n.outputs:
                deferred_out.add(o.id)
            continue
        if reads_group or reads_deferred:
            close()
        g = _seed(n, shapes, exclude_ids, plan)
        if g is not None:
            close()
            cur = g
            add(cur, n, i)
    close()
    for grp in groups:
        # deferred nodes positioned after the last member run in place
        grp.deferred = [n for n in grp.deferred if order.index(n) < grp.last_pos]
    return groups


# ---------------------------------------------------------------- codegen

_PRELUDE = r"""
typedef long long i64;
typedef unsigned char u8;
#define TX_R %(R)d
#define TX_T %(T)d
struct TxRowArgs { i64 N; int K; int pad; void* ptr[%(MAXOPS)d]; i64 rs[%(MAXOPS)d]; i64 cs[%(MAXOPS)d];
                   double* ws; unsigned int* counter; };
__device__ __forceinline__ float tx_sigmoid(float x) { float z = expf(-fabsf(x)); return x >= 0.0f ? 1.0f / (1.0f + z) : z / (1.0f + z); }
__device__ __forceinline__ double tx_sigmoid(double x) { double z = exp(-fabs(x)); return x >= 0.0 ? 1.0 / (1.0 + z) : z / (1.0 + z); }
__device__ __forceinline__ float tx_exp(float x) { return expf(x); }
__device__ __forceinline__ double tx_exp(double x) { return exp(x); }
__device__ __forceinline__ float tx_log(float x) { return logf(x); }
__device__ __forceinline__ double tx_log(double x) { return log(x); }
__device__ __forceinline__ float tx_log1p(float x) { return log1pf(x); }
__device__ __forceinline__ double tx_log1p(double x) { return log1p(x); }
__device__ __forceinline__ float tx_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double tx_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float tx_tanh(float x) { return tanhf(x); }
__device__ __forceinline__ double tx_tanh(double x) { return tanh(x); }
__device__ __forceinline__ float tx_pow(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double tx_pow(double a, double b) { return pow(a, b); }
template <class T> __device__ __forceinline__ T tx_exp(T x) { return (T)exp((double)x); }
template <class T> __device__ __forceinline__ T tx_log(T x) { return (T)log((double)x); }
template <class T> __device__ __forceinline__ T tx_log1p(T x) { return (T)log1p((double)x); }
template <class T> __device__ __forceinline__ T tx_sqrt(T x) { return (T)sqrt((double)x); }
template <class T> __device__ __forceinline__ T tx_tanh(T x) { return (T)tanh((double)x); }
template <class T> __device__ __forceinline__ T tx_sigmoid(T x) { return (T)tx_sigmoid((double)x); }
template <class T> __device__ __forceinline__ T tx_pow(T a, T b) { if (b < 0) return (T)0; T r = 1; while (b) { if (b & 1) r *= a; a *= a; b >>= 1; } return r; }
__device__ __forceinline__ float tx_maximum(float a, float b) { return (a != a) ? a : (b != b) ? b : (a > b ? a : b); }
__device__ __forceinline__ double tx_maximum(double a, double b) { return (a != a) ? a : (b != b) ? b : (a > b ? a : b); }
template <class T> __device__ __forceinline__ T tx_maximum(T a, T b) { return a > b ? a : b; }
__device__ __forceinline__ float tx_div(float a, float b, int*) { return a / b; }
__device__ __forceinline__ double tx_div(double a, double b, int*) { return a / b; }
__device__ __forceinline__ u8 tx_isnan(float a) { return a != a; }
__device__ __forceinline__ u8 tx_isnan(double a) { return a != a; }
template <class T> __device__ __forceinline__ T tx_wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class T> __device__ __forceinline__ T tx_wmax(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T w = __shfl_xor_sync(0xffffffffu, v, o); v = (v != v) ? v : ((w != w) ? w : (w > v ? w : v)); }
  return v;
}
// first maximal (NaN counts as maximal) with index tie-break across lanes
template <class T> __device__ __forceinline__ void tx_wargmax(T& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    int j = __shfl_xor_sync(0xffffffffu, i, o);
    bool vn = v != v, wn = w != w;
    bool take = (j >= 0) && ((i < 0) || (vn && wn ? j < i : vn ? false : wn ? true : (w > v || (w == v && j < i))));
    if (take) { v = w; i = j; }
  }
}
// block-wide forms (one row per CTA, wide rows): warp trees, then every
// warp combines the per-warp partials in the same fixed order
template <class T> __device__ __forceinline__ T tx_bsum(T v) {
  __shared__ T sh[32];
  v = tx_wsum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  T r = (l < (int)(blockDim.x >> 5)) ? sh[l] : (T)0;
  return tx_wsum(r);
}
template <class T> __device__ __forceinline__ T tx_bmax(T v) {
  __shared__ T sh[32];
  v = tx_wmax(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  T r = (l < (int)(blockDim.x >> 5)) ? sh[l] : sh[0];
  return tx_wmax(r);
}
template <class T> __device__ __forceinline__ void tx_bargmax(T& v, int& i) {
  __shared__ T shv[32];
  __shared__ int shi[32];
  tx_wargmax(v, i);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { shv[w] = v; shi[w] = i; }
  __syncthreads();
  if (l < (int)(blockDim.x >> 5)) { v = shv[l]; i = shi[l]; } else { v = shv[0]; i = -1; }
  tx_wargmax(v, i);
}
"""


class _Gen:
    def __init__(self, grp: RowGroup, plan, fgraph):
        self.grp, self.plan, self.fg = grp, plan, fgraph
        self.N, self.K = grp.N, grp.K
        self.block = grp.K > MAX_K          # one row per CTA of wide_threads(K) threads
        self.T = wide_threads(grp.K) if self.block else 32
        self.R = (grp.K + self.T - 1) // self.T
        rs = "tx_b" if self.block else "tx_w"
        self.rsum, self.rmax, self.rarg = rs + "sum", rs + "max", rs + "argmax"
        self.lines = []
        self.name = {}      # var id -> C identifier
        self.cls = {}       # var id -> class
        self.dt = {}        # var id -> dtype
        self.ops = []       # (var, role) operand slots: role in {"in", "out", "sink"}
        self.slot = {}
        self.sinks = []     # (var, class_of_sink_output, acc identifier, dtype, length)

    def shape(self, v):
        return self.plan.lay[v.id].shape if v.id in self.plan.lay else tuple(v.value.shape)

    def operand(self, v, role):
        key = (v.id, role)
        if key not in self.slot:
            self.slot[key] = len(self.ops)
            self.ops.append((v, role))
        return self.slot[key]

    def emit(self, s):
        self.lines.append(s)

    # value access: per-element expression for class V/C arrays or scalar name
    def at(self, vid, j="j"):
        c = self.cls[vid]
        return f"{self.name[vid]}[{j}]" if c in (V, C) else self.name[vid]

    def leaf(self, v):
        if v.id in self.name:
            return
        cls = classify(self.shape(v), self.grp.lead, self.K)
        ct = C_TYPE[v.type.dtype]
        k = self.operand(v, "in")
        nm = f"L{k}"
        p = f"((const {ct}*)a.ptr[{k}])"
        if cls == V:
            self.emit(f"{ct} {nm}[TX_R];")
            self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                      f"{nm}[j] = (active && c < K) ? {p}[row * a.rs[{k}] + (i64)c * a.cs[{k}]] : ({ct})0; }}")
        elif cls == C:
            self.emit(f"{ct} {nm}[TX_R];")
            self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                      f"{nm}[j] = (c < K) ? {p}[(i64)c * a.cs[{k}]] : ({ct})0; }}")
        elif cls == S:
            self.emit(f"const {ct} {nm} = active ? {p}[row * a.rs[{k}]] : ({ct})0;")
        else:
            self.emit(f"const {ct} {nm} = {p}[0];")
        self.name[v.id], self.cls[v.id], self.dt[v.id] = nm, cls, v.type.dtype

    def elementwise(self, out_id, out_dt, kernel, arg_ids_or_lits):
        """arg_ids_or_lits: list of ("var", id) or ("lit", c_expr, dtype)."""
        classes = [self.cls[a[1]] if a[0] == "var" else U for a in arg_ids_or_lits]
        oc = _combine(classes)
        dts = [self.dt[a[1]] if a[0] == "var" else a[2] for a in arg_ids_or_lits]
        ct = C_TYPE[out_dt]
        nm = f"t{len(self.name)}"

        def args(j):
            return [(self.at(a[1], j) if a[0] == "var" else a[1]) for a in arg_ids_or_lits]

        if oc in (V, C):
            self.emit(f"{ct} {nm}[TX_R];")
            self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {nm}[j] = "
                      f"{codegen.scalar_expr(kernel, args('j'), dts, out_dt)};")
        else:
            self.emit(f"const {ct} {nm} = {codegen.scalar_expr(kernel, args('j'), dts, out_dt)};")
        self.name[out_id], self.cls[out_id], self.dt[out_id] = nm, oc, out_dt

    def node(self, n):
        op = n.op
        for x in n.inputs:
            if x.id not in self.name:
                self.leaf(x)
        if getattr(op, "view_capable", False):
            o, x = n.outputs[0], n.inputs[0]
            self.name[o.id], self.cls[o.id], self.dt[o.id] = self.name[x.id], self.cls[x.id], self.dt[x.id]
            return
        if isinstance(op, Elemwise):
            self.elementwise(n.outputs[0].id, n.outputs[0].type.dtype, op.kernel,
                             [("var", x.id) for x in n.inputs])
            return
        if isinstance(op, Composite):
            p = op.program
            inner = []
            for j, (k, refs, dt) in enumerate(p.nodes):
                args = []
                for kind, i in refs:
                    if kind == "in":
                        args.append(("var", n.inputs[i].id))
                    elif kind == "node":
                        args.append(("var", inner[i]))
                    else:
                        d, val = p.consts[i]
                        args.append(("lit", codegen.literal(d, val), d))
                vid = ("c", n.id, j)
                self.elementwise(vid, dt, k, args)
                inner.append(vid)
            for o, (kind, i) in zip(n.outputs, p.outputs):
                src = inner[i] if kind == "node" else n.inputs[i].id if kind == "in" else None
                if src is None:
                    d, val = p.consts[i]
                    self.elementwise(o.id, o.type.dtype, "second", [("lit", "0", d), ("lit", codegen.literal(d, val), d)])
                else:
                    self.name[o.id], self.cls[o.id], self.dt[o.id] = self.name[src], self.cls[src], self.dt[src]
            return
        x, o = n.inputs[0], n.outputs[0]
        ct = C_TYPE[x.type.dtype]
        xn = self.name[x.id]
        nm = f"t{len(self.name)}"
        ra = (self.grp.row_axis,)
        if isinstance(op, Sum) and op.axes == ra:
            self.emit(f"{ct} {nm} = 0;")
            self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) if (tc + TX_T * j < K) {nm} += {xn}[j];")
            self.emit(f"{nm} = {self.rsum}({nm});")
            self.name[o.id], self.cls[o.id], self.dt[o.id] = nm, S, o.type.dtype
        elif isinstance(op, Max) and op.axes == ra:
            self.emit(f"{ct} {nm} = {xn}[0];")
            self.emit(f"#pragma unroll\nfor (int j = 1; j < TX_R; ++j) if (tc + TX_T * j < K) {{ {ct} w = {xn}[j]; "
                      f"{nm} = ({nm} != {nm}) ? {nm} : ((w != w) ? w : (w > {nm} ? w : {nm})); }}")
            self.emit(f"if (tc >= K) {nm} = -__int_as_float(0x7f800000);" if ct == "float" else f"if (tc >= K) {nm} = -__longlong_as_double(0x7ff0000000000000LL);")
            self.emit(f"{nm} = {self.rmax}({nm});")
            # a zero maximum takes the sign of the row's LAST zero (np.maximum.reduce
            # keeps the later operand on ties, so +0/-0 ties resolve by position)
            self.emit(f"if ({nm} == ({ct})0) {{ int zk = -1;\n#pragma unroll\nfor (int j = 0; j < TX_R; ++j) "
                      f"{{ const int c = tc + TX_T * j; if (c < K && {xn}[j] == ({ct})0) zk = 2 * c + (signbit({xn}[j]) ? 1 : 0); }}\n"
                      f"zk = {self.rmax}(zk); {nm} = (zk & 1) ? -({ct})0 : ({ct})0; }}")
            self.name[o.id], self.cls[o.id], self.dt[o.id] = nm, S, o.type.dtype
        elif isinstance(op, (Argmax, ArgmaxOnehot)) and op.axes == ra:
            iv, ii = f"{nm}_v", f"{nm}_i"
            self.emit(f"{ct} {iv} = {xn}[0]; int {ii} = tc < K ? tc : -1;")
            self.emit(f"#pragma unroll\nfor (int j = 1; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                      f"if (c < K) {{ {ct} w = {xn}[j]; if ({ii} < 0 || w > {iv} || (w != w && {iv} == {iv})) "
                      f"{{ {iv} = w; {ii} = c; }} }} }}")
            self.emit(f"{self.rarg}({iv}, {ii});")
            if isinstance(op, Argmax):
                self.emit(f"const i64 {nm} = (i64){ii};")
                self.name[o.id], self.cls[o.id], self.dt[o.id] = nm, S, o.type.dtype
            else:
                ot = C_TYPE[o.type.dtype]
                self.emit(f"{ot} {nm}[TX_R];")
                self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {nm}[j] = (tc + TX_T * j == {ii}) ? "
                          f"({ot})1 : ({ot})0;")
                self.name[o.id], self.cls[o.id], self.dt[o.id] = nm, V, o.type.dtype
        elif isinstance(op, Sum):  # sinks: reduce over the batch
            cin = self.cls[x.id]
            acc = f"SK{len(self.sinks)}"
            if op.axes == tuple(range(len(self.grp.lead))) and cin == V:
                self.emit(f"{ct} {acc}[TX_R];")
                self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {acc}[j] = "
                          f"(active && tc + TX_T * j < K) ? {xn}[j] : ({ct})0;")
                self.sinks.append((o, C, acc, x.type.dtype, self.K))
            else:
                if cin == V:
                    self.emit(f"double {acc} = 0;")
                    self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) if (tc + TX_T * j < K) {acc} += (double){xn}[j];")
                    self.emit(f"{acc} = {self.rsum}({acc});")
                    self.emit(f"{acc} = active ? {acc} : 0.0;")
                else:
                    self.emit(f"const double {acc} = active ? (double){xn} : 0.0;")
                self.sinks.append((o, U, acc, x.type.dtype, 1))
            self.operand(o, "sink")
        else:  # pragma: no cover
            raise NotImplementedError(op.name)

    def stores(self, store_ids):
        for vid in store_ids:
            v = store_ids[vid]
            k = self.operand(v, "out")
            ct = C_TYPE[v.type.dtype]
            p = f"(({ct}*)a.ptr[{k}])"
            c = self.cls[vid]
            src = self.name[vid]
            if c == V:
                self.emit(f"if (active) {{\n#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                          f"if (c < K) {p}[row * a.rs[{k}] + (i64)c * a.cs[{k}]] = ({ct}){src}[j]; }} }}")
            elif c == S:
                self.emit(f"if (active && tc == 0) {p}[row * a.rs[{k}]] = ({ct}){src};")
            elif c == C:
                self.emit(f"if (blockIdx.x == 0 && {'true' if self.block else 'warp == 0'}) {{\n#pragma unroll\nfor (int j = 0; j < TX_R; ++j) "
                          f"{{ const int c = tc + TX_T * j; if (c < K) {p}[(i64)c * a.cs[{k}]] = ({ct}){src}[j]; }} }}")
            else:
                self.emit(f"if (blockIdx.x == 0 && threadIdx.x == 0) {p}[0] = ({ct}){src};")

    def finish_sinks(self):
        if not self.sinks:
            return 0
        total = sum(L for *_, L in self.sinks)
        off = 0
        offs = []
        if self.block:
            # one row per CTA: the CTA partial is the row's own contribution
            for (o, c, acc, dt, L) in self.sinks:
                offs.append(off)
                if c == C:
                    self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                              f"if (c < K) a.ws[(i64)blockIdx.x * {total} + {off} + c] = (double){acc}[j]; }}")
                else:
                    self.emit(f"if (tc == 0) a.ws[(i64)blockIdx.x * {total} + {off}] = (double){acc};")
                off += L
        else:
            self.emit(f"__shared__ double sk_smem[8][{total}];")
            for (o, c, acc, dt, L) in self.sinks:
                offs.append(off)
                if c == C:
                    self.emit(f"#pragma unroll\nfor (int j = 0; j < TX_R; ++j) {{ const int c = tc + TX_T * j; "
                              f"if (c < K) sk_smem[warp][{off} + c] = (double){acc}[j]; }}")
                else:
                    self.emit(f"if (lane == 0) sk_smem[warp][{off}] = (double){acc};")
                off += L
            self.emit("__syncthreads();")
            # CTA partial in fixed warp order, in the sink's own precision
            self.emit(f"for (int e = threadIdx.x; e < {total}; e += blockDim.x) {{")
            for (o, c, acc, dt, L), so in zip(self.sinks, offs):
                self.emit(f"  if (e >= {so} && e < {so + L}) {{ double s = 0; for (int w = 0; w < 8; ++w) "
                          f"s += sk_smem[w][e]; a.ws[(i64)blockIdx.x * {total} + e] = s; }}")
            self.emit("}")
        self.emit("__threadfence(); __syncthreads();")
        self.emit("__shared__ unsigned int sk_ticket; if (threadIdx.x == 0) sk_ticket = atomicAdd(a.counter, 1u);")
        self.emit("__syncthreads();")
        self.emit("if (sk_ticket == gridDim.x - 1) {")
        self.emit("  __threadfence();")
        # one warp per sink element (elements strided over the 8 warps): lanes
        # sum a fixed strided slice of the block partials, then a fixed xor
        # tree -> deterministic, and no CTA-wide barriers in the loop
        self.emit(f"  for (int e = warp; e < {total}; e += (int)(blockDim.x >> 5)) {{")
        self.emit("    double s = 0;")
        self.emit(f"    for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(a.ws + (i64)b * {total} + e);")
        self.emit("    s = tx_wsum(s);")
        self.emit("    if (lane == 0) {")
        for (o, c, acc, dt, L), so in zip(self.sinks, offs):
            ot = C_TYPE[o.type.dtype]
            k = self.slot[(o.id, "sink")]
            self.emit(f"      if (e >= {so} && e < {so + L}) (({ot}*)a.ptr[{k}])[(i64)(e - {so}) * a.cs[{k}]] = ({ot})s;")
        self.emit("    }")
        self.emit("  }")
        self.emit("  if (threadIdx.x == 0) *a.counter = 0u;")
        self.emit("}")
        return total

    def source(self, body, total):
        head = _PRELUDE % {"R": self.R, "T": self.T, "MAXOPS": MAX_OPS}
        if self.block:
            pre = [f'extern "C" __global__ void __launch_bounds__({self.T}) tx_row(const TxRowArgs a) {{',
                   _GRID_WAIT,
                   "const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;",
                   "const i64 row = (i64)blockIdx.x;", "const int tc = threadIdx.x;"]
        else:
            pre = ['extern "C" __global__ void __launch_bounds__(256) tx_row(const TxRowArgs a) {',
                   _GRID_WAIT,
                   "const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;",
                   "const i64 row = (i64)blockIdx.x * 8 + warp;", "const int tc = lane;"]
        return "\n".join([head] + pre + ["const bool active = row < a.N;", "const int K = a.K;",
                                          "(void)lane; (void)warp; (void)tc;", "int* err = nullptr; (void)err;"]
                         + body + ["}"])


_CACHE: dict = {}
_LOCK = threading.Lock()


def emit_group(plan, grp: RowGroup, fgraph):
    """Generate, compile (cached by source) and register the group's launch."""
    import torch
    members = grp.member_ids
    # values consumed outside the group (or returned) must be stored
    store = {}
    for n in grp.members:
        for o in n.outputs:
            if o.id in grp.sink_vars:
                continue
            outside = fgraph.is_output(o) or any(c.id not in members for c in fgraph.node_clients(o))
            if outside:
                base = o
                while base.owner is not None and getattr(base.owner.op, "view_capable", False) \
                        and base.owner.id in members:
                    base = base.owner.inputs[0]
                if base.owner is not None and base.owner.id in members:
                    store[base.id] = base
    gen = _Gen(grp, plan, fgraph)
    for n in grp.members:
        gen.node(n)
    gen.stores(store)
    total = gen.finish_sinks()
    src = gen.source(gen.lines, total)
    lib = plan.lib
    with _LOCK:
        h = _CACHE.get(src)
        if h is None:
            h = lib.kernel_compile(src, f"row{len(_CACHE)}", "tx_row")
            _CACHE[src] = h
    args = RowArgs()
    args.N, args.K = grp.N, grp.K
    for k, (v, role) in enumerate(gen.ops):
        lay = plan.lay[v.id] if v.id in plan.lay else plan._const_layout(v)
        t = plan.tx(lay)
        args.ptr[k] = t.data
        shp, st = lay.shape, lay.strides
        cls = classify(shp, grp.lead, grp.K)
        r = len(grp.lead)
        if cls == V:
            args.rs[k], args.cs[k] = st[r - 1], st[r]      # rank-3: rows flattened (checked by _flat_ok)
        elif cls == S:
            args.rs[k], args.cs[k] = st[r - 1], 0
        elif cls == C:
            args.rs[k], args.cs[k] = 0, st[-1]
        else:
            args.rs[k], args.cs[k] = 0, 1
    grid = grp.N if gen.block else (grp.N + 7) // 8
    threads = gen.T if gen.block else 256
    if total:
        ws = torch.zeros(grid * total * 8 + 256, dtype=torch.uint8, device="cuda")
        plan.keep.append(ws)
        args.ws = ws.data_ptr()
        args.counter = ws.data_ptr() + grid * total * 8
    f = lib.lib.tx_kernel_launch
    ap = ctypes.cast(ctypes.pointer(args), ctypes.c_void_p)
    plan.keep.append(args)

    def launch(stream):
        lib.check(f(h, grid, threads, ap, stream))
    return launch, src
