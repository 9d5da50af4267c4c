"""Python mirror of the reference recording surface and of the batch oracle.

`Tape` keeps the names, argument meaning and error behaviour of the
reference's C++ API (tapegrad::Tape, /root/reference/proj/include/tapegrad/
tape.hpp:68-353, and the ops.hpp free functions :38-307), recording through
the C-ABI recorder of libtg.so.  `Program` is the GPU replacement of the
reference's per-sample train_step loop: compile once, then
`forward_backward` / `gd_update` for whole batches on the device.

PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib


class OpKind(enum.IntEnum):
    """Reference op_kind.hpp:10-44 numbering (+ the stop-gradient max)."""
    Leaf = 0
    Relu = 1
    Tanh = 2
    Exp = 3
    NegLog = 4
    Sigmoid = 5
    Inv = 6
    Sqr = 7
    Cub = 8
    Log = 9
    Sqrt = 10
    InvSqrt = 11
    Add = 12
    Sub = 13
    Mul = 14
    MulByConst = 15
    Div = 16
    Mean = 17
    AddSquares = 18
    MeanSquares = 19
    NegativeMean = 20
    AddVarying = 21
    SubVarying = 22
    MulVarying = 23
    MeanVarying = 24
    SumOfSquaresVarying = 25
    MeanSquaresVarying = 26
    NegativeMeanVarying = 27
    InnerProductNoBias = 28
    InnerProductWithBias = 29
    StopGradMax = 64


def op_name(op: int) -> str:
    return lib.tg_op_name(int(op)).decode()


MODELS = {"fig1": 1, "listing1": 2, "moons": 3, "char_mlp": 4, "gpt": 5, "wide_mlp": 6}
DEFAULT_DTYPE = {1: "f64", 2: "f64", 3: "f64", 4: "f32", 5: "f32", 6: "f32"}
_DT = {"f64": _lib.TG_F64, "f32": _lib.TG_F32}
_NP = {"f64": np.float64, "f32": np.float32}


def model_id(model) -> int:
    return MODELS[model] if isinstance(model, str) else int(model)


@dataclass
class TapeDesc:
    """Plain-array copy of a recorded tape (tg_tape_desc)."""
    op: np.ndarray
    child_offset: np.ndarray
    child: np.ndarray
    constant: np.ndarray
    leaf_class: np.ndarray
    leaf_index: np.ndarray
    leaf_value: np.ndarray
    gathers: np.ndarray          # [n_gathers, 5] uint32
    root: int
    n_params: int
    n_inputs: int
    n_index_inputs: int
    dtype: str
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_nodes(self) -> int:
        return int(self.op.shape[0])

    @property
    def n_edges(self) -> int:
        return int(self.child.shape[0])

    def children(self, i: int) -> np.ndarray:
        return self.child[self.child_offset[i]:self.child_offset[i + 1]]

    def param_values(self) -> np.ndarray:
        """Initial parameter vector (recorded leaf values), float64."""
        p = np.zeros(self.n_params, np.float64)
        m = self.leaf_class == _lib.TG_LEAF_PARAM
        p[self.leaf_index[m]] = self.leaf_value[m]
        return p

    def to_c(self) -> _lib.tg_tape_desc:
        def ptr(a, t):
            return a.ctypes.data_as(C.POINTER(t))
        arrs = [np.ascontiguousarray(a) for a in (
            self.op.astype(np.uint8), self.child_offset.astype(np.uint64), self.child.astype(np.uint32),
            self.constant.astype(np.float64), self.leaf_class.astype(np.uint8),
            self.leaf_index.astype(np.uint32), self.leaf_value.astype(np.float64),
            self.gathers.astype(np.uint32).reshape(-1, 5))]
        self._keep = arrs
        d = _lib.tg_tape_desc()
        d.n_nodes = self.n_nodes
        d.dtype = _DT[self.dtype]
        d.op = ptr(arrs[0], C.c_uint8)
        d.child_offset = ptr(arrs[1], C.c_uint64)
        d.child = ptr(arrs[2], C.c_uint32)
        d.constant = ptr(arrs[3], C.c_double)
        d.leaf_class = ptr(arrs[4], C.c_uint8)
        d.leaf_index = ptr(arrs[5], C.c_uint32)
        d.leaf_value = ptr(arrs[6], C.c_double)
        d.n_gathers = arrs[7].shape[0]
        d.gathers = arrs[7].ctypes.data_as(C.POINTER(_lib.tg_gather))
        d.root = int(self.root)
        d.n_params = int(self.n_params)
        d.n_inputs = int(self.n_inputs)
        d.n_index_inputs = int(self.n_index_inputs)
        return d


def _desc_from_c(d: _lib.tg_tape_desc) -> TapeDesc:
    n = d.n_nodes
    def arr(p, cnt, dt):
        if cnt == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True)
    off = arr(d.child_offset, n + 1, np.uint64)
    ne = int(off[-1]) if n else 0
    g = np.zeros((d.n_gathers, 5), np.uint32)
    for i in range(d.n_gathers):
        gg = d.gathers[i]
        g[i] = (gg.first_node, gg.stride, gg.n_rows, gg.index_col, gg.offset)
    return TapeDesc(
        op=arr(d.op, n, np.uint8), child_offset=off, child=arr(d.child, ne, np.uint32),
        constant=arr(d.constant, n, np.float64), leaf_class=arr(d.leaf_class, n, np.uint8),
        leaf_index=arr(d.leaf_index, n, np.uint32), leaf_value=arr(d.leaf_value, n, np.float64),
        gathers=g, root=d.root, n_params=d.n_params, n_inputs=d.n_inputs,
        n_index_inputs=d.n_index_inputs, dtype="f64" if d.dtype == _lib.TG_F64 else "f32")


class Tape:
    """Recording tape with the reference API (tape.hpp / ops.hpp names).

    Handles (ValueRef) are plain ints.  Ops evaluate eagerly and raise the
    reference's errors: DomainError (std::domain_error), InvalidArgument
    (std::invalid_argument), TgError(TG_INVALID_HANDLE) for stale handles.
    """

    def __init__(self, capacity: int = 1024, dtype: str = "f64", _handle=None, fixed_capacity: bool = False,
                 child_capacity: int = 0):
        self.dtype = dtype
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            if fixed_capacity:   # TapeConfig{capacity, fixed_capacity, child_capacity} (tape.hpp:40-53)
                check(lib.tg_recorder_new_fixed(_DT[dtype], capacity, child_capacity, C.byref(h)))
            else:
                check(lib.tg_recorder_new(_DT[dtype], capacity, C.byref(h)))
            self._h = h

    # ---- checkpoint / rewind / high-water marks (tape.hpp:98-125, :228-242) ----
    def checkpoint(self) -> _lib.tg_checkpoint:
        cp = _lib.tg_checkpoint()
        check(lib.tg_rec_checkpoint(self._h, C.byref(cp)))
        return cp

    def rewind(self, cp: _lib.tg_checkpoint) -> None:
        check(lib.tg_rec_rewind(self._h, C.byref(cp)))

    def stats(self) -> dict:
        s = _lib.tg_rec_stats()
        check(lib.tg_rec_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_}

    def size(self) -> int:
        return self.stats()["size"]

    def peak_nodes(self) -> int:
        return self.stats()["peak_nodes"]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and lib is not None:
            lib.tg_recorder_free(h)
            self._h = None

    # ---- leaves ----
    def leaf(self, value: float) -> int:
        """Reference Tape::leaf: a constant leaf (not trained, same for all samples)."""
        return self.constant(value)

    def constant(self, value: float) -> int:
        out = C.c_uint32()
        check(lib.tg_rec_const(self._h, float(value), C.byref(out)))
        return out.value

    def param(self, value: float) -> int:
        out = C.c_uint32()
        check(lib.tg_rec_param(self._h, float(value), C.byref(out)))
        return out.value

    def input(self, col: int, value: float) -> int:
        out = C.c_uint32()
        check(lib.tg_rec_input(self._h, int(col), float(value), C.byref(out)))
        return out.value

    def gather(self, first: int, stride: int, n_rows: int, col: int, offset: int, template_index: int) -> int:
        out = C.c_uint32()
        check(lib.tg_rec_gather(self._h, first, stride, n_rows, col, offset, template_index, C.byref(out)))
        return out.value

    # ---- ops ----
    def op(self, kind: int, children, constant: float = 0.0) -> int:
        ch = (C.c_uint32 * max(1, len(children)))(*[int(c) for c in children])
        out = C.c_uint32()
        check(lib.tg_rec_op(self._h, int(kind), ch, len(children), float(constant), C.byref(out)))
        return out.value

    def unary(self, kind, x):
        return self.op(kind, [x])

    def binary(self, kind, x, y):
        return self.op(kind, [x, y])

    def varying(self, kind, xs):
        return self.op(kind, list(xs))

    relu = lambda self, x: self.op(OpKind.Relu, [x])
    tanh = lambda self, x: self.op(OpKind.Tanh, [x])
    exp = lambda self, x: self.op(OpKind.Exp, [x])
    negative_log = lambda self, x: self.op(OpKind.NegLog, [x])
    sigmoid = lambda self, x: self.op(OpKind.Sigmoid, [x])
    inv = lambda self, x: self.op(OpKind.Inv, [x])
    sqr = lambda self, x: self.op(OpKind.Sqr, [x])
    pow3 = lambda self, x: self.op(OpKind.Cub, [x])
    log = lambda self, x: self.op(OpKind.Log, [x])
    sqrt = lambda self, x: self.op(OpKind.Sqrt, [x])
    inv_sqrt = lambda self, x: self.op(OpKind.InvSqrt, [x])
    add = lambda self, x, y: self.op(OpKind.Add, [x, y])
    sub = lambda self, x, y: self.op(OpKind.Sub, [x, y])
    mul = lambda self, x, y: self.op(OpKind.Mul, [x, y])
    div = lambda self, x, y: self.op(OpKind.Div, [x, y])
    mean = lambda self, x, y: self.op(OpKind.Mean, [x, y])
    add_squares = lambda self, x, y: self.op(OpKind.AddSquares, [x, y])
    mean_squares = lambda self, x, y: self.op(OpKind.MeanSquares, [x, y])
    negative_mean = lambda self, x, y: self.op(OpKind.NegativeMean, [x, y])
    reduce_sum = lambda self, xs: self.op(OpKind.AddVarying, xs)
    reduce_sub = lambda self, xs: self.op(OpKind.SubVarying, xs)
    reduce_mul = lambda self, xs: self.op(OpKind.MulVarying, xs)
    reduce_mean = lambda self, xs: self.op(OpKind.MeanVarying, xs)
    reduce_sum_of_squares = lambda self, xs: self.op(OpKind.SumOfSquaresVarying, xs)
    reduce_mean_squares = lambda self, xs: self.op(OpKind.MeanSquaresVarying, xs)
    reduce_negative_mean = lambda self, xs: self.op(OpKind.NegativeMeanVarying, xs)
    stopgrad_max = lambda self, xs: self.op(OpKind.StopGradMax, xs)

    def mul_by_constant(self, x, c):
        return self.op(OpKind.MulByConst, [x], c)

    def inner_product(self, xs, ys):
        if len(xs) == 0:
            raise _lib.InvalidArgument(1, "innerProduct: empty input sequence")
        if len(xs) != len(ys):
            raise _lib.InvalidArgument(1, f"innerProduct: sequence lengths differ ({len(xs)} vs {len(ys)})")
        return self.op(OpKind.InnerProductNoBias, list(xs) + list(ys))

    def inner_product_with_bias(self, xs, ys, b):
        if len(xs) == 0:
            raise _lib.InvalidArgument(1, "innerProductWithBias: empty input sequence")
        if len(xs) != len(ys):
            raise _lib.InvalidArgument(1, f"innerProductWithBias: sequence lengths differ ({len(xs)} vs {len(ys)})")
        return self.op(OpKind.InnerProductWithBias, list(xs) + list(ys) + [b])

    def value_of(self, ref: int) -> float:
        out = C.c_double()
        check(lib.tg_rec_value(self._h, int(ref), C.byref(out)))
        return out.value

    def set_root(self, ref: int) -> None:
        check(lib.tg_rec_set_root(self._h, int(ref)))

    def describe(self) -> TapeDesc:
        d = _lib.tg_tape_desc()
        check(lib.tg_rec_describe(self._h, C.byref(d)))
        return _desc_from_c(d)


def _args(model: int, dims, dtype: str) -> _lib.tg_model_args:
    a = _lib.tg_model_args()
    for i, v in enumerate(dims or []):
        a.dims[i] = int(v)
    a.dtype = _DT[dtype]
    return a


def build_model(model, dims=None, dtype: str | None = None, seed: int = 0) -> Tape:
    """Records one template sample of a built-in workload (tg_build_model)."""
    m = model_id(model)
    dtype = dtype or DEFAULT_DTYPE[m]
    h = C.c_void_p()
    check(lib.tg_build_model(m, C.byref(_args(m, dims, dtype)), int(seed), C.byref(h)))
    return Tape(dtype=dtype, _handle=h)


def io_shape(desc: TapeDesc):
    return desc.n_inputs, desc.n_index_inputs


def synth_batch(model, dims=None, dtype: str | None = None, seed: int = 0, batch: int = 1,
                n_inputs: int | None = None, n_index: int | None = None):
    """Host synthetic batch [col][batch] (inputs, int32 index inputs)."""
    m = model_id(model)
    dtype = dtype or DEFAULT_DTYPE[m]
    if n_inputs is None or n_index is None:
        d = build_model(m, dims, dtype, seed=0).describe()
        n_inputs, n_index = d.n_inputs, d.n_index_inputs
    x = np.zeros((max(n_inputs, 1), batch), _NP[dtype])
    k = np.zeros((max(n_index, 1), batch), np.int32)
    check(lib.tg_synth_batch(m, C.byref(_args(m, dims, dtype)), int(seed), int(batch),
                             x.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.POINTER(C.c_int32))))
    return x[:n_inputs], k[:n_index]


def _io_cols(m, dims, dtype, n_inputs, n_index):
    if n_inputs is None or n_index is None:
        d = build_model(m, dims, dtype, seed=0).describe()
        n_inputs, n_index = d.n_inputs, d.n_index_inputs
    return n_inputs, n_index


def synth_ctr(model, dims=None, dtype: str | None = None, seed: int = 0, first: int = 0, batch: int = 1,
              n_inputs: int | None = None, n_index: int | None = None):
    """Host counter-based batch of samples [first, first + batch) (tg_synth_ctr):
    the bits synth_ctr_device writes on the GPU."""
    m = model_id(model)
    dtype = dtype or DEFAULT_DTYPE[m]
    n_inputs, n_index = _io_cols(m, dims, dtype, n_inputs, n_index)
    x = np.zeros((max(n_inputs, 1), batch), _NP[dtype])
    k = np.zeros((max(n_index, 1), batch), np.int32)
    check(lib.tg_synth_ctr(m, C.byref(_args(m, dims, dtype)), int(seed), int(first), int(batch),
                           x.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.POINTER(C.c_int32))))
    return x[:n_inputs], k[:n_index]


def synth_ctr_device(model, x, k, dims=None, dtype: str | None = None, seed: int = 0, first: int = 0,
                     batch: int | None = None, stream=None):
    """Writes samples [first, first + batch) into device tensors x [n_inputs][batch]
    and k [n_index][batch] (either may be None when the model has no such columns)
    on `stream` (tg_synth_ctr_device)."""
    import torch
    m = model_id(model)
    dtype = dtype or DEFAULT_DTYPE[m]
    if batch is None:
        batch = (x if x is not None else k).shape[-1]
    s = stream if stream is not None else torch.cuda.current_stream()
    check(lib.tg_synth_ctr_device(m, C.byref(_args(m, dims, dtype)), int(seed), int(first), int(batch),
                                  None if x is None else C.c_void_p(x.data_ptr()),
                                  None if k is None else C.cast(C.c_void_p(k.data_ptr()), C.POINTER(C.c_int32)),
                                  C.c_void_p(s.cuda_stream)))


class Program:
    """A compiled tape: batch forward/backward + GD on the GPU (tg_compile)."""

    def __init__(self, desc: TapeDesc | Tape):
        if isinstance(desc, Tape):
            desc = desc.describe()
        self.desc = desc
        cd = desc.to_c()
        h = C.c_void_p()
        check(lib.tg_compile(C.byref(cd), C.byref(h)))
        self._h = h
        self.dtype = desc.dtype

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and lib is not None:
            lib.tg_program_free(h)
            self._h = None

    @property
    def info(self) -> dict:
        i = _lib.tg_program_info()
        check(lib.tg_program_info_get(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    def order(self) -> np.ndarray:
        p = C.POINTER(C.c_uint32)()
        n = C.c_uint32()
        check(lib.tg_program_order(self._h, C.byref(p), C.byref(n)))
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0, np.uint32)

    def workspace_size(self, batch: int) -> int:
        out = C.c_size_t()
        check(lib.tg_workspace_size(self._h, int(batch), C.byref(out)))
        return out.value

    def set_memory_budget(self, nbytes: int) -> None:
        """Sequential-accumulation mode: staged rows of at most `nbytes` per chunk (0: default)."""
        check(lib.tg_set_memory_budget(self._h, int(nbytes)))

    def chunk_samples(self, batch: int) -> int:
        out = C.c_size_t()
        check(lib.tg_chunk_samples(self._h, int(batch), C.byref(out)))
        return out.value

    @property
    def launches(self) -> int:
        return int(lib.tg_launch_count(self._h))

    # ---- device calls (torch tensors; plumbing only) ----
    @staticmethod
    def _ptr(t):
        return None if t is None else C.c_void_p(t.data_ptr())

    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def alloc_workspace(self, batch: int):
        import torch
        return torch.empty(max(self.workspace_size(batch), 1), dtype=torch.uint8, device="cuda")

    def forward_backward(self, inputs, index_inputs, batch, params, loss=None, input_grad=None, grad_sum=None,
                         workspace=None, stream=None):
        if workspace is None:
            workspace = self.alloc_workspace(batch)
        check(lib.tg_forward_backward(self._h, self._ptr(inputs), self._ptr(index_inputs), int(batch),
                                      self._ptr(params), self._ptr(loss), self._ptr(input_grad),
                                      self._ptr(grad_sum), self._ptr(workspace), workspace.numel(),
                                      self._stream(stream)))

    def gd_update(self, params, grad_sum, gamma: float, global_batch: int, stream=None):
        check(lib.tg_gd_update(self._h, self._ptr(params), self._ptr(grad_sum), float(gamma),
                               int(global_batch), self._stream(stream)))

    def allreduce_gd_step(self, params, grad_sum, gamma: float, global_batch: int, comm=None, stream=None):
        """In-place NCCL all-reduce (sum) of grad_sum, then the GD update with the
        global batch (tg_allreduce_gd_step); comm None: the update only."""
        c = None if comm is None else C.c_void_p(comm.handle if hasattr(comm, "handle") else int(comm))
        check(lib.tg_allreduce_gd_step(self._h, self._ptr(params), self._ptr(grad_sum), float(gamma),
                                       int(global_batch), c, self._stream(stream)))

    def train_step(self, inputs, index_inputs, batch, params, loss, grad_sum, gamma, workspace, stream=None):
        check(lib.tg_train_step(self._h, self._ptr(inputs), self._ptr(index_inputs), int(batch),
                                self._ptr(params), self._ptr(loss), self._ptr(grad_sum), float(gamma),
                                self._ptr(workspace), workspace.numel(), self._stream(stream)))

    def pipeline(self, batch: int, params, stream=None) -> "Pipeline":
        """Host-buffer training loop with overlapped copies (tg_pipeline_new)."""
        return Pipeline(self, batch, params, stream)

    def jit(self):
        """(source, log, compile_ms) of the register-resident kernel, or None."""
        src, log, ms = C.c_char_p(), C.c_char_p(), C.c_double()
        st = lib.tg_program_jit(self._h, C.byref(src), C.byref(log), C.byref(ms))
        if st == 9:
            return None
        check(st)
        return src.value.decode(), log.value.decode(), ms.value

    def profile(self, on: bool = True):
        check(lib.tg_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        """(total ms, launches) of the tape kernel since the last read."""
        ms, n = C.c_double(), C.c_uint64()
        check(lib.tg_profile_read(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def check_device_error(self, stream=None):
        """Raises DomainError for the first per-sample domain violation."""
        s = C.c_int64(-1)
        n = C.c_uint32(0)
        st = lib.tg_check_device_error(self._h, self._stream(stream), C.byref(s), C.byref(n))
        if st != 0:
            msg = lib.tg_last_error().decode()
            err = _lib.DomainError(st, msg) if st == 5 else _lib.TgError(st, msg)
            err.sample, err.node = s.value, n.value
            raise err


class Pipeline:
    """The reference's training loop over host buffers (tg_pipeline_*).

    Each step() takes that step's samples from host memory (numpy arrays or
    pinned torch tensors: inputs [n_inputs, batch], index_inputs
    [n_index_inputs, batch]) and writes its per-sample losses to a host array.
    Parameters stay on the device and are updated in place.  Up to four steps
    are in flight: a host buffer passed to step i may be reused after step i+4
    is submitted or after sync()."""

    def __init__(self, prog: Program, batch: int, params, stream=None):
        self.prog = prog
        self.batch = int(batch)
        self._params = params   # keep the device tensor alive
        h = C.c_void_p()
        check(lib.tg_pipeline_new(prog._h, self.batch, Program._ptr(params), Program._stream(stream), C.byref(h)))
        self._h = h

    @staticmethod
    def _host(a):
        if a is None:
            return None
        if isinstance(a, np.ndarray):
            if not a.flags["C_CONTIGUOUS"]:
                raise ValueError("host buffers must be C-contiguous")
            return C.c_void_p(a.ctypes.data)
        if a.is_cuda:
            raise ValueError("Pipeline.step takes host buffers")
        return C.c_void_p(a.data_ptr())

    def step(self, inputs, index_inputs, loss, gamma: float) -> None:
        check(lib.tg_pipeline_step(self._h, self._host(inputs), self._host(index_inputs), self._host(loss),
                                   float(gamma)))

    def join(self, stream=None) -> None:
        """Makes `stream` wait for every enqueued step (no host block)."""
        check(lib.tg_pipeline_join(self._h, Program._stream(stream)))

    def sync(self) -> None:
        check(lib.tg_pipeline_sync(self._h))

    def grad_sum_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.tg_pipeline_grad_sum(self._h, C.byref(p)))
        return p.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and lib is not None:
            lib.tg_pipeline_free(h)
            self._h = None
