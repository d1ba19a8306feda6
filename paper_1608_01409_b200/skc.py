"""ctypes binding of libskc (include/skc.h) -- argument marshalling only.

Every step of the hot path runs in libskc's CUDA kernels; this module converts NumPy
arrays / torch CUDA tensors to pointers and raises on error statuses.  There is no CPU
fallback: if libskc.so is missing or a call fails, it raises.

Names mirror the C-ABI: skc_pack_csr, skc_pad_input, skc_sparse_conv_forward, ...
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libskc.so")

SKC_KERNEL_AUTO, SKC_KERNEL_DIRECT, SKC_KERNEL_REGTILE, SKC_KERNEL_JIT, SKC_KERNEL_SPMDM = 0, 1, 2, 3, 4
SKC_LAYOUT_NCHW, SKC_LAYOUT_PAIRS, SKC_LAYOUT_RAW = 0, 1, 2
STATUS = {0: "SKC_OK", -1: "SKC_ERR_ARG", -2: "SKC_ERR_GEOMETRY", -3: "SKC_ERR_NONFINITE",
          -4: "SKC_ERR_OVERFLOW", -5: "SKC_ERR_UNSUPPORTED", -6: "SKC_ERR_ALIGN",
          -7: "SKC_ERR_STATE", -8: "SKC_ERR_CUDA"}

# Every symbol include/skc.h declares (checked by tests/test_abi.py).
EXPORTS = ("skc_pack_csr", "skc_pack_csr_ex", "skc_pack_csr_batch", "skc_plan_info", "skc_plan_csr", "skc_plan_perm",
           "skc_plan_upload", "skc_pad_input", "skc_sparse_conv_forward", "skc_forward_host",
           "skc_layout_offset", "skc_plan_destroy", "skc_last_error", "skc_model_layer_cost",
           "skc_model_project", "skc_model_window", "skc_bench_ffma", "skc_bench_lds",
           "skc_plan_verify", "skc_sparse_conv_forward_ex", "skc_im2col", "skc_im2col_ex", "skc_pack_fc",
           "skc_plan_compile", "skc_sparse_conv_forward_into", "skc_plan_tune",
           "skc_sm_topology", "skc_bench_ffma2", "skc_bench_lds64")


class SkcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class skc_info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("K", "C", "R", "S", "H", "W", "stride", "pad", "groups", "Ho", "Wo", "Hp", "Wp")] + [
        ("nnz", ctypes.c_int64), ("padded_elems_per_image", ctypes.c_size_t),
        ("out_elems_per_image", ctypes.c_size_t), ("device_bytes", ctypes.c_size_t),
        ("kernel", ctypes.c_int), ("band_rows", ctypes.c_int), ("chunk_channels", ctypes.c_int),
        ("stages", ctypes.c_int), ("warps", ctypes.c_int), ("channels_per_warp", ctypes.c_int),
        ("pixels_per_lane", ctypes.c_int), ("smem_bytes", ctypes.c_size_t),
        ("lane_mapping", ctypes.c_int), ("tile_h", ctypes.c_int), ("tile_w", ctypes.c_int),
        ("images_per_cta", ctypes.c_int), ("jit_blocks", ctypes.c_int),
        ("jit_compiled", ctypes.c_int), ("jit_cache_hit", ctypes.c_int),
        ("jit_compile_s", ctypes.c_double), ("code_bytes", ctypes.c_size_t),
        ("model_instr_per_image", ctypes.c_double), ("layout", ctypes.c_int), ("bands", ctypes.c_int), ("jit_whole", ctypes.c_int),
        ("jit_split", ctypes.c_int), ("jit_sched", ctypes.c_int), ("jit_np", ctypes.c_int),
        ("jit_deal", ctypes.c_int)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class skc_layer_cost(ctypes.Structure):
    _fields_ = [("C", ctypes.c_double), ("S_A", ctypes.c_double), ("S_W", ctypes.c_double)]


class skc_platform(ctypes.Structure):
    _fields_ = [("F", ctypes.c_double), ("B", ctypes.c_double), ("alpha", ctypes.c_double),
                ("beta", ctypes.c_double)]


class skc_projection(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("t_dense", "t_sparse_compute", "t_sparse_bw",
                                               "t_sparse", "speedup", "effective_flops",
                                               "actual_flops")]


class skc_window(ctypes.Structure):
    _fields_ = [("x_lo", ctypes.c_double), ("x_hi", ctypes.c_double),
                ("has_speedup_potential", ctypes.c_int)]


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int


def lib():
    """Load libskc.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1608_01409_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "skc_pack_csr": [_P] + [_I] * 9 + [ctypes.POINTER(_P)],
            "skc_pack_csr_ex": [_P] + [_I] * 10 + [ctypes.POINTER(_P)],
            "skc_pack_csr_batch": [_P] + [_I] * 11 + [ctypes.POINTER(_P)],
            "skc_plan_info": [_P, ctypes.POINTER(skc_info)],
            "skc_plan_verify": [_P],
            "skc_plan_compile": [_P],
            "skc_plan_tune": [_P, _I, _P, _P, _P, ctypes.c_size_t, _P, ctypes.POINTER(ctypes.c_double)],
            "skc_sm_topology": [ctypes.POINTER(_I), _I, ctypes.POINTER(_I)],
            "skc_plan_csr": [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)],
            "skc_plan_perm": [_P, ctypes.POINTER(_P)],
            "skc_plan_upload": [_P, _P, ctypes.c_size_t, _P],
            "skc_pad_input": [_P, _P, _P, _I, _P],
            "skc_sparse_conv_forward": [_P, _P, _P, _I, _P],
            "skc_sparse_conv_forward_ex": [_P, _P, _P, _I, _P, _I, _I, _P],
            "skc_sparse_conv_forward_into": [_P, _P, _P, _P, _I, _P, _I, _P],
            "skc_im2col": [_P, _P, _P, _I, _P],
            "skc_im2col_ex": [_P, _P, _P, _I, _I, _P],
            "skc_pack_fc": [_P, _I, _I, _I, _I, ctypes.POINTER(_P)],
            "skc_forward_host": [_P, _P, _P, _I, _P, _P, _P, _P],
            "skc_model_layer_cost": [_I] * 9 + [ctypes.c_int64, _I, ctypes.POINTER(skc_layer_cost)],
            "skc_model_project": [ctypes.POINTER(skc_layer_cost), ctypes.c_double,
                                  ctypes.POINTER(skc_platform), ctypes.POINTER(skc_projection)],
            "skc_model_window": [ctypes.POINTER(skc_layer_cost), ctypes.POINTER(skc_platform),
                                 ctypes.POINTER(skc_window)],
            "skc_bench_ffma": [_P, _I, _I, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)],
            "skc_bench_lds": [_P, _I, _I, ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_double)],
            "skc_bench_ffma2": [_P, _I, _I, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double)],
            "skc_bench_lds64": [_P, _I, _I, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.skc_layout_offset.argtypes = [_P, _I, _I, _I]
        L.skc_layout_offset.restype = ctypes.c_int64
        L.skc_plan_destroy.argtypes = [_P]
        L.skc_plan_destroy.restype = None
        L.skc_last_error.argtypes = []
        L.skc_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise SkcError(status, lib().skc_last_error().decode())


def _dptr(t) -> int:
    """Device pointer of a contiguous CUDA tensor (or an int pointer)."""
    if isinstance(t, int):
        return t
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """Owns one skc_plan* (host arrays) and, after upload(), its device workspace tensor."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        self.workspace = None

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.skc_plan_destroy(h)
            self._h = ctypes.c_void_p(0)

    def info(self) -> dict:
        i = skc_info()
        _check(lib().skc_plan_info(self._h, ctypes.byref(i)))
        return i.as_dict()

    def csr(self):
        """Canonical CSR copied out as NumPy arrays (rowptr int32, colidx int32, values f32)."""
        inf = self.info()
        rp, ci, va = _P(), _P(), _P()
        _check(lib().skc_plan_csr(self._h, ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(va)))
        K, nnz = inf["K"], inf["nnz"]
        rowptr = np.ctypeslib.as_array(ctypes.cast(rp, ctypes.POINTER(ctypes.c_int32)), (K + 1,)).copy()
        if nnz:
            colidx = np.ctypeslib.as_array(ctypes.cast(ci, ctypes.POINTER(ctypes.c_int32)), (nnz,)).copy()
            values = np.ctypeslib.as_array(ctypes.cast(va, ctypes.POINTER(ctypes.c_float)), (nnz,)).copy()
        else:
            colidx, values = np.zeros(0, np.int32), np.zeros(0, np.float32)
        return rowptr, colidx, values

    def perm(self) -> np.ndarray:
        K = self.info()["K"]
        pp = _P()
        _check(lib().skc_plan_perm(self._h, ctypes.byref(pp)))
        return np.ctypeslib.as_array(ctypes.cast(pp, ctypes.POINTER(ctypes.c_int32)), (K,)).copy()

    def upload(self, device=None, stream=None):
        """Allocate the workspace as a torch uint8 CUDA tensor and copy the plan into it."""
        import torch
        nbytes = self.info()["device_bytes"]
        ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device or "cuda")
        skc_plan_upload(self, ws, stream)
        self.workspace = ws
        return ws


# ------------------------------------------------------------------ C-ABI mirrors
def skc_pack_csr(w: np.ndarray, H: int, W: int, stride: int = 1, pad: int = 0, groups: int = 1,
                 kernel: int = SKC_KERNEL_AUTO, batch_hint: int = None) -> Plan:
    """a1: pruned dense weights float32 [K, C/g, R, S] (host) -> Plan, configured for
    batch_hint images per forward call (None: skc_pack_csr_ex's default, 256)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    K, Cg, R, S = w.shape
    h = _P()
    if batch_hint is None:
        _check(lib().skc_pack_csr_ex(w.ctypes.data, K, Cg * groups, R, S, H, W, stride, pad, groups,
                                     kernel, ctypes.byref(h)))
    else:
        _check(lib().skc_pack_csr_batch(w.ctypes.data, K, Cg * groups, R, S, H, W, stride, pad,
                                        groups, kernel, int(batch_hint), ctypes.byref(h)))
    return Plan(h.value)


def skc_plan_verify(plan: Plan):
    """Static self-check of the plan's kernel-private data (raises SkcError on a violation)."""
    _check(lib().skc_plan_verify(plan.handle))


def skc_plan_compile(plan: Plan):
    """JIT kernel: generate + compile + link the plan's code now (host only, no GPU)."""
    _check(lib().skc_plan_compile(plan.handle))


def skc_sm_topology(cap: int = 1024):
    """GPC-major SM order of the current device: list vid[smid] (diagnostic)."""
    arr = (ctypes.c_int * cap)()
    n = ctypes.c_int(0)
    _check(lib().skc_sm_topology(arr, cap, ctypes.byref(n)))
    return list(arr[:n.value])


def skc_plan_tune(plan: Plan, N: int, d_in, d_out, d_flush=None, stream=None) -> float:
    """JIT kernel: time the launch-schedule variants on caller-owned scratch of N images
    (d_in: padded input in the plan's layout, d_out: output, d_flush: optional buffer larger
    than L2 written before every timed launch), keep the fastest; returns its time in ms
    (0.0 for other kernels).  Outputs are bitwise unaffected."""
    ms = ctypes.c_double(0.0)
    fl = _dptr(d_flush) if d_flush is not None else None
    nfl = d_flush.numel() * d_flush.element_size() if d_flush is not None else 0
    _check(lib().skc_plan_tune(plan.handle, int(N), _dptr(d_in), _dptr(d_out), fl, nfl,
                               _stream(stream), ctypes.byref(ms)))
    return ms.value


def skc_plan_upload(plan: Plan, workspace, stream=None):
    _check(lib().skc_plan_upload(plan.handle, _dptr(workspace), workspace.numel(), _stream(stream)))


def skc_pad_input(plan: Plan, d_in, d_in_padded, N: int, stream=None):
    """a2: NCHW -> [N, C, Hp, Wp] with a zero border (CUDA kernel)."""
    _check(lib().skc_pad_input(plan.handle, _dptr(d_in), _dptr(d_in_padded), int(N), _stream(stream)))


def skc_sparse_conv_forward(plan: Plan, d_in_padded, d_out, N: int, stream=None):
    """a3..a6: the direct sparse convolution (CUDA kernel)."""
    _check(lib().skc_sparse_conv_forward(plan.handle, _dptr(d_in_padded), _dptr(d_out), int(N),
                                         _stream(stream)))


def skc_sparse_conv_forward_ex(plan: Plan, d_in_padded, d_out, N: int, d_bias=None,
                               relu: bool = False, out_pad: int = 0, stream=None):
    """f1: conv + bias + ReLU written into the interior of an out_pad-wide padded output."""
    _check(lib().skc_sparse_conv_forward_ex(plan.handle, _dptr(d_in_padded), _dptr(d_out), int(N),
                                            _dptr(d_bias) if d_bias is not None else None,
                                            int(bool(relu)), int(out_pad), _stream(stream)))


def skc_sparse_conv_forward_into(plan: Plan, d_in_padded, next_plan: Plan, d_next_in, N: int,
                                 d_bias=None, relu: bool = False, stream=None):
    """f1 chain: conv + bias + ReLU written into the next plan's padded input (its layout)."""
    _check(lib().skc_sparse_conv_forward_into(plan.handle, _dptr(d_in_padded), next_plan.handle,
                                              _dptr(d_next_in), int(N),
                                              _dptr(d_bias) if d_bias is not None else None,
                                              int(bool(relu)), _stream(stream)))


def padded_shape(info: dict, N: int) -> tuple:
    """Shape of the padded-input buffer of N images in the plan's layout (skc_info.layout)."""
    if info["layout"] == SKC_LAYOUT_PAIRS:
        return ((N + 1) // 2, info["C"], info["Hp"], info["Wp"], 2)
    if info["layout"] == SKC_LAYOUT_RAW:  # unpadded: the kernel pads while staging
        return (N, info["C"], info["H"], info["W"])
    return (N, info["C"], info["Hp"], info["Wp"])


def unpad_view(info: dict, xp, N: int):
    """NCHW-padded view [N][C][Hp][Wp] (a copy for the pair layout) of a padded buffer."""
    if info["layout"] == SKC_LAYOUT_PAIRS:
        return xp.movedim(-1, 1).reshape(-1, *xp.shape[1:4])[:N]
    return xp


def skc_im2col(plan: Plan, d_in, d_lowered, N: int, stream=None):
    """f3: lowered (im2col) tensor [N][C*R*S][Ho][Wo] of an NCHW input (CUDA kernel)."""
    _check(lib().skc_im2col(plan.handle, _dptr(d_in), _dptr(d_lowered), int(N), _stream(stream)))


def skc_im2col_ex(plan: Plan, d_in, d_lowered, N: int, layout: int, stream=None):
    """f3: the lowered tensor in layout SKC_LAYOUT_NCHW or SKC_LAYOUT_PAIRS (the padded layout
    of a JIT 1x1 plan over it)."""
    _check(lib().skc_im2col_ex(plan.handle, _dptr(d_in), _dptr(d_lowered), int(N), int(layout),
                               _stream(stream)))


def skc_pack_fc(w: np.ndarray, batch: int, kernel: int = SKC_KERNEL_AUTO) -> Plan:
    """f2: pruned FC weights float32 [M, K] -> plan for Y[M x B] = W X[K x B] (B = batch)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    M, K = w.shape
    h = _P()
    _check(lib().skc_pack_fc(w.ctypes.data, M, K, int(batch), kernel, ctypes.byref(h)))
    return Plan(h.value)


class SparseLinear:
    """f2: a pruned FC layer on the GPU, Y[M x B] = W[M x K] X[K x B] (batch-minor layout)."""

    def __init__(self, w: np.ndarray, batch: int, kernel=SKC_KERNEL_AUTO, device="cuda"):
        self.plan = skc_pack_fc(w, batch, kernel)
        self.plan.upload(device)
        self.M, self.K, self.B = w.shape[0], w.shape[1], int(batch)

    def forward(self, x, out=None, bias=None, relu=False, stream=None):
        import torch
        if tuple(x.shape) != (self.K, self.B):
            raise ValueError(f"expected X of shape {(self.K, self.B)}")
        if out is None:
            out = torch.empty((self.M, self.B), dtype=torch.float32, device=x.device)
        skc_sparse_conv_forward_ex(self.plan, x, out, 1, bias, relu, 0, stream)
        return out


class LoweredSparseConv2d:
    """f3 baseline: im2col + CSR SpMDM (a 1x1 conv over the lowered tensor, with the direct
    kernel by default or the compiled-weights kernel with kernel=SKC_KERNEL_AUTO, whose
    image-pair layout im2col then writes directly).  Same weights, same nonzero order as
    SparseConv2d -> identical results."""

    def __init__(self, w: np.ndarray, H: int, W: int, stride=1, pad=0, groups=1,
                 kernel=SKC_KERNEL_DIRECT, device="cuda"):
        K, Cg, R, S = w.shape
        self.geom_plan = skc_pack_csr(w, H, W, stride, pad, groups, SKC_KERNEL_DIRECT)
        g = self.geom_plan.info()
        self.Ho, self.Wo, self.K, self.CRS = g["Ho"], g["Wo"], K, g["C"] * R * S
        w1 = np.ascontiguousarray(w.reshape(K, Cg * R * S, 1, 1))
        self.conv = SparseConv2d.from_dense(w1, self.Ho, self.Wo, 1, 0, groups, kernel, device)

    def _layout(self):
        return SKC_LAYOUT_PAIRS if self.conv.geom["layout"] == SKC_LAYOUT_PAIRS else SKC_LAYOUT_NCHW

    def lowered_shape(self, N):
        if self._layout() == SKC_LAYOUT_PAIRS:
            return ((N + 1) // 2, self.CRS, self.Ho, self.Wo, 2)
        return (N, self.CRS, self.Ho, self.Wo)

    def forward(self, x, lowered=None, out=None, stream=None):
        import torch
        N = x.shape[0]
        if lowered is None:
            lowered = torch.empty(self.lowered_shape(N), dtype=torch.float32, device=x.device)
        skc_im2col_ex(self.geom_plan, x, lowered, N, self._layout(), stream)
        return self.conv.forward_padded(lowered, out, stream, N=N)


def skc_forward_host(plan: Plan, h_in, h_out, N: int, d_in, d_pad, d_out, stream=None):
    """H2D + pad + conv + D2H on one stream; h_in/h_out are (pinned) CPU tensors."""
    _check(lib().skc_forward_host(plan.handle, h_in.data_ptr(), h_out.data_ptr(), int(N),
                                  _dptr(d_in), _dptr(d_pad), _dptr(d_out), _stream(stream)))


def skc_layout_offset(plan: Plan, c: int, y: int, x: int) -> int:
    return int(lib().skc_layout_offset(plan.handle, c, y, x))


def skc_model_layer_cost(K, C, R, S, H, W, stride=1, pad=0, groups=1, batch=1, amortised=False):
    out = skc_layer_cost()
    _check(lib().skc_model_layer_cost(K, C, R, S, H, W, stride, pad, groups, int(batch),
                                      int(bool(amortised)), ctypes.byref(out)))
    return dict(C=out.C, S_A=out.S_A, S_W=out.S_W)


def skc_model_project(cost: dict, x: float, F: float, B: float, alpha: float, beta: float = 2.0):
    c = skc_layer_cost(cost["C"], cost["S_A"], cost["S_W"])
    p = skc_platform(F, B, alpha, beta)
    o = skc_projection()
    _check(lib().skc_model_project(ctypes.byref(c), float(x), ctypes.byref(p), ctypes.byref(o)))
    return {n: getattr(o, n) for n, _ in o._fields_}


def skc_model_window(cost: dict, F: float, B: float, alpha: float, beta: float = 2.0):
    c = skc_layer_cost(cost["C"], cost["S_A"], cost["S_W"])
    p = skc_platform(F, B, alpha, beta)
    o = skc_window()
    _check(lib().skc_model_window(ctypes.byref(c), ctypes.byref(p), ctypes.byref(o)))
    return dict(x_lo=o.x_lo, x_hi=o.x_hi, has_speedup_potential=bool(o.has_speedup_potential))


def skc_bench_ffma(scratch, blocks: int, iters: int):
    ms, fl = ctypes.c_double(), ctypes.c_double()
    _check(lib().skc_bench_ffma(_dptr(scratch), blocks, iters, ctypes.byref(ms), ctypes.byref(fl)))
    return ms.value, fl.value


def skc_bench_lds(scratch, blocks: int, iters: int):
    ms, by = ctypes.c_double(), ctypes.c_double()
    _check(lib().skc_bench_lds(_dptr(scratch), blocks, iters, ctypes.byref(ms), ctypes.byref(by)))
    return ms.value, by.value


def skc_bench_ffma2(scratch, blocks: int, iters: int):
    ms, fl = ctypes.c_double(), ctypes.c_double()
    _check(lib().skc_bench_ffma2(_dptr(scratch), blocks, iters, ctypes.byref(ms), ctypes.byref(fl)))
    return ms.value, fl.value


def skc_bench_lds64(scratch, blocks: int, iters: int):
    ms, by = ctypes.c_double(), ctypes.c_double()
    _check(lib().skc_bench_lds64(_dptr(scratch), blocks, iters, ctypes.byref(ms), ctypes.byref(by)))
    return ms.value, by.value


# ------------------------------------------------------------------ convenience layer
@dataclass
class SparseConv2d:
    """One pruned conv layer on the GPU: plan + workspace + padded-input scratch.

    forward(x) runs skc_pad_input then skc_sparse_conv_forward on the current stream."""
    plan: Plan
    geom: dict

    @classmethod
    def from_dense(cls, w: np.ndarray, H: int, W: int, stride=1, pad=0, groups=1,
                   kernel=SKC_KERNEL_AUTO, device="cuda", batch_hint=None):
        plan = skc_pack_csr(w, H, W, stride, pad, groups, kernel, batch_hint)
        plan.upload(device)
        return cls(plan, plan.info())

    @classmethod
    def from_plan(cls, plan: Plan, device="cuda"):
        """Wrap an already packed (and possibly already compiled) plan; uploads it."""
        plan.upload(device)
        return cls(plan, plan.info())

    def out_shape(self, N):
        g = self.geom
        return (N, g["K"], g["Ho"], g["Wo"])

    def padded_shape(self, N):
        """Padded-input buffer shape in the plan's layout (NCHW, or image pairs)."""
        return padded_shape(self.geom, N)

    def tune(self, N: int = 256, stream=None, flush=True) -> float:
        """JIT plans: pick the fastest launch schedule for batches of N on this device
        (skc_plan_tune, on scratch buffers allocated here as torch tensors); returns the
        chosen variant's time in ms (0.0 for other kernels)."""
        import torch
        if self.geom["kernel"] != SKC_KERNEL_JIT:
            return 0.0
        dev = self.plan.workspace.device
        xp = torch.zeros(self.padded_shape(N), dtype=torch.float32, device=dev)
        out = torch.empty(self.out_shape(N), dtype=torch.float32, device=dev)
        fl = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
        return skc_plan_tune(self.plan, N, xp, out, fl, stream)

    def forward_padded(self, xp, out=None, stream=None, N=None):
        """Conv of a padded input in the plan's layout.  N defaults to out's batch, else to
        the padded buffer's images (2 per leading index in the image-pair layout)."""
        import torch
        if N is None:
            if out is not None:
                N = out.shape[0]
            else:
                N = xp.shape[0] * (2 if self.geom["layout"] == SKC_LAYOUT_PAIRS else 1)
        if out is None:
            out = torch.empty(self.out_shape(N), dtype=torch.float32, device=xp.device)
        skc_sparse_conv_forward(self.plan, xp, out, N, stream)
        return out

    def forward(self, x, xp=None, out=None, stream=None):
        import torch
        N = x.shape[0]
        if xp is None:
            if self.geom["layout"] == SKC_LAYOUT_RAW and x.is_contiguous():
                xp = x  # the kernel pads while staging
            else:
                xp = torch.empty(self.padded_shape(N), dtype=torch.float32, device=x.device)
        skc_pad_input(self.plan, x, xp, N, stream)
        return self.forward_padded(xp, out, stream, N)
