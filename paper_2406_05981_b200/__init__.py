"""B200-native ShiftAddLLM LUT-GEMV hot path (arxiv 2406.05981) -- thin Python binding.

Every step of the path runs in the CUDA kernels of ``libshiftadd.so`` (built from ``csrc/``
for sm_100a by ``__graft_entry__.build()``) behind the C ABI declared in
``include/shiftadd.h``.  This module only marshals arguments: torch provides device memory,
the current stream and (in ``dist``) the process group.  There is no CPU or eager fallback:
if the library is missing or the device is not sm_100a, calls raise.

    layer = pack(signs, alpha, g)          # §8 a1, on the device
    y = lut_gemm(x, layer)                 # §8 a2-a7, x: fp16 [M][K] (M <= 16) or [K]
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field

import torch

__all__ = [
    "LAYOUT_CANONICAL", "LAYOUT_TILED", "FLAG_PDL", "FLAG_SPLITK", "EXP_ZERO", "ShiftAddError", "lib",
    "PackedLayer", "packed_bytes", "pack", "lut_gemm", "lut_gemv", "workspace_bytes",
    "gemm_plan", "Workspace", "pack_colwise", "lut_gemv_colwise", "pack_apot2", "bcq_quantize",
    "lut_gemv_fused", "workspace_bytes_fused", "pack_blockwise", "lut_gemv_blockwise", "Program", "Chain",
    "CALL_WAIT",
]

LAYOUT_CANONICAL = 0
LAYOUT_TILED = 1
FLAG_PDL = 1
FLAG_SPLITK = 2
FLAG_CLUSTER = 4
EXP_ZERO = -128
_ABI_VERSION = 1
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libshiftadd.so")

_lib = None
_lib_lock = threading.Lock()


class ShiftAddError(RuntimeError):
    pass


class _Segment(ctypes.Structure):
    """shiftadd_segment (include/shiftadd.h)."""
    _fields_ = [("planes", ctypes.c_void_p), ("exps", ctypes.c_void_p), ("N", ctypes.c_int), ("q", ctypes.c_int),
                ("y", ctypes.c_void_p)]


class _Call(ctypes.Structure):
    """shiftadd_call (include/shiftadd.h)."""
    _fields_ = [("x", ctypes.c_void_p), ("K", ctypes.c_int), ("g", ctypes.c_int), ("nseg", ctypes.c_int),
                ("flags", ctypes.c_uint), ("seg", _Segment * 4)]


def lib():
    """Load libshiftadd.so (once) and declare its C signatures.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ShiftAddError(
                "libshiftadd.so not built (%s); run __graft_entry__.build() -- there is no "
                "fallback path" % _LIB_PATH)
        L = ctypes.CDLL(_LIB_PATH)
        c_int, c_size, vp = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
        L.shiftadd_abi_version.restype = c_int
        L.shiftadd_status_string.restype = ctypes.c_char_p
        L.shiftadd_status_string.argtypes = [c_int]
        L.shiftadd_last_error.restype = ctypes.c_char_p
        L.shiftadd_packed_bytes.restype = c_size
        L.shiftadd_packed_bytes.argtypes = [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_size)]
        L.shiftadd_pack.restype = c_int
        L.shiftadd_pack.argtypes = [vp, vp, c_int, c_int, c_int, c_int, c_int, vp, vp, vp, vp]
        L.shiftadd_workspace_bytes.restype = c_size
        L.shiftadd_workspace_bytes.argtypes = [c_int] * 6
        L.shiftadd_lut_gemm.restype = c_int
        L.shiftadd_lut_gemm.argtypes = [vp, c_int, vp, vp, c_int, c_int, c_int, c_int, c_int, c_int,
                                        vp, c_int, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_lut_gemv.restype = c_int
        L.shiftadd_lut_gemv.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, c_int, vp, vp, c_size,
                                        ctypes.c_uint, vp]
        L.shiftadd_pack_colwise.restype = c_int
        L.shiftadd_pack_colwise.argtypes = [vp, vp, c_int, c_int, c_int, c_int, vp, vp, vp, vp]
        L.shiftadd_lut_gemv_colwise.restype = c_int
        L.shiftadd_lut_gemv_colwise.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, vp, ctypes.c_uint, vp]
        L.shiftadd_workspace_bytes_colwise.restype = c_size
        L.shiftadd_workspace_bytes_colwise.argtypes = [c_int, c_int]
        L.shiftadd_lut_gemv_colwise_ws.restype = c_int
        L.shiftadd_lut_gemv_colwise_ws.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, vp, vp, c_size,
                                                   ctypes.c_uint, vp]
        L.shiftadd_lut_gemm_colwise.restype = c_int
        L.shiftadd_lut_gemm_colwise.argtypes = [vp, c_int, vp, vp, c_int, c_int, c_int, c_int, c_int, vp, c_int, vp,
                                                c_size, ctypes.c_uint, vp]
        L.shiftadd_workspace_bytes_apot2.restype = c_size
        L.shiftadd_workspace_bytes_apot2.argtypes = [c_int, c_int]
        L.shiftadd_lut_gemm_apot2_ws.restype = c_int
        L.shiftadd_lut_gemm_apot2_ws.argtypes = [vp, c_int, vp, vp, vp, c_int, c_int, c_int, c_int, c_int, c_int,
                                                 vp, c_int, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_pack_apot2.restype = c_int
        L.shiftadd_pack_apot2.argtypes = [vp, vp, c_int, c_int, c_int, c_int, c_int, vp, vp, vp, vp, vp]
        L.shiftadd_lut_gemm_apot2.restype = c_int
        L.shiftadd_lut_gemm_apot2.argtypes = [vp, c_int, vp, vp, vp, c_int, c_int, c_int, c_int, c_int, c_int,
                                              vp, c_int, ctypes.c_uint, vp]
        L.shiftadd_bcq_quantize.restype = c_int
        L.shiftadd_bcq_quantize.argtypes = [vp, c_int, c_int, c_int, c_int, c_int, ctypes.c_uint, vp, vp, vp]
        L.shiftadd_lut_gemv_gather.restype = c_int
        L.shiftadd_lut_gemv_gather.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, c_int, vp, vp, c_int, c_int,
                                               vp, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_lut_gemm_gather.restype = c_int
        L.shiftadd_lut_gemm_gather.argtypes = [vp, c_int, vp, vp, c_int, c_int, c_int, c_int, c_int, c_int, vp, vp,
                                               c_int, c_int, vp, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_gather_wait.restype = c_int
        L.shiftadd_gather_wait.argtypes = [vp, c_int, vp, vp]
        L.shiftadd_copy.restype = c_int
        L.shiftadd_copy.argtypes = [vp, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_workspace_bytes_fused.restype = c_size
        L.shiftadd_workspace_bytes_fused.argtypes = [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(_Segment)]
        L.shiftadd_lut_gemv_fused.restype = c_int
        L.shiftadd_lut_gemv_fused.argtypes = [vp, c_int, c_int, c_int, c_int, ctypes.POINTER(_Segment), vp, c_size,
                                              ctypes.c_uint, vp]
        L.shiftadd_pack_blockwise.restype = c_int
        L.shiftadd_pack_blockwise.argtypes = [vp, vp, c_int, c_int, c_int, c_int, vp, vp, vp, vp]
        L.shiftadd_workspace_bytes_blockwise.restype = c_size
        L.shiftadd_workspace_bytes_blockwise.argtypes = [c_int, c_int]
        L.shiftadd_lut_gemv_blockwise.restype = c_int
        L.shiftadd_lut_gemv_blockwise.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, vp, vp, c_size,
                                                  ctypes.c_uint, vp]
        L.shiftadd_program_bytes.restype = c_size
        L.shiftadd_program_bytes.argtypes = [c_int]
        L.shiftadd_program_encode.restype = c_int
        L.shiftadd_program_encode.argtypes = [ctypes.POINTER(_Call), c_int, vp, c_size]
        L.shiftadd_workspace_bytes_program.restype = c_size
        L.shiftadd_workspace_bytes_program.argtypes = [ctypes.POINTER(_Call), c_int]
        L.shiftadd_lut_gemv_program.restype = c_int
        L.shiftadd_lut_gemv_program.argtypes = [ctypes.POINTER(_Call), c_int, vp, c_size, vp, c_size,
                                                ctypes.c_uint, vp]
        L.shiftadd_workspace_bytes_chain.restype = c_size
        L.shiftadd_workspace_bytes_chain.argtypes = [ctypes.POINTER(_Call), c_int]
        L.shiftadd_lut_gemv_chain.restype = c_int
        L.shiftadd_lut_gemv_chain.argtypes = [ctypes.POINTER(_Call), c_int, vp, c_size, ctypes.c_uint, vp]
        L.shiftadd_gemm_plan.restype = c_int
        L.shiftadd_gemm_plan.argtypes = [c_int] * 6 + [ctypes.POINTER(c_int * 4)]
        v = L.shiftadd_abi_version()
        if v != _ABI_VERSION:
            raise ShiftAddError("libshiftadd ABI %d, binding expects %d" % (v, _ABI_VERSION))
        _lib = L
        return L


def _check(status: int, what: str):
    if status != 0:
        L = lib()
        raise ShiftAddError("%s failed: %s: %s" % (
            what, L.shiftadd_status_string(status).decode(), L.shiftadd_last_error().decode()))


def _stream_ptr(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def packed_bytes(layout: int, q: int, N: int, K: int, g: int):
    """(plane bytes, exponent bytes) of a packed layer in ``layout``."""
    e = ctypes.c_size_t(0)
    p = lib().shiftadd_packed_bytes(layout, q, N, K, g, ctypes.byref(e))
    if p == 0:
        _check(2, "packed_bytes")
    return int(p), int(e.value)


@dataclass
class PackedLayer:
    """A reparameterised linear layer on the device (output of ``pack``)."""
    planes: torch.Tensor      # uint8, layout-dependent permutation of [q][N][K/8]
    exps: torch.Tensor        # int8, layout-dependent permutation of [q][N][K/g]
    q: int
    N: int
    K: int
    g: int
    layout: int
    counts: torch.Tensor      # int32[2] on device: clamped exponents, invalid inputs
    _ws_bytes: dict = field(default_factory=dict, repr=False)   # M -> workspace bytes
    colwise: bool = False     # NEXT-f1: exps is exps_col [q][K] (column-wise scales)
    blockwise: bool = False   # NEXT-f1: exps is exps_bw [q][8][K/8] (block-wise scales, "Ours (Lat.)")
    exps2: torch.Tensor | None = None   # NEXT-f2: second additive-PoT term codes (like exps)

    @property
    def device(self):
        return self.planes.device

    def nbytes(self) -> int:
        return self.planes.numel() + self.exps.numel()


def pack(signs: torch.Tensor, alpha: torch.Tensor, g: int, layout: int = LAYOUT_TILED,
         stream=None) -> PackedLayer:
    """§8 a1 on the device: int8 sign planes [q][N][K] and fp32 scales [q][N][K/g] -> key
    bytes + PoT exponents (shiftadd_pack)."""
    if signs.dtype != torch.int8 or alpha.dtype != torch.float32:
        raise TypeError("signs must be int8 and alpha float32")
    if not (signs.is_cuda and alpha.is_cuda):
        raise ValueError("pack runs on the GPU; pass CUDA tensors")
    if signs.dim() != 3 or alpha.dim() != 3:
        raise ValueError("signs [q][N][K], alpha [q][N][K/g]")
    q, N, K = signs.shape
    if tuple(alpha.shape) != (q, N, K // g if g else 0):
        raise ValueError("alpha must be [q][N][K/g]")
    signs = signs.contiguous()
    alpha = alpha.contiguous()
    pb, eb = packed_bytes(layout, q, N, K, g)
    dev = signs.device
    planes = torch.empty(pb, dtype=torch.uint8, device=dev)
    exps = torch.empty(eb, dtype=torch.int8, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib().shiftadd_pack(_ptr(signs), _ptr(alpha), q, N, K, g, layout, _ptr(planes), _ptr(exps),
                                 _ptr(counts), _stream_ptr(stream, dev))
    _check(st, "shiftadd_pack")
    return PackedLayer(planes, exps, q, N, K, g, layout, counts)


BCQ_POT = 1


def bcq_quantize(w: torch.Tensor, q: int, g: int, T: int = 15, pot: bool = False, stream=None):
    """NEXT-f4: Alg. 1 alternating multi-bit BCQ of an fp32 weight matrix [N][K] on the device
    (shiftadd_bcq_quantize).  Returns (signs int8 [q][N][K], alpha fp32 [q][N][K/g]) -- the
    inputs of ``pack``."""
    if w.dtype != torch.float32 or not w.is_cuda or w.dim() != 2:
        raise ValueError("w must be a CUDA fp32 [N][K] tensor")
    w = w.contiguous()
    N, K = w.shape
    if g <= 0 or K % g:
        raise ValueError("g must divide K")
    signs = torch.empty((q, N, K), dtype=torch.int8, device=w.device)
    alpha = torch.empty((q, N, K // g), dtype=torch.float32, device=w.device)
    with torch.cuda.device(w.device):
        st = lib().shiftadd_bcq_quantize(_ptr(w), N, K, q, g, T, BCQ_POT if pot else 0, _ptr(signs), _ptr(alpha),
                                         _stream_ptr(stream, w.device))
    _check(st, "shiftadd_bcq_quantize")
    return signs, alpha


def pack_apot2(signs: torch.Tensor, alpha: torch.Tensor, g: int, layout: int = LAYOUT_TILED,
               stream=None) -> PackedLayer:
    """NEXT-f2: as ``pack`` plus the second additive-PoT term of every scale (K = 2,
    Eq. 2) in ``exps2`` (shiftadd_pack_apot2)."""
    if signs.dtype != torch.int8 or alpha.dtype != torch.float32:
        raise TypeError("signs must be int8 and alpha float32")
    if not (signs.is_cuda and alpha.is_cuda):
        raise ValueError("pack_apot2 runs on the GPU; pass CUDA tensors")
    if signs.dim() != 3 or alpha.dim() != 3:
        raise ValueError("signs [q][N][K], alpha [q][N][K/g]")
    q, N, K = signs.shape
    if tuple(alpha.shape) != (q, N, K // g if g else 0):
        raise ValueError("alpha must be [q][N][K/g]")
    signs = signs.contiguous()
    alpha = alpha.contiguous()
    pb, eb = packed_bytes(layout, q, N, K, g)
    dev = signs.device
    planes = torch.empty(pb, dtype=torch.uint8, device=dev)
    exps = torch.empty(eb, dtype=torch.int8, device=dev)
    exps2 = torch.empty(eb, dtype=torch.int8, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib().shiftadd_pack_apot2(_ptr(signs), _ptr(alpha), q, N, K, g, layout, _ptr(planes), _ptr(exps),
                                       _ptr(exps2), _ptr(counts), _stream_ptr(stream, dev))
    _check(st, "shiftadd_pack_apot2")
    return PackedLayer(planes, exps, q, N, K, g, layout, counts, exps2=exps2)


def pack_colwise(signs: torch.Tensor, alpha_col: torch.Tensor, layout: int = LAYOUT_TILED,
                 stream=None) -> PackedLayer:
    """NEXT-f1 on the device: int8 sign planes [q][N][K] and column-wise fp32 scales [q][K]
    -> key bytes (column signs folded) + exps_col int8 [q][K] (shiftadd_pack_colwise)."""
    if signs.dtype != torch.int8 or alpha_col.dtype != torch.float32:
        raise TypeError("signs must be int8 and alpha_col float32")
    if not (signs.is_cuda and alpha_col.is_cuda):
        raise ValueError("pack_colwise runs on the GPU; pass CUDA tensors")
    if signs.dim() != 3 or alpha_col.dim() != 2:
        raise ValueError("signs [q][N][K], alpha_col [q][K]")
    q, N, K = signs.shape
    if tuple(alpha_col.shape) != (q, K):
        raise ValueError("alpha_col must be [q][K]")
    signs = signs.contiguous()
    alpha_col = alpha_col.contiguous()
    pb, _ = packed_bytes(layout, q, N, K, K)   # plane bytes do not depend on g
    dev = signs.device
    planes = torch.empty(pb, dtype=torch.uint8, device=dev)
    exps = torch.empty(q * K, dtype=torch.int8, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib().shiftadd_pack_colwise(_ptr(signs), _ptr(alpha_col), q, N, K, layout, _ptr(planes), _ptr(exps),
                                         _ptr(counts), _stream_ptr(stream, dev))
    _check(st, "shiftadd_pack_colwise")
    return PackedLayer(planes, exps, q, N, K, K, layout, counts, colwise=True)


def pack_blockwise(signs: torch.Tensor, alpha_bw: torch.Tensor, layout: int = LAYOUT_TILED,
                   stream=None) -> PackedLayer:
    """NEXT-f1 block-wise scales ("Ours (Lat.)") on the device: int8 sign
    planes [q][N][K] and fp32 scales [q][8][K/8] (8 columns x N/8 rows per scale) -> key bytes
    (each block's sign folded) + compact exps_bw int8 [q][8][K/8] (shiftadd_pack_blockwise)."""
    if signs.dtype != torch.int8 or alpha_bw.dtype != torch.float32:
        raise TypeError("signs must be int8 and alpha_bw float32")
    if not (signs.is_cuda and alpha_bw.is_cuda):
        raise ValueError("pack_blockwise runs on the GPU; pass CUDA tensors")
    q, N, K = signs.shape
    if tuple(alpha_bw.shape) != (q, 8, K // 8):
        raise ValueError("alpha_bw must be [q][8][K/8]")
    signs = signs.contiguous()
    alpha_bw = alpha_bw.contiguous()
    pb, _ = packed_bytes(layout, q, N, K, K)
    dev = signs.device
    planes = torch.empty(pb, dtype=torch.uint8, device=dev)
    exps = torch.empty(q * K, dtype=torch.int8, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib().shiftadd_pack_blockwise(_ptr(signs), _ptr(alpha_bw), q, N, K, layout, _ptr(planes), _ptr(exps),
                                           _ptr(counts), _stream_ptr(stream, dev))
    _check(st, "shiftadd_pack_blockwise")
    return PackedLayer(planes, exps, q, N, K, 8, layout, counts, blockwise=True)


def lut_gemv_blockwise(x: torch.Tensor, layer: PackedLayer, out: torch.Tensor | None = None, pdl: bool = False,
                       workspace: Workspace | None = None, stream=None) -> torch.Tensor:
    """y = x (.) the block-wise layer, batch 1 (shiftadd_lut_gemv_blockwise)."""
    x = x.reshape(-1)
    if not layer.blockwise:
        raise ValueError("layer was not packed by pack_blockwise")
    if x.dtype != torch.float16 or not x.is_cuda or x.numel() != layer.K:
        raise ValueError("x must be fp16 [K] on the device")
    dev = layer.device
    if out is None:
        out = torch.empty(layer.N, dtype=torch.float16, device=dev)
    need = int(lib().shiftadd_workspace_bytes_blockwise(layer.N, layer.K))
    ws = (workspace or _workspace_for(dev, stream)).get(need)
    if torch.cuda.current_device() != dev.index:
        torch.cuda.set_device(dev)
    sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
    _check(lib().shiftadd_lut_gemv_blockwise(x.data_ptr(), layer.planes.data_ptr(), layer.exps.data_ptr(), layer.layout,
                                             layer.N, layer.K, layer.q, out.data_ptr(),
                                             ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
                                             FLAG_PDL if pdl else 0, sptr), "shiftadd_lut_gemv_blockwise")
    return out


def lut_gemv_colwise(x: torch.Tensor, layer: PackedLayer, out: torch.Tensor | None = None, pdl: bool = False,
                     stream=None, workspace: "Workspace | None" = None, splitk: bool = False) -> torch.Tensor:
    """NEXT-f1: y = x (.) a column-wise-scaled layer, fp16 (shiftadd_lut_gemm_colwise).  x: [K]
    or [1][K] (returns [N]) or [M][K] with M <= 16 (returns [M][N]).  M = 1: the cluster kernel for
    K <= 4096, else -- or with splitk -- the all-SM streaming kernel; M > 1: pairs of rows per
    weight pass on the streaming kernel."""
    if not layer.colwise:
        raise ValueError("layer was not packed with pack_colwise")
    vec = x.dim() == 1
    x2 = x.reshape(1, -1) if vec else x
    if x2.dtype != torch.float16 or not x2.is_cuda or x2.shape[1] != layer.K or x2.dim() != 2:
        raise ValueError("x must be fp16 [K] or [M][K] on the layer's device")
    x2 = x2.contiguous()
    M = x2.shape[0]
    if out is None:
        out = torch.empty((M, layer.N), dtype=torch.float16, device=layer.device)
    out2 = out.reshape(M, layer.N)
    if out.dtype != torch.float16 or not out.is_contiguous():
        raise ValueError("out must be contiguous fp16 [M][N]")
    dev = layer.device
    if torch.cuda.current_device() != dev.index:
        torch.cuda.set_device(dev)
    need = int(lib().shiftadd_workspace_bytes_colwise(layer.N, layer.K)) if layer.layout == LAYOUT_TILED else 0
    ws = (workspace or _workspace_for(dev, stream)).get(need)
    sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
    flags = (FLAG_PDL if pdl else 0) | (FLAG_SPLITK if splitk else 0)
    st = lib().shiftadd_lut_gemm_colwise(x2.data_ptr(), layer.K, layer.planes.data_ptr(), layer.exps.data_ptr(),
                                         layer.layout, M, layer.N, layer.K, layer.q, out2.data_ptr(), layer.N,
                                         ws.data_ptr() if ws is not None else None,
                                         ws.numel() if ws is not None else 0, flags, sptr)
    if st:
        _check(st, "shiftadd_lut_gemm_colwise")
    return out.reshape(layer.N) if M == 1 else out


def workspace_bytes(layer: PackedLayer, M: int) -> int:
    return int(lib().shiftadd_workspace_bytes(layer.layout, M, layer.N, layer.K, layer.q, layer.g))


class Workspace:
    """A zero-initialised device scratch buffer that grows on demand.  Calls leave it zeroed
    (the kernels reset their arrival counters), so it is reused without re-clearing.  Do not
    share one Workspace between calls that may run concurrently on different streams."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = None

    def get(self, nbytes: int):
        if nbytes == 0:
            return None
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws = {}


def _workspace_for(device, stream=None):
    """Default workspace of (device, launch stream): calls on different streams never share
    one (their split-K partials / epoch counters would race)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (device.index, s.cuda_stream)
    ws = _default_ws.get(key)
    if ws is None:
        ws = _default_ws[key] = Workspace(device)
    return ws


def lut_gemm(x: torch.Tensor, layer: PackedLayer, out: torch.Tensor | None = None,
             workspace: Workspace | None = None, pdl: bool = False, stream=None,
             splitk: bool = False, cluster: bool = False) -> torch.Tensor:
    """§8 a2-a7: y[M][N] = x[M][K] (.) the packed layer, fp16 in/out (shiftadd_lut_gemm).

    splitk / cluster force the all-SM streaming kernel / the thread-block-cluster kernels
    (SHIFTADD_FLAG_SPLITK / SHIFTADD_FLAG_CLUSTER), for testing and measurement."""
    squeeze = x.dim() == 1
    x2 = x.unsqueeze(0) if squeeze else x
    if x2.dtype != torch.float16 or not x2.is_cuda or x2.device != layer.device:
        raise ValueError("x must be fp16 on the layer's device")
    if x2.stride(-1) != 1:
        x2 = x2.contiguous()
    M, K = x2.shape
    if K != layer.K:
        raise ValueError("x has K=%d, layer has K=%d" % (K, layer.K))
    dev = layer.device
    if out is None:
        out = torch.empty((M, layer.N), dtype=torch.float16, device=dev)
    if out.dtype != torch.float16 or out.dim() != 2 or out.shape[0] != M or out.stride(-1) != 1:
        raise ValueError("out must be fp16 [M][>=N] with unit column stride")
    if layer.blockwise:
        if M != 1:
            raise ShiftAddError("block-wise layers: batch-1 only (shiftadd_lut_gemv_blockwise)")
        lut_gemv_blockwise(x2[0], layer, out=out[0], pdl=pdl, workspace=workspace, stream=stream)
        return out[0] if squeeze else out
    if layer.colwise:
        lut_gemv_colwise(x2, layer, out=out[:, :layer.N] if M > 1 else out[0], pdl=pdl, stream=stream,
                         workspace=workspace, splitk=splitk)
        return out[0] if squeeze else out
    if layer.exps2 is not None:
        if torch.cuda.current_device() != dev.index:
            torch.cuda.set_device(dev)
        sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
        need = int(lib().shiftadd_workspace_bytes_apot2(layer.N, layer.K)) if layer.layout == LAYOUT_TILED else 0
        ws = (workspace or _workspace_for(dev, stream)).get(need)
        st = lib().shiftadd_lut_gemm_apot2_ws(x2.data_ptr(), x2.stride(0), layer.planes.data_ptr(),
                                              layer.exps.data_ptr(), layer.exps2.data_ptr(), layer.layout, M,
                                              layer.N, layer.K, layer.q, layer.g, out.data_ptr(), out.stride(0),
                                              ws.data_ptr() if ws is not None else None,
                                              ws.numel() if ws is not None else 0,
                                              (FLAG_PDL if pdl else 0) | (FLAG_SPLITK if splitk else 0), sptr)
        if st:
            _check(st, "shiftadd_lut_gemm_apot2_ws")
        return out[0] if squeeze else out
    need = layer._ws_bytes.get(M)
    if need is None:
        need = layer._ws_bytes[M] = workspace_bytes(layer, M)
    ws = (workspace or _workspace_for(dev, stream)).get(need)
    if torch.cuda.current_device() != dev.index:
        torch.cuda.set_device(dev)
    sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
    st = lib().shiftadd_lut_gemm(x2.data_ptr(), x2.stride(0), layer.planes.data_ptr(), layer.exps.data_ptr(),
                                 layer.layout, M, layer.N, layer.K, layer.q, layer.g, out.data_ptr(),
                                 out.stride(0), ws.data_ptr() if ws is not None else None,
                                 ws.numel() if ws is not None else 0,
                                 (FLAG_PDL if pdl else 0) | (FLAG_SPLITK if splitk else 0)
                                 | (FLAG_CLUSTER if cluster else 0), sptr)
    if st:
        _check(st, "shiftadd_lut_gemm")
    return out[0] if squeeze else out


def _segments(layers, outs):
    arr = (_Segment * len(layers))()
    for i, (L, y) in enumerate(zip(layers, outs)):
        arr[i].planes = L.planes.data_ptr()
        arr[i].exps = L.exps.data_ptr()
        arr[i].N = L.N
        arr[i].q = L.q
        arr[i].y = y.data_ptr() if y is not None else None
    return arr


def workspace_bytes_fused(layers, M: int = 1) -> int:
    L0 = layers[0]
    return int(lib().shiftadd_workspace_bytes_fused(L0.layout, M, L0.K, L0.g, len(layers),
                                                    _segments(layers, [None] * len(layers))))


def lut_gemv_fused(x: torch.Tensor, layers, outs=None, workspace: Workspace | None = None, pdl: bool = False,
                   stream=None, splitk: bool = False):
    """Fused projections sharing x (shiftadd_lut_gemv_fused): one launch computes
    y_i = x (.) layers[i] for every segment i, each with its own bit width.  x: fp16 [K];
    layers: tiled PackedLayers with the same K and g; returns the list of y_i (fp16 [N_i]).
    K <= 4096 with <= 24 MB of planes runs on the cluster TMA ring (kernel 10) unless splitk
    forces the all-SM streaming kernel (8), which takes the rest."""
    x = x.reshape(-1)
    if x.dtype != torch.float16 or not x.is_cuda:
        raise ValueError("x must be fp16 on the device")
    if not 1 <= len(layers) <= 4:
        raise ValueError("1..4 segments")
    dev = layers[0].device
    if outs is None:
        outs = [torch.empty(L.N, dtype=torch.float16, device=dev) for L in layers]
    for L, y in zip(layers, outs):
        if L.K != x.numel() or L.g != layers[0].g or L.layout != LAYOUT_TILED or L.colwise or L.exps2 is not None:
            raise ValueError("fused segments: tiled row-wise layers with the K and g of x")
        if y.dtype != torch.float16 or y.numel() != L.N or not y.is_contiguous():
            raise ValueError("outs must be contiguous fp16 [N_i]")
    segs = _segments(layers, outs)
    need = int(lib().shiftadd_workspace_bytes_fused(LAYOUT_TILED, 1, x.numel(), layers[0].g, len(layers), segs))
    ws = (workspace or _workspace_for(dev, stream)).get(need)
    if torch.cuda.current_device() != dev.index:
        torch.cuda.set_device(dev)
    sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
    _check(lib().shiftadd_lut_gemv_fused(x.data_ptr(), x.numel(), layers[0].g, LAYOUT_TILED, len(layers), segs,
                                         ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
                                         (FLAG_PDL if pdl else 0) | (FLAG_SPLITK if splitk else 0), sptr),
           "shiftadd_lut_gemv_fused")
    return outs


def lut_gemv(x: torch.Tensor, layer: PackedLayer, **kw) -> torch.Tensor:
    """Batch-1 form: x fp16 [K] -> y fp16 [N]."""
    return lut_gemm(x.reshape(-1), layer, **kw)


CALL_WAIT = 1


def _encode_calls(calls):
    arr = (_Call * len(calls))()
    keep = []
    for j, (x, layers, outs, wait) in enumerate(calls):
        x = x.reshape(-1)
        if x.dtype != torch.float16 or not x.is_cuda or not 1 <= len(layers) <= 4 or len(outs) != len(layers):
            raise ValueError("call %d: fp16 x on the device and 1..4 segments with outputs" % j)
        for L, y in zip(layers, outs):
            if L.K != x.numel() or L.g != layers[0].g or L.layout != LAYOUT_TILED or L.colwise or \
                    L.exps2 is not None:
                raise ValueError("call %d: tiled row-wise layers with the K and g of x" % j)
            if y.dtype != torch.float16 or y.numel() != L.N or not y.is_contiguous():
                raise ValueError("call %d: outputs must be contiguous fp16 [N_i]" % j)
        c = arr[j]
        c.x, c.K, c.g, c.nseg, c.flags = x.data_ptr(), x.numel(), layers[0].g, len(layers), CALL_WAIT if wait else 0
        for i, (L, y) in enumerate(zip(layers, outs)):
            c.seg[i] = _Segment(L.planes.data_ptr(), L.exps.data_ptr(), L.N, L.q, y.data_ptr())
        keep.append((x, layers, outs))
    return arr, keep


class Chain:
    """An ordered list of calls launched from C as one kernel per call (shiftadd_lut_gemv_chain):
    a decode step costs one ctypes call.  calls: as for Program; with pdl=True every launch
    waits for the previous one (the ``wait`` entries are implied).  The tensors must stay alive
    and in place while the Chain is used."""

    def __init__(self, calls, device=None):
        if not calls:
            raise ValueError("empty chain")
        self.device = torch.device(device) if device is not None else calls[0][1][0].device
        self.calls, self._keep = _encode_calls(calls)
        self.n = len(calls)
        need = int(lib().shiftadd_workspace_bytes_chain(self.calls, self.n))
        self.workspace = Workspace(self.device)
        self.workspace.get(need)

    def __call__(self, stream=None, pdl: bool = True):
        if torch.cuda.current_device() != self.device.index:
            torch.cuda.set_device(self.device)
        sptr = (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream
        ws = self.workspace.buf
        _check(lib().shiftadd_lut_gemv_chain(self.calls, self.n, ws.data_ptr() if ws is not None else None,
                                             ws.numel() if ws is not None else 0, FLAG_PDL if pdl else 0, sptr),
               "shiftadd_lut_gemv_chain")


class Program:
    """A decode step as one persistent launch (shiftadd_lut_gemv_program, kernel id 9).

    calls: list of (x, layers, outs, wait) in execution order -- x fp16 [K] on the device,
    layers: 1..4 tiled PackedLayers sharing x (same K and g), outs: their fp16 [N_i] outputs,
    wait: x is read only after every earlier call stored its outputs (SHIFTADD_CALL_WAIT).
    The encoded program (device pointers of the calls) is copied to the device once here; the
    tensors must stay alive and in place while the Program is used.  The workspace is owned by
    the Program (program launches do not share it with other calls)."""

    def __init__(self, calls, device=None):
        if not calls:
            raise ValueError("empty program")
        self.device = torch.device(device) if device is not None else calls[0][1][0].device
        arr, self._keep = _encode_calls(calls)
        self.calls, self.n = arr, len(calls)
        nb = int(lib().shiftadd_program_bytes(self.n))
        host = torch.empty(nb, dtype=torch.uint8).pin_memory()
        _check(lib().shiftadd_program_encode(arr, self.n, host.data_ptr(), nb), "shiftadd_program_encode")
        self.program = host.to(self.device)
        need = int(lib().shiftadd_workspace_bytes_program(arr, self.n))
        if need == 0:
            raise ShiftAddError("shiftadd_workspace_bytes_program: " + lib().shiftadd_last_error().decode())
        self.workspace = torch.zeros(need, dtype=torch.uint8, device=self.device)

    def __call__(self, stream=None):
        if torch.cuda.current_device() != self.device.index:
            torch.cuda.set_device(self.device)
        sptr = (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream
        _check(lib().shiftadd_lut_gemv_program(self.calls, self.n, self.program.data_ptr(), self.program.numel(),
                                               self.workspace.data_ptr(), self.workspace.numel(), 0, sptr),
               "shiftadd_lut_gemv_program")


COPY_SRC_READY = 4


def copy(dst: torch.Tensor, src: torch.Tensor, pdl: bool = False, src_ready: bool = False, stream=None):
    """Kernel copy between device memory and pinned host memory (shiftadd_copy): the e2e
    host<->device transfers of a decode step inside its PDL chain.  src_ready: src is not
    written by the preceding kernel on the stream (it may be read before the PDL wait)."""
    nbytes = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() != nbytes:
        raise ValueError("copy: size mismatch")
    for t in (dst, src):
        if not (t.is_cuda or t.is_pinned()):
            raise ValueError("copy: tensors must be on the device or in pinned host memory")
        if not t.is_contiguous():
            raise ValueError("copy: tensors must be contiguous")
    dev = dst.device if dst.is_cuda else src.device
    flags = (FLAG_PDL if pdl else 0) | (COPY_SRC_READY if src_ready else 0)
    _check(lib().shiftadd_copy(_ptr(dst), _ptr(src), nbytes, flags, _stream_ptr(stream, dev)), "shiftadd_copy")
    return dst


def gemm_plan(layer: PackedLayer, M: int):
    """(grid, threads, dynamic smem bytes, kernel id) the call would launch with."""
    out = (ctypes.c_int * 4)()
    _check(lib().shiftadd_gemm_plan(layer.layout, M, layer.N, layer.K, layer.q, layer.g, ctypes.byref(out)),
           "shiftadd_gemm_plan")
    return tuple(out)
