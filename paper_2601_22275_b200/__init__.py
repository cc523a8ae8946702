"""B200-native VMonarch attention forward (arXiv 2601.22275).

Python mirror of the reference operator API (/root/reference/proj/include/vmonarch/video.hpp,
monarch.hpp, flash_entropy.hpp) on top of the C ABI in include/vmb.h (libvmb.so, hand-written
sm_100a kernels).  Tensors are torch CUDA tensors (torch is the device-memory/stream plumbing);
every compute call goes through libvmb.so.  There is no CPU fallback: if the extension is
missing, importing this package raises.

Reference -> here
  TokenGrid / VMonarchConfig (video.hpp:16-36)          TokenGrid / VMonarchConfig
  vmonarch_attention<T> (video.hpp:84-150)              vmonarch_attention
  r_update / l_update (monarch.hpp:53-147)              r_update / l_update
  flash_entropy_fwd (flash_entropy.hpp:85-139)          flash_entropy_fwd
  flash_entropy_bwd (flash_entropy.hpp:141-221)         flash_entropy_bwd
  dense_forward (oracle.hpp:36-72)                      dense_forward
  factorize / flops_estimate (video.cpp:13-59)          factorize / flops_estimate
  make_perm (perm.hpp:19-30)                            make_perm
  std::invalid_argument / domain_error / logic_error    DimensionError / DomainError / StateError
Beyond the reference API: vmonarch_attention_host (host buffers, pipelined H2D / forward /
D2H), vmonarch_attention_slab + seq_assemble (sequence sharding, one process per GPU),
vmonarch_attention_multi (one process, several GPUs), torch_op (DiT integration), dist
(partitions and NCCL collectives), matn (MATN files).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import torch

__all__ = [
    "TokenGrid", "VMonarchConfig", "CostReport", "DimensionError", "DomainError", "StateError",
    "vmonarch_attention", "r_update", "l_update", "flash_entropy_fwd", "dense_forward",
    "factorize", "flops_estimate", "make_perm", "preset_grid", "export_factors", "lib",
    "kernel_launch_count", "LIB_PATH", "vmonarch_attention_slab", "seq_assemble", "vmonarch_attention_host",
    "flash_entropy_bwd", "vmonarch_attention_multi", "shard_range", "SHARD_MODES", "CudaError",
    "workspace_size",
]

LIB_PATH = os.environ.get("VMB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvmb.so")


class DimensionError(ValueError):
    """std::invalid_argument("dimension error: ...") in the reference (check.hpp:10-12)."""


class DomainError(ArithmeticError):
    """std::domain_error("domain error: ...") in the reference (check.hpp:14-16)."""


class StateError(RuntimeError):
    """std::logic_error("state error: ...") in the reference (check.hpp:18-20)."""


class CudaError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python __graft_entry__.py build` (make -C "
            "paper_2601_22275_b200/csrc).  There is no CPU fallback.")
    return C.CDLL(LIB_PATH)


lib = _load()

_P, _I64, _I32, _D, _F = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_float


class _Grid(C.Structure):
    _fields_ = [("t_frames", _I64), ("h", _I64), ("w", _I64), ("head_dim", _I64), ("heads", _I64),
                ("batch", _I64)]


class _Cfg(C.Structure):
    _fields_ = [("iters", _I64), ("clamp_min", _D), ("clamp_enabled", _I32),
                ("recompute_first_frame", _I32), ("override_m", _I64), ("override_b", _I64),
                ("tile_br", _I64), ("tile_bc", _I64)]


class _Strides(C.Structure):
    _fields_ = [("batch", _I64), ("head", _I64), ("token", _I64)]


def _sig(name, args, res=C.c_int):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


_vmb_last_error = _sig("vmb_last_error", [], C.c_char_p)
_vmb_factorize = _sig("vmb_factorize", [C.POINTER(_Grid), C.POINTER(_Cfg), C.POINTER(_I64), C.POINTER(_I64)])
_vmb_make_perm = _sig("vmb_make_perm", [_I64, _I64, _P])
_vmb_flops = _sig("vmb_flops_estimate", [C.POINTER(_Grid), C.POINTER(_Cfg), _I64] + [_P] * 6)
_vmb_ws_size = _sig("vmb_workspace_size", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int], C.c_size_t)
_vmb_fwd = _sig("vmb_vmonarch_fwd", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int, _P, _P, _P, _P,
                                     C.POINTER(_Strides), C.POINTER(_Strides), _P, C.c_size_t, _P])
_vmb_ws_status = _sig("vmb_workspace_status", [_P, _P])
_vmb_export = _sig("vmb_export_factors", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int, _P, _P,
                                          C.POINTER(_Strides), _P, _P, _P, _P])
_vmb_rstep = _sig("vmb_rstep", [_I64, _I64, _I64, _I64, C.c_int, _P, _P, _P, _D, _I32, _P, _P, _P, _P])
_vmb_lstep = _sig("vmb_lstep", [_I64, _I64, _I64, _I64, C.c_int, _P, _P, _P, _P, _P, _P, _P])
_vmb_flash = _sig("vmb_flash_entropy_fwd", [_I64, _I64, _I64, _I64, C.c_int, _P, _P, _P, _F, _P, _P, _P, _P])
_vmb_flash_bwd = _sig("vmb_flash_entropy_bwd", [_I64, _I64, _I64, _I64, C.c_int] + [_P] * 8 + [_I32, _P, _P, _P, _P])
_vmb_dense = _sig("vmb_dense_fwd", [_I64, _I64, _I64, C.c_int, _P, _P, _P, _P, _P])
_vmb_launches = _sig("vmb_kernel_launch_count", [], C.c_uint64)
_vmb_ws_size_seq = _sig("vmb_workspace_size_seq", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int, _I64], C.c_size_t)
_vmb_fwd_seq = _sig("vmb_vmonarch_fwd_seq", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int, _I64, _I64, _P, _P, _P, _P,
                                             _P, C.c_size_t, _P])
_vmb_fwd_seq_v = _sig("vmb_vmonarch_fwd_seq_v", [C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int, _I64, _I64, _P, _P, _P,
                                                 _P, _P, C.c_size_t, _P, _P])
_vmb_seq_assemble = _sig("vmb_seq_assemble", [C.POINTER(_Grid), C.c_int, _I32, _P, _P, _I64, _P, _P, _P])
_vmb_shard_range = _sig("vmb_shard_range", [_I64, _I32, _I32, C.POINTER(_I64), C.POINTER(_I64)], None)
_vmb_ws_size_multi = _sig("vmb_workspace_size_multi", [_I32, _I32, C.c_int, C.POINTER(_Grid), C.POINTER(_Cfg),
                                                       C.c_int], C.c_size_t)
_vmb_fwd_multi = _sig("vmb_vmonarch_fwd_multi", [_I32, _P, C.c_int, C.POINTER(_Grid), C.POINTER(_Cfg), C.c_int]
                      + [_P] * 7)
_vmb_selftest = _sig("vmb_selftest_umma", [_I32, _P, _P, _P, _P])

VMB_F32, VMB_BF16, VMB_F64 = 0, 1, 2
_ERRORS = {1: DimensionError, 2: DomainError, 3: StateError, 4: CudaError, 5: CudaError}


def _check(status: int):
    if status != 0:
        msg = (_vmb_last_error() or b"").decode()
        raise _ERRORS.get(status, CudaError)(msg)


def kernel_launch_count() -> int:
    """Kernels libvmb.so has launched in this process (all entry points)."""
    return int(_vmb_launches())


# ----------------------------------------------------------------------------- config types
@dataclass
class TokenGrid:
    """video.hpp:16-27.  Frame-major tokens: token = t*(h*w) + r*w + c."""
    t_frames: int = 1
    h: int = 1
    w: int = 1
    head_dim: int = 64
    heads: int = 1
    batch: int = 1

    def tokens(self) -> int:
        return self.t_frames * self.h * self.w

    def frame_tokens(self) -> int:
        return self.h * self.w

    def units(self) -> int:
        return self.heads * self.batch

    def _c(self) -> _Grid:
        return _Grid(self.t_frames, self.h, self.w, self.head_dim, self.heads, self.batch)


@dataclass
class VMonarchConfig:
    """video.hpp:29-36 (+ TileConfig flash_entropy.hpp:13-16, accepted for API parity)."""
    iters: int = 2
    clamp_min: float = 0.1
    clamp_enabled: bool = True
    recompute_first_frame: bool = True
    override_m_b: Optional[Tuple[int, int]] = None
    tiles: Tuple[int, int] = (64, 64)

    def _c(self) -> _Cfg:
        om, ob = self.override_m_b if self.override_m_b else (0, 0)
        return _Cfg(self.iters, self.clamp_min, int(self.clamp_enabled), int(self.recompute_first_frame),
                    om, ob, self.tiles[0], self.tiles[1])


@dataclass
class CostReport:
    """video.hpp:38-47."""
    sparsity: float = 0.0
    sparsity_approx: float = 0.0
    monarch_flops: int = 0
    full_attn_flops: int = 0
    recompute_flops: int = 0
    reduction_ratio: float = 0.0


_PRESETS = {"wan-61f": (16, 28, 52), "wan-141f": (36, 28, 52), "wan-321f": (81, 28, 52)}


def preset_grid(name: str) -> Optional[Tuple[int, int, int]]:
    """video.cpp:5-11 preset latent grids (T, h, w)."""
    return _PRESETS.get(name)


def factorize(grid: TokenGrid, cfg: VMonarchConfig = VMonarchConfig()) -> Tuple[int, int]:
    """video.cpp:13-22: (m, b) = (T, h*w) unless overridden with m*b = N."""
    m, b = _I64(), _I64()
    g, c = grid._c(), cfg._c()
    _check(_vmb_factorize(C.byref(g), C.byref(c), C.byref(m), C.byref(b)))
    return m.value, b.value


def flops_estimate(grid: TokenGrid, cfg: VMonarchConfig, d: int) -> CostReport:
    """video.cpp:36-59 — the FLOP convention of the headline metric (2 FLOPs/MAC, matmuls)."""
    vals = [C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_double()]
    g, c = grid._c(), cfg._c()
    _check(_vmb_flops(C.byref(g), C.byref(c), d, *[C.addressof(x) for x in vals]))
    return CostReport(vals[0].value, vals[1].value, vals[2].value, vals[3].value, vals[4].value,
                      vals[5].value)


def make_perm(b: int, n: int) -> list:
    """perm.hpp:19-30 forward_index (bit-exact)."""
    out = (C.c_int64 * max(n, 1))()
    _check(_vmb_make_perm(b, n, C.addressof(out)))
    return list(out)[:n]


# ----------------------------------------------------------------------------- helpers
def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return VMB_F32
    if t.dtype == torch.float64:
        return VMB_F64
    if t.dtype == torch.bfloat16:
        return VMB_BF16
    raise DimensionError(f"dimension error: unsupported dtype {t.dtype} (bfloat16, float32 or float64)")


def _stream(device: Optional[torch.device] = None) -> C.c_void_p:
    """The current stream of `device` (of the current device when None)."""
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _call(device: torch.device, fn, *args):
    """One ABI call ordered on `device`'s current stream (passed last), with that device
    current for its duration."""
    with torch.cuda.device(device):
        _check(fn(*args, _stream(device)))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise DimensionError("dimension error: tensors must be CUDA tensors (no CPU path)")


def _bhsd_strides(t: torch.Tensor, grid: TokenGrid) -> _Strides:
    """Accept (units, N, d), (B, H, N, d) or BSHD (B, N, H, d) given as a (B, H, N, d) view."""
    n, d = grid.tokens(), grid.head_dim
    if t.dim() == 3:
        if tuple(t.shape) != (grid.units(), n, d):
            raise DimensionError("dimension error: expected one Q/K/V matrix per batch*head unit "
                                 f"of shape ({grid.units()}, {n}, {d}), got {tuple(t.shape)}")
        if t.stride(2) != 1:
            raise DimensionError("dimension error: head dim must be contiguous")
        su = t.stride(0)
        return _Strides(su * grid.heads, su, t.stride(1))
    if t.dim() == 4:
        if tuple(t.shape) != (grid.batch, grid.heads, n, d):
            raise DimensionError(f"dimension error: expected (B, H, N, d) = ({grid.batch}, {grid.heads}, "
                                 f"{n}, {d}), got {tuple(t.shape)}")
        if t.stride(3) != 1:
            raise DimensionError("dimension error: head dim must be contiguous")
        return _Strides(t.stride(0), t.stride(1), t.stride(2))
    raise DimensionError("dimension error: Q/K/V must be 3-D (units, N, d) or 4-D (B, H, N, d)")


class _WorkspaceCache:
    """Workspaces keyed by (device, stream, kind).

    The ABI's rule is one workspace per concurrent call (vmb.h).  A buffer here is only ever
    handed to calls on the stream it is keyed by, so calls on different streams (CFG
    branches, the host pipeline's compute stream, user streams) never share one, and a buffer
    that is replaced or evicted was last used on its own allocation stream -- the caching
    allocator reuses it in that stream's order, so dropping it needs no record_stream.  Under
    CUDA-graph capture a fresh workspace comes from the capture's pool on every call."""

    def __init__(self, max_entries: int = 8):
        self._d: "OrderedDict" = OrderedDict()
        self.max_entries = max_entries

    def get(self, device: torch.device, stream: torch.cuda.Stream, kind: str, nbytes: int) -> torch.Tensor:
        if torch.cuda.is_current_stream_capturing():
            return torch.empty(nbytes, dtype=torch.uint8, device=device)
        key = (device.index, stream.cuda_stream, kind)
        ws = self._d.get(key)
        if ws is None or ws.numel() < nbytes:
            self._d.pop(key, None)
            ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._d[key] = ws
        self._d.move_to_end(key)
        while len(self._d) > self.max_entries:
            self._d.popitem(last=False)
        return ws

    def clear(self):
        self._d.clear()


_WS_CACHE = _WorkspaceCache()


def _workspace(grid: TokenGrid, cfg: VMonarchConfig, dt: int, device: torch.device,
               stream: torch.cuda.Stream) -> torch.Tensor:
    g, c = grid._c(), cfg._c()
    nbytes = int(_vmb_ws_size(C.byref(g), C.byref(c), dt))
    if nbytes == 0:
        _check(1)
    return _WS_CACHE.get(device, stream, "fwd", nbytes)


def _check_out(out: torch.Tensor, q: torch.Tensor):
    """A caller-supplied output must match q's dtype and device: the ABI writes it with q's
    element size (vmb.h), so a mismatch would write outside the buffer."""
    if out.dtype != q.dtype:
        raise DimensionError(f"dimension error: out dtype {out.dtype} != q dtype {q.dtype}")
    if out.device != q.device:
        raise DimensionError(f"dimension error: out on {out.device}, q on {q.device}")


# ----------------------------------------------------------------------------- the operator
def vmonarch_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, grid: TokenGrid,
                       cfg: VMonarchConfig = VMonarchConfig(), out: Optional[torch.Tensor] = None,
                       factors_out: Optional[list] = None, check: bool = True,
                       workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """video.hpp:84-150 on the GPU.

    q, k, v: CUDA tensors (units, N, d) [unit u = b*H + h], or (B, H, N, d) views (BSHD
    activations pass as ``x.transpose(1, 2)``), float32 (parity mode), float64 (the
    reference's T = double, CUDA cores) or bfloat16 (tcgen05).
    Returns O with the layout of ``q`` (3-D) or a (B, H, N, d) tensor.
    ``factors_out``: if a list, receives per-unit (L (b,m,m), R (m,b,b)) fp32 tensors (small N).
    ``check``: synchronise and raise DomainError for device-detected domain errors
    (non-finite Q, monarch.hpp:44).  Set False inside timed loops.
    ``workspace``: optional caller-owned uint8 scratch of >= workspace_size(grid, cfg) bytes;
    by default one is cached per (device, stream).  The call is ordered on q.device's current
    stream.
    """
    _require_cuda(q, k, v, out)
    dt = _dtype_code(q)
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise DimensionError("dimension error: Q, K, V must share dtype")
    if k.device != q.device or v.device != q.device:
        raise DimensionError("dimension error: Q, K, V must be on one device")
    sq, sk, sv = _bhsd_strides(q, grid), _bhsd_strides(k, grid), _bhsd_strides(v, grid)
    if (sk.batch, sk.head, sk.token) != (sq.batch, sq.head, sq.token) or \
            (sv.batch, sv.head, sv.token) != (sq.batch, sq.head, sq.token):
        # the ABI takes one stride set for Q/K/V; normalise the odd ones out
        k = k.contiguous() if (sk.batch, sk.head, sk.token) != (sq.batch, sq.head, sq.token) else k
        v = v.contiguous() if (sv.batch, sv.head, sv.token) != (sq.batch, sq.head, sq.token) else v
        if not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
            q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        sq = _bhsd_strides(q, grid)
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    _check_out(out, q)
    so = _bhsd_strides(out, grid)
    dev = q.device
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = workspace if workspace is not None else _workspace(grid, cfg, dt, dev, stream)
        g, c = grid._c(), cfg._c()
        need = int(_vmb_ws_size(C.byref(g), C.byref(c), dt))
        if ws.device != dev or ws.dtype != torch.uint8 or not ws.is_contiguous() or ws.numel() < need:
            raise DimensionError(f"dimension error: workspace must be a contiguous uint8 tensor of >= {need} "
                                 f"bytes on {dev}")
        st = C.c_void_p(stream.cuda_stream)
        _check(_vmb_fwd(C.byref(g), C.byref(c), dt, _ptr(q), _ptr(k), _ptr(v), _ptr(out), C.byref(sq),
                        C.byref(so), _ptr(ws), ws.numel(), st))
        if check or factors_out is not None:
            _check(_vmb_ws_status(_ptr(ws), st))
        if factors_out is not None:
            m, b = factorize(grid, cfg)
            U = grid.units()
            fdt = torch.float64 if dt == VMB_F64 else torch.float32  # the state type of the mode
            L = torch.empty((U, b, m, m), dtype=fdt, device=dev)
            R = torch.empty((U, m, b, b), dtype=fdt, device=dev)
            _check(_vmb_export(C.byref(g), C.byref(c), dt, _ptr(q), _ptr(k), C.byref(sq), _ptr(ws), _ptr(L),
                               _ptr(R), st))
            factors_out.clear()
            factors_out.extend((L[u], R[u]) for u in range(U))
    return out


def workspace_size(grid: TokenGrid, cfg: VMonarchConfig = VMonarchConfig(), dtype=torch.bfloat16) -> int:
    """Bytes of scratch one vmonarch_attention call needs (vmb_workspace_size)."""
    g, c = grid._c(), cfg._c()
    code = {torch.bfloat16: VMB_BF16, torch.float32: VMB_F32, torch.float64: VMB_F64}[dtype]
    n = int(_vmb_ws_size(C.byref(g), C.byref(c), code))
    if n == 0:
        _check(1)
    return n


# ----------------------------------------------------------------------------- host-buffer pipeline
class _HostPipeline:
    """Device buffers + streams reused across vmonarch_attention_host calls of one shape."""

    def __init__(self, shape, dtype, device, chunk, nbuf):
        self.key = (shape, dtype, device, chunk, nbuf)
        self.bufs = [tuple(torch.empty((chunk,) + tuple(shape[1:]), dtype=dtype, device=device) for _ in range(4))
                     for _ in range(nbuf)]
        self.h2d = torch.cuda.Stream(device)
        self.comp = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)


_PIPE: dict = {}


def vmonarch_attention_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, grid: TokenGrid,
                            cfg: VMonarchConfig = VMonarchConfig(), out: Optional[torch.Tensor] = None,
                            chunk_units: int = 8, device=None, sync: bool = True) -> torch.Tensor:
    """video.hpp:84-150 for HOST tensors (units, N, d): batch*head units are independent
    (video.hpp:131-148), so chunks of units stream through the device -- the H2D copy of chunk
    c+1, the forward of chunk c and the D2H copy of chunk c-1 run on three CUDA streams.
    Inputs should be pinned for the copies to overlap.  Returns the host output.

    Like the reference operator, the call returns finished results (``sync=True``: the host
    waits for the last D2H copy).  With ``sync=False`` it returns as soon as the work is
    queued: ``out`` is complete once the device's current stream reaches this point, and the
    inputs must stay unchanged until then (the H2D copies read them asynchronously)."""
    if q.is_cuda or k.is_cuda or v.is_cuda:
        raise DimensionError("dimension error: vmonarch_attention_host takes host tensors")
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    U = q.shape[0]
    if U != grid.units() or q.dim() != 3:
        raise DimensionError(f"dimension error: expected (units={grid.units()}, N, d) host tensors")
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    chunk = max(1, min(chunk_units, U))
    nbuf = 2
    key = (tuple(q.shape), q.dtype, device, chunk, nbuf)
    pipe = _PIPE.get(key)
    if pipe is None:
        for old in _PIPE.values():  # an unsynchronised call may still use the old buffers
            old.d2h.synchronize()
        _PIPE.clear()
        pipe = _PIPE[key] = _HostPipeline(tuple(q.shape), q.dtype, device, chunk, nbuf)
    cur = torch.cuda.current_stream(device)
    h2d, comp, d2h = pipe.h2d, pipe.comp, pipe.d2h
    h2d.wait_stream(cur)
    ev_in = [None] * nbuf      # chunk's inputs resident
    ev_done = [None] * nbuf    # chunk's output computed
    ev_free = [None] * nbuf    # buffer set drained to host
    starts = list(range(0, U, chunk))
    for c, a in enumerate(starts):
        b = min(a + chunk, U)
        n = b - a
        slot = c % nbuf
        dq, dk, dv, do = pipe.bufs[slot]
        with torch.cuda.stream(h2d):
            if ev_free[slot] is not None:
                h2d.wait_event(ev_free[slot])
            dq[:n].copy_(q[a:b], non_blocking=True)
            dk[:n].copy_(k[a:b], non_blocking=True)
            dv[:n].copy_(v[a:b], non_blocking=True)
            ev_in[slot] = torch.cuda.Event()
            ev_in[slot].record(h2d)
        with torch.cuda.stream(comp):
            comp.wait_event(ev_in[slot])
            g = TokenGrid(grid.t_frames, grid.h, grid.w, grid.head_dim, n, 1)
            vmonarch_attention(dq[:n], dk[:n], dv[:n], g, cfg, out=do[:n], check=False)
            ev_done[slot] = torch.cuda.Event()
            ev_done[slot].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_done[slot])
            out[a:b].copy_(do[:n], non_blocking=True)
            ev_free[slot] = torch.cuda.Event()
            ev_free[slot].record(d2h)
    cur.wait_stream(d2h)
    if sync:
        d2h.synchronize()
    return out


# ----------------------------------------------------------------------------- sequence-sharded mode
def vmonarch_attention_slab(q_local: torch.Tensor, k_full: torch.Tensor, v_full: torch.Tensor, grid: TokenGrid,
                            pos_begin: int, pos_count: int, cfg: VMonarchConfig = VMonarchConfig(),
                            out: Optional[torch.Tensor] = None, check: bool = True,
                            v_ready: Optional[torch.cuda.Event] = None) -> torch.Tensor:
    """The forward for the spatial slab [pos_begin, pos_begin + pos_count) of every frame
    (SURVEY §8e): q_local / output (units, T * pos_count, d) with local token
    t * pos_count + (position - pos_begin); k_full, v_full (units, N, d).  Slab outputs of all
    ranks are exactly the rows of the unsharded forward (queries are row-independent)."""
    _require_cuda(q_local, k_full, v_full, out)
    dt = _dtype_code(q_local)
    U, n, d = grid.units(), grid.tokens(), grid.head_dim
    nl = grid.t_frames * pos_count
    if tuple(q_local.shape) != (U, nl, d) or tuple(k_full.shape) != (U, n, d) or tuple(v_full.shape) != (U, n, d):
        raise DimensionError(f"dimension error: expected q_local ({U}, {nl}, {d}) and k/v ({U}, {n}, {d})")
    if k_full.dtype != q_local.dtype or v_full.dtype != q_local.dtype:
        raise DimensionError("dimension error: Q, K, V must share dtype")
    if k_full.device != q_local.device or v_full.device != q_local.device:
        raise DimensionError("dimension error: Q, K, V must be on one device")
    q_local, k_full, v_full = q_local.contiguous(), k_full.contiguous(), v_full.contiguous()
    if out is None:
        out = torch.empty_like(q_local)
    _check_out(out, q_local)
    if tuple(out.shape) != (U, nl, d) or not out.is_contiguous():
        raise DimensionError(f"dimension error: out must be a contiguous ({U}, {nl}, {d}) tensor")
    g, c = grid._c(), cfg._c()
    nbytes = int(_vmb_ws_size_seq(C.byref(g), C.byref(c), dt, pos_count))
    if nbytes == 0:
        _check(1)
    dev = q_local.device
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = _WS_CACHE.get(dev, stream, "seq", nbytes)
        st = C.c_void_p(stream.cuda_stream)
        ev = C.c_void_p(v_ready.cuda_event) if v_ready is not None else None
        _check(_vmb_fwd_seq_v(C.byref(g), C.byref(c), dt, pos_begin, pos_count, _ptr(q_local), _ptr(k_full),
                              _ptr(v_full), _ptr(out), _ptr(ws), ws.numel(), st, ev))
        if check:
            _check(_vmb_ws_status(_ptr(ws), st))
    return out


def seq_assemble(gathered: torch.Tensor, grid: TokenGrid, pos_begin: Sequence[int], pos_count: Sequence[int],
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """(world, units, T, slab_max, d) all-gathered slabs -> (units, N, d) frame-major keys."""
    _require_cuda(gathered, out)
    world, U, T, smax, d = gathered.shape
    if out is None:
        out = torch.empty((U, grid.tokens(), d), dtype=gathered.dtype, device=gathered.device)
    b = (C.c_int64 * world)(*pos_begin)
    cn = (C.c_int64 * world)(*pos_count)
    g = grid._c()
    if out.dtype != gathered.dtype or out.device != gathered.device or not out.is_contiguous() or \
            tuple(out.shape) != (U, grid.tokens(), d):
        raise DimensionError(f"dimension error: out must be a contiguous ({U}, {grid.tokens()}, {d}) tensor "
                             "of the gathered dtype and device")
    if len(pos_begin) != world or len(pos_count) != world or T != grid.t_frames or \
            any(c_ > smax for c_ in pos_count) or sum(pos_count) != grid.h * grid.w:
        raise DimensionError("dimension error: slab partition does not match the gathered tensor")
    gathered = gathered.contiguous()
    with torch.cuda.device(gathered.device):
        _check(_vmb_seq_assemble(C.byref(g), _dtype_code(gathered), world, C.addressof(b), C.addressof(cn), smax,
                                 _ptr(gathered), _ptr(out), _stream(gathered.device)))
    return out


# ----------------------------------------------------------------------------- single-process multi-GPU
SHARD_MODES = {"heads": 0, "seq": 1}


def shard_range(n: int, parts: int, r: int) -> Tuple[int, int]:
    """(begin, count) of part r of n items split into `parts` contiguous parts (vmb_shard_range);
    the same partition as dist.unit_shards / dist.slab_partition."""
    b, c = _I64(0), _I64(0)
    _vmb_shard_range(n, parts, r, C.byref(b), C.byref(c))
    return b.value, c.value


def vmonarch_attention_multi(qs: Sequence[torch.Tensor], ks: Sequence[torch.Tensor], vs: Sequence[torch.Tensor],
                             grid: TokenGrid, cfg: VMonarchConfig = VMonarchConfig(), mode: str = "heads",
                             check: bool = True) -> List[torch.Tensor]:
    """One process drives len(qs) GPUs (vmb_vmonarch_fwd_multi).  Part r lives
    on qs[r].device; mode "heads": (units_r, N, d) unit blocks of shard_range(units, n, r);
    mode "seq": (units, T*count_r, d) spatial slabs of shard_range(h*w, n, r), with the K/V
    all-gather done device-to-device over peer memory inside the call.  Returns the per-part
    outputs, ordered on each device's current stream."""
    n = len(qs)
    if not (len(ks) == len(vs) == n) or n == 0:
        raise DimensionError("dimension error: need one q/k/v tensor per device")
    _require_cuda(*qs, *ks, *vs)
    if mode not in SHARD_MODES:
        raise DimensionError(f"dimension error: unknown shard mode {mode!r}")
    dt = _dtype_code(qs[0])
    g, c = grid._c(), cfg._c()
    U, N, d, T = grid.units(), grid.tokens(), grid.head_dim, grid.t_frames
    for r in range(n):
        if mode == "heads":
            want = (shard_range(U, n, r)[1], N, d)
        else:
            want = (U, T * shard_range(grid.h * grid.w, n, r)[1], d)
        for name, x in (("q", qs[r]), ("k", ks[r]), ("v", vs[r])):
            if tuple(x.shape) != want:
                raise DimensionError(f"dimension error: part {r} {name} has shape {tuple(x.shape)}, expected {want}")
            if x.dtype != qs[0].dtype:
                raise DimensionError(f"dimension error: part {r} {name} dtype {x.dtype} != {qs[0].dtype}")
            if x.device != qs[r].device:
                raise DimensionError(f"dimension error: part {r} q/k/v must share one device")
    qs = [x.contiguous() for x in qs]
    ks = [x.contiguous() for x in ks]
    vs = [x.contiguous() for x in vs]
    outs = [torch.empty_like(x) for x in qs]
    wss, sizes, streams = [], [], []
    for r in range(n):
        nb = int(_vmb_ws_size_multi(n, r, SHARD_MODES[mode], C.byref(g), C.byref(c), dt))
        if nb == 0:
            _check(1)
        wss.append(torch.empty(nb, dtype=torch.uint8, device=qs[r].device))
        sizes.append(nb)
        streams.append(torch.cuda.current_stream(qs[r].device).cuda_stream)
    # the ctypes arrays are kept in locals so they outlive the call
    pq, pk, pv, po, pw = ((C.c_void_p * n)(*[_ptr(t) for t in ts]) for ts in (qs, ks, vs, outs, wss))
    devs = (C.c_int32 * n)(*[x.device.index for x in qs])
    szs = (C.c_size_t * n)(*sizes)
    sts = (C.c_void_p * n)(*streams)
    _check(_vmb_fwd_multi(n, C.addressof(devs), SHARD_MODES[mode], C.byref(g), C.byref(c), dt, C.addressof(pq),
                          C.addressof(pk), C.addressof(pv), C.addressof(po), C.addressof(pw), C.addressof(szs),
                          C.addressof(sts)))
    if check:
        for r in range(n):
            _check(_vmb_ws_status(_ptr(wss[r]), C.c_void_p(streams[r])))
    return outs


def export_factors(q, k, grid, cfg, dtype_code):
    """Factor export for the last vmonarch_attention call on this device (MonarchFactors)."""
    m, b = factorize(grid, cfg)
    U = grid.units()
    fdt = torch.float64 if dtype_code == VMB_F64 else torch.float32
    L = torch.empty((U, b, m, m), dtype=fdt, device=q.device)
    R = torch.empty((U, m, b, b), dtype=fdt, device=q.device)
    stream = torch.cuda.current_stream(q.device)
    ws = _workspace(grid, cfg, dtype_code, q.device, stream)
    g, c = grid._c(), cfg._c()
    sq = _bhsd_strides(q, grid)
    _call(q.device, _vmb_export, C.byref(g), C.byref(c), dtype_code, _ptr(q), _ptr(k), C.byref(sq), _ptr(ws),
          _ptr(L), _ptr(R))
    return L, R


# ----------------------------------------------------------------------------- half steps
def r_update(aR: torch.Tensor, cR: torch.Tensor, Kb: torch.Tensor, clamp_min: float = 0.1,
             clamp_enabled: bool = True, want_R: bool = False):
    """monarch.hpp:53-103 for (units, m, b, d) state.  Returns (aL (units,b,m,d), cL (units,b,m) f32, R)."""
    _require_cuda(aR, cR, Kb)
    U, m, b, d = aR.shape
    dt = _dtype_code(aR)
    aR, Kb = aR.contiguous(), Kb.contiguous().to(aR.dtype)
    cR = cR.contiguous().float()
    aL = torch.empty((U, b, m, d), dtype=aR.dtype, device=aR.device)
    cL = torch.empty((U, b, m), dtype=torch.float32, device=aR.device)
    R = torch.empty((U, m, b, b), dtype=torch.float32, device=aR.device) if want_R else None
    _call(aR.device, _vmb_rstep, U, m, b, d, dt, _ptr(aR), _ptr(cR), _ptr(Kb), clamp_min, int(clamp_enabled),
          _ptr(aL), _ptr(cL), _ptr(R))
    return aL, cL, R


def l_update(Qb: torch.Tensor, aL: torch.Tensor, cL: torch.Tensor, want_L: bool = False):
    """monarch.hpp:105-147 for (units, b, m, d) state.  Returns (aR (units,m,b,d), cR (units,m,b) f32, L)."""
    _require_cuda(Qb, aL, cL)
    U, b, m, d = Qb.shape
    dt = _dtype_code(Qb)
    Qb = Qb.contiguous()
    # aL / cL of None (no r_update yet) reach the ABI as NULL -> StateError, as in the reference
    aL = aL.contiguous().to(Qb.dtype) if aL is not None else None
    cL = cL.contiguous().float() if cL is not None else None
    aR = torch.empty((U, m, b, d), dtype=Qb.dtype, device=Qb.device)
    cR = torch.empty((U, m, b), dtype=torch.float32, device=Qb.device)
    L = torch.empty((U, b, m, m), dtype=torch.float32, device=Qb.device) if want_L else None
    _call(Qb.device, _vmb_lstep, U, m, b, d, dt, _ptr(Qb), _ptr(aL), _ptr(cL), _ptr(aR), _ptr(cR), _ptr(L))
    return aR, cR, L


# ----------------------------------------------------------------------------- attention kernels
def flash_entropy_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_scale: float = 1.0,
                      want_entropy: bool = True):
    """flash_entropy.hpp:85-139: (out, lse, entropy) for (units, nq, d) / (units, nk, d) inputs.
    Q must carry its scale (q_scale multiplies the logits; 1.0 = reference semantics)."""
    _require_cuda(q, k, v)
    squeeze = q.dim() == 2
    if squeeze:
        q, k, v = q[None], k[None], v[None]
    U, nq, d = q.shape
    nk = k.shape[1]
    if k.shape[2] != d or v.shape[2] != d:
        raise DimensionError("dimension error: Q, K, V must share head dim")
    if v.shape[1] != nk:
        raise DimensionError("dimension error: K and V must share row count")
    if nk < 1:
        raise DomainError("domain error: attention over empty keys")
    dt = _dtype_code(q)
    q, k, v = q.contiguous(), k.contiguous().to(q.dtype), v.contiguous().to(q.dtype)
    o = torch.empty_like(q)
    lse = torch.empty((U, nq), dtype=torch.float32, device=q.device)
    ent = torch.empty((U, nq), dtype=torch.float32, device=q.device) if want_entropy else None
    _call(q.device, _vmb_flash, U, nq, nk, d, dt, _ptr(q), _ptr(k), _ptr(v), q_scale, _ptr(o), _ptr(lse), _ptr(ent))
    if squeeze:
        return o[0], lse[0], (ent[0] if ent is not None else None)
    return o, lse, ent


def flash_entropy_bwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, dout: torch.Tensor,
                      lse: torch.Tensor, entropy: Optional[torch.Tensor] = None,
                      dentropy: Optional[torch.Tensor] = None, entropy_grad: bool = False):
    """flash_entropy.hpp:146-221 (Alg. 2): (dq, dk, dv) for (units, n, d) or (n, d) inputs.
    q must be the pre-scaled query of the matching flash_entropy_fwd; lse / entropy come from
    that forward; entropy_grad adds the -dH P (S - lse + H) correction to dS."""
    _require_cuda(q, k, v, o, dout, lse, entropy, dentropy)
    squeeze = q.dim() == 2
    if squeeze:
        q, k, v, o, dout = q[None], k[None], v[None], o[None], dout[None]
        lse = lse[None]
        entropy = entropy[None] if entropy is not None else None
        dentropy = dentropy[None] if dentropy is not None else None
    U, nq, d = q.shape
    nk = k.shape[1]
    if k.shape[2] != d or v.shape[2] != d or o.shape[2] != d or dout.shape[2] != d:
        raise DimensionError("dimension error: all operands must share head dim")
    if v.shape[1] != nk:
        raise DimensionError("dimension error: K and V must share row count")
    if o.shape[1] != nq or dout.shape[1] != nq:
        raise DimensionError("dimension error: O and dO must have N_q rows")
    if lse.shape[-1] != nq or (entropy is not None and entropy.shape[-1] != nq) or \
            (dentropy is not None and dentropy.shape[-1] != nq):
        raise DimensionError("dimension error: lse / entropy / dH length must equal N_q")
    dt = _dtype_code(q)
    q, k, v, o, dout = (x.contiguous().to(q.dtype) for x in (q, k, v, o, dout))
    f32 = lambda x: None if x is None else x.contiguous().float()  # noqa: E731
    lse, entropy, dentropy = f32(lse), f32(entropy), f32(dentropy)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    _call(q.device, _vmb_flash_bwd, U, nq, nk, d, dt, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout), _ptr(lse),
          _ptr(entropy), _ptr(dentropy), int(entropy_grad), _ptr(dq), _ptr(dk), _ptr(dv))
    if squeeze:
        return dq[0], dk[0], dv[0]
    return dq, dk, dv


def dense_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """oracle.hpp:36-72 semantics (softmax(Q K^T / sqrt d) V) on the tcgen05 attention kernel."""
    _require_cuda(q, k, v)
    U, n, d = q.shape
    dt = _dtype_code(q)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(q)
    _call(q.device, _vmb_dense, U, n, d, dt, _ptr(q), _ptr(k), _ptr(v), _ptr(o))
    return o


def selftest_umma(mode: int, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """tcgen05/TMA building-block check (see csrc/kernels/selftest.cu)."""
    C_ = torch.empty((128, 128), dtype=torch.float32, device=A.device)
    _call(A.device, _vmb_selftest, mode, _ptr(A.contiguous()), _ptr(B.contiguous()), _ptr(C_))
    return C_
