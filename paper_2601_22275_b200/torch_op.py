"""DiT-side integration: a thin torch op and attention module.

The Wan-style DiT attention produces Q/K/V with one fused projection, (B, S, 3, H, D); the
three BSHD slices are strided views (token stride 3*H*D) that the C ABI takes as they are
(vmb_strides), so there is no permute or copy on either side: the output is written BSHD
and flows into the out-projection as (B, S, H*D).  Forward only, like the reference
operator (video.hpp:84-150); ``torch.library.custom_op`` makes it a graph-capturable,
fake-tensor-aware op so it can sit inside a model that is otherwise plain PyTorch.
"""
from __future__ import annotations

import torch

from . import TokenGrid, VMonarchConfig, vmonarch_attention


@torch.library.custom_op("vmb::vmonarch_attention", mutates_args=())
def vmonarch_attention_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, t_frames: int, h: int, w: int,
                          iters: int = 2, clamp_min: float = 0.1, clamp_enabled: bool = True,
                          recompute_first_frame: bool = True, override_m: int = 0, override_b: int = 0,
                          check: bool = False) -> torch.Tensor:
    """q, k, v: (B, S, H, D) CUDA tensors (any token/batch strides, D contiguous), S = t*h*w
    frame-major.  Returns (B, S, H, D).  ``check`` synchronises to raise DomainError for a
    non-finite Q (monarch.hpp:44); off by default so the op stays asynchronous."""
    B, S, H, D = q.shape
    grid = TokenGrid(t_frames, h, w, D, H, B)
    cfg = VMonarchConfig(iters=iters, clamp_min=clamp_min, clamp_enabled=clamp_enabled,
                         recompute_first_frame=recompute_first_frame,
                         override_m_b=(override_m, override_b) if override_m or override_b else None)
    out = torch.empty((B, S, H, D), dtype=q.dtype, device=q.device)
    vmonarch_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), grid, cfg,
                       out=out.transpose(1, 2), check=check)
    return out


@vmonarch_attention_op.register_fake
def _(q, k, v, t_frames, h, w, iters=2, clamp_min=0.1, clamp_enabled=True, recompute_first_frame=True,
      override_m=0, override_b=0, check=False):
    torch._check(q.shape[1] == t_frames * h * w)
    return torch.empty_like(q, memory_format=torch.contiguous_format)


class VMonarchSelfAttention(torch.nn.Module):
    """Self-attention block of a video DiT with VMonarch as the attention kernel:
    fused QKV projection -> strided BSHD views -> vmb::vmonarch_attention -> out-projection.
    (QK-norm / RoPE of a full Wan block would act on the same views before the op.)"""

    def __init__(self, dim: int, heads: int, grid_thw, cfg: VMonarchConfig = VMonarchConfig(), bias: bool = True,
                 device=None, dtype=None):
        super().__init__()
        if dim % heads:
            raise ValueError("dim must be a multiple of heads")
        self.heads, self.head_dim = heads, dim // heads
        self.grid_thw = tuple(grid_thw)
        self.cfg = cfg
        self.qkv = torch.nn.Linear(dim, 3 * dim, bias=bias, device=device, dtype=dtype)
        self.proj = torch.nn.Linear(dim, dim, bias=bias, device=device, dtype=dtype)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        B, S, _ = x.shape
        qkv = self.qkv(x).view(B, S, 3, self.heads, self.head_dim)
        q, k, v = qkv.unbind(2)  # (B, S, H, D) views, token stride 3*H*D: no copies
        t, h, w = self.grid_thw
        c = self.cfg
        om, ob = c.override_m_b or (0, 0)
        o = vmonarch_attention_op(q, k, v, t, h, w, c.iters, c.clamp_min, c.clamp_enabled, c.recompute_first_frame,
                                  om, ob)
        return self.proj(o.reshape(B, S, self.heads * self.head_dim))
