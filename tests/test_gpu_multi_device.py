"""GPU, two or more devices: the multi-GPU paths on real ordinals.

Skipped on a one-GPU box (gpurun and the driver's round-end tests have one B200); they run
as soon as a multi-GPU box is available:
* vmb_vmonarch_fwd_multi on devices 0 and 1: heads bitwise equal to one call, sequence slabs
  with the K/V all-gather as P2P loads over NVLink (peer_gather);
* the process-per-GPU NCCL path dist.vmonarch_attention_seq on 2 ranks, against the
  unsharded forward."""
import json
import os
import subprocess
import sys

import pytest
import torch

from vmb_testutil import relfro

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")


def _inputs(vm, grid, device, seed):
    g = torch.Generator(device=device).manual_seed(seed)
    return [torch.randn((grid.units(), grid.tokens(), grid.head_dim), device=device, generator=g).bfloat16()
            for _ in range(3)]


@pytest.mark.parametrize("mode", ["heads", "seq"])
def test_multi_on_two_devices(vm, mode):
    _need(2)
    from paper_2601_22275_b200.dist import local_slab
    grid = vm.TokenGrid(6, 10, 26, 128, 4, 1)
    q, k, v = _inputs(vm, grid, "cuda:0", 11)
    full = vm.vmonarch_attention(q, k, v, grid)
    devs = [torch.device("cuda", i) for i in range(2)]
    if mode == "heads":
        parts = [vm.shard_range(4, 2, r) for r in range(2)]
        sl = lambda x: [x[a:a + c].to(d) for (a, c), d in zip(parts, devs)]  # noqa: E731
    else:
        parts = [vm.shard_range(grid.h * grid.w, 2, r) for r in range(2)]
        sl = lambda x: [local_slab(x, grid, a, c).to(d) for (a, c), d in zip(parts, devs)]  # noqa: E731
    outs = vm.vmonarch_attention_multi(sl(q), sl(k), sl(v), grid, mode=mode)
    for d in devs:
        torch.cuda.synchronize(d)
    if mode == "heads":
        assert torch.equal(torch.cat([o.to("cuda:0") for o in outs], 0), full)
    else:
        for (a, c), o in zip(parts, outs):
            want = local_slab(full, grid, a, c)
            T, hw = grid.t_frames, c
            w4, o4 = want.view(4, T, hw, 128), o.to("cuda:0").view(4, T, hw, 128)
            assert torch.equal(w4[:, 1:], o4[:, 1:])
            assert relfro(o4[:, 0].float().cpu().numpy(), w4[:, 0].float().cpu().numpy()) <= 5e-3


NCCL2 = r"""
import os, sys, json
import torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
import paper_2601_22275_b200 as vm
from paper_2601_22275_b200.dist import vmonarch_attention_seq, local_slab, slab_partition
grid = vm.TokenGrid(6, 10, 26, 128, 2, 1)
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn((2, grid.tokens(), 128), generator=g, device="cuda").bfloat16() for _ in range(3))
full = vm.vmonarch_attention(q, k, v, grid)
a, c = slab_partition(grid.h * grid.w, dist.get_world_size())[rank]
sl = lambda x: local_slab(x, grid, a, c)
out = vmonarch_attention_seq(sl(q), sl(k), sl(v), grid)
torch.cuda.synchronize()
f, o = sl(full).view(2, grid.t_frames, c, 128).float(), out.view(2, grid.t_frames, c, 128).float()
e0 = float(((o[:, 0] - f[:, 0]).norm() / f[:, 0].norm()).item())
print(json.dumps({"rank": rank, "frames_ge1_equal": bool(torch.equal(o[:, 1:], f[:, 1:])), "frame0_relfro": e0}))
dist.destroy_process_group()
"""


def test_nccl_seq_two_ranks():
    _need(2)
    script = os.path.join("/tmp", "vmb_nccl2.py")
    with open(script, "w") as f:
        f.write(NCCL2 % {"root": ROOT})
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29533", script], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(res) == 2
    for x in res:
        assert x["frames_ge1_equal"] and x["frame0_relfro"] <= 5e-3
