"""GPU: every attention-kernel family (the A/B variants behind VMB_RSTEP / VMB_ATTN /
VMB_FA_MC, csrc/vmb_api.cu attn_impl) against the CPU oracle.  The switches are read once
per process, so each variant runs in a subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_2601_22275_b200 as vm
from oracle.oracle import Oracle, bf16_round, workload
orc = Oracle("port")
res = {}
for gridt, heads, sigma in [((4, 8, 16), 2, 1.0), ((6, 10, 26), 2, 2.0), ((3, 12, 27), 3, 1.0)]:
    grid = vm.TokenGrid(*gridt, 128, heads, 1)
    q, k, v = workload(heads, grid.tokens(), 128, seed=5, sigma=sigma)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = orc.vmonarch_attention(q, k, v, gridt, iters=2)
    out = vm.vmonarch_attention(*(torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)), grid)
    got = out.float().cpu().numpy()
    res[str(gridt)] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
# dense / flash over the same attention family
qd = torch.randn(2, 700, 128, device="cuda").bfloat16()
od = vm.dense_forward(qd, qd, qd)
ref = torch.softmax(qd.float() @ qd.float().transpose(1, 2) / 128 ** 0.5, -1) @ qd.float()
res["dense"] = float((od.float() - ref).norm() / ref.norm())
print(json.dumps(res))
"""


@pytest.mark.parametrize("env", [{"VMB_RSTEP": "1"}, {"VMB_RSTEP": "4"}, {"VMB_RSTEP": "5"}, {"VMB_ATTN": "2"},
                                 {"VMB_ATTN": "4"}, {"VMB_ATTN": "5"}, {"VMB_RSTEP": "1", "VMB_FA_MC": "1"},
                                 {"VMB_LSTEP": "2"}, {"VMB_ATTN": "6"}, {"VMB_RSTEP": "6"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_kernel_family_parity(cuda, env):
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], capture_output=True, text=True,
                       env={**os.environ, **env}, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for k, err in res.items():
        assert err <= 2e-2, (env, k, err)
