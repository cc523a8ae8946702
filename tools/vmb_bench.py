#!/usr/bin/env python3
"""vmb_bench — the reference benchmark harness (tools/bench_main.cpp) on the B200 path.

Same command line, modes, report schema and exit codes as the reference `vmonarch_bench`
(bench_main.cpp:510-565), so GPU results drop into the reference's report pipeline:

  --mode dense|flash|monarch|vmonarch   (or --sweep FROM:TO[:STEP], monarch vs dense over T)
  --preset wan-61f|wan-141f|wan-321f, --grid TxHxW, --n, --d, --heads, --batch, --m/--b,
  --t (iterations), --clamp-min, --no-clamp, --no-recompute, --br/--bc, --seed, --repeats,
  --verify on|off, --precision f32|bf16, --csv, --dist normal|uniform, --threads, --in, --out

JSON keys and CSV columns keep the reference order (bench_main.cpp:332-402); `wall_ns` is
device time (CUDA events) per call, median over --repeats.  Workloads come from the
reference generator (mt19937_64 + normal/uniform, seeds s+3u, s+3u+1, s+3u+2;
vmb_workload_fill in libvmb).  --verify on compares against an fp64 reference computed on
the device: the materialised Monarch map M[j*b+i, k*b+l] = L[i,j,k] R[k,i,l] applied to V
(oracle.cpp:72-90) with the dense first-frame rows, or dense attention for dense/flash
(bench_main.cpp:180-198) -- capped at N <= 8192 like the reference (exit code 2 above it).
Precision: f32 runs the fp32 parity kernels, bf16 the tcgen05 path (the reference's f64 has
no GPU counterpart and is refused).  Exit codes: 0 ok, 1 error, 2 refusal.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

VERIFY_CAP = 8192  # bench_main.cpp:31 (dense oracle memory cap)
PRESETS = {"wan-61f": (16, 28, 52), "wan-141f": (36, 28, 52), "wan-321f": (81, 28, 52)}  # video.cpp:5-11
CSV_HEADER = ("mode,precision,seed,n,d,m,b,iters,heads,batch,clamp,clamp_min,recompute,br,bc,dist,"
              "threads,repeats,wall_ns_median,macs,sparsity,sparsity_approx,monarch_flops,"
              "full_attn_flops,recompute_flops,reduction_ratio,max_abs_err,rel_fro_err")
SWEEP_HEADER = ("T,h,w,n,d,iters,precision,seed,dense_wall_ns,monarch_wall_ns,speedup,dense_macs,"
                "monarch_macs,sparsity,max_abs_err,status")


class Refusal(Exception):
    """Validation refusal: exit code 2 (bench_main.cpp:33-36)."""


def fmt_double(v: float) -> str:
    """C++ ostream with precision 12 (bench_main.cpp:372-377)."""
    s = f"{v:.12g}"
    return s


def parse_args(argv):
    ap = argparse.ArgumentParser(prog="vmb_bench", description="Monarch-factorized attention benchmark harness (B200)")
    ap.add_argument("--mode", choices=["dense", "flash", "monarch", "vmonarch"])
    ap.add_argument("--preset", default="")
    ap.add_argument("--grid", dest="grid_spec", default="")
    ap.add_argument("--t", dest="iters", type=int, default=2)
    ap.add_argument("--clamp-min", type=float, default=0.1)
    ap.add_argument("--no-clamp", action="store_true")
    ap.add_argument("--no-recompute", action="store_true")
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--b", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--heads", type=int, default=1)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--br", type=int, default=64)
    ap.add_argument("--bc", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--verify", choices=["on", "off"], default="off")
    ap.add_argument("--precision", choices=["f32", "f64", "bf16"], default="f32")
    ap.add_argument("--csv", action="store_true")
    ap.add_argument("--dist", choices=["normal", "uniform"], default="normal")
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--in", dest="in_path", default="")
    ap.add_argument("--out", dest="out_path", default="")
    ap.add_argument("--sweep", dest="sweep_spec", default="")
    return ap.parse_args(argv)


def resolve_grid(opt):
    """bench_main.cpp:92-107."""
    if opt.preset:
        if opt.preset not in PRESETS:
            raise ValueError(f"unknown preset '{opt.preset}'")
        return PRESETS[opt.preset]
    if opt.grid_spec:
        parts = opt.grid_spec.split("x")
        try:
            t, h, w = (int(x) for x in parts)
        except ValueError:
            raise ValueError("--grid expects TxHxW, e.g. 16x28x52")
        if len(parts) != 3 or t < 1 or h < 1 or w < 1:
            raise ValueError("--grid expects TxHxW, e.g. 16x28x52")
        return (t, h, w)
    return None


class Runner:
    def __init__(self, opt):
        import torch

        import paper_2601_22275_b200 as vm
        self.torch, self.vm, self.opt = torch, vm, opt
        if opt.precision == "f64":
            raise ValueError("precision f64 has no GPU path (use f32 for the parity kernels or bf16)")
        if not torch.cuda.is_available():
            raise RuntimeError("vmb_bench runs on a CUDA device (no CPU path)")
        self.dev = torch.device("cuda", 0)
        self.dtype = torch.float32 if opt.precision == "f32" else torch.bfloat16
        fill = vm.lib.vmb_workload_fill
        fill.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_void_p]
        fill.restype = C.c_int
        self._fill = fill

    # -------------------------------------------------------------- workloads
    def random_mat(self, rows, cols, seed):
        import numpy as np
        a = np.empty((rows, cols), dtype=np.float32)
        st = self._fill(seed & 0xFFFFFFFFFFFFFFFF, rows * cols, 1 if self.opt.dist == "uniform" else 0,
                        a.ctypes.data_as(C.c_void_p))
        if st != 0:
            raise RuntimeError("workload generation failed")
        return a

    def workload(self, n, units):
        """bench_main.cpp:149-175: per unit Q, K, V from seeds s+3u, s+3u+1, s+3u+2, or --in."""
        import numpy as np
        opt = self.opt
        if opt.in_path:
            from paper_2601_22275_b200.matn import MatnError, read_matn
            if units != 1:
                raise ValueError("--in supports a single batch*head unit")
            arr = read_matn(opt.in_path)
            if arr.ndim != 3:
                raise MatnError(f"matn: field 'rank': expected rank 3, got {arr.ndim}")
            if arr.shape[0] != 3:
                raise MatnError("matn: field 'dims': --in expects a (3, N, d) stack of Q, K, V")
            arr = arr.astype(np.float32)
            q, k, v = (arr[i][None] for i in range(3))
        else:
            q = np.stack([self.random_mat(n, opt.d, opt.seed + 3 * u) for u in range(units)])
            k = np.stack([self.random_mat(n, opt.d, opt.seed + 3 * u + 1) for u in range(units)])
            v = np.stack([self.random_mat(n, opt.d, opt.seed + 3 * u + 2) for u in range(units)])
        t = self.torch
        return tuple(t.from_numpy(np.ascontiguousarray(x)).to(self.dev, self.dtype) for x in (q, k, v))

    # -------------------------------------------------------------- timing
    def timed(self, fn):
        t = self.torch
        runs, out = [], None
        for _ in range(max(1, self.opt.repeats)):
            e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            t.cuda.synchronize()
            runs.append(int(round(e0.elapsed_time(e1) * 1e6)))
        return out, runs

    # -------------------------------------------------------------- fp64 device references
    def dense_ref(self, q, k, v):
        t = self.torch
        q64, k64, v64 = q.double(), k.double(), v.double()
        s = q64 @ k64.transpose(-1, -2) / math.sqrt(q.shape[-1])
        return t.softmax(s, dim=-1) @ v64

    def monarch_ref(self, L, R, v, b, recompute_rows, q, k):
        """oracle.cpp:72-90 materialize_monarch + bench_main.cpp:180-198 first-frame rows."""
        t = self.torch
        Lb = L.double()  # (b, m, m): L[i, j, k]
        Rb = R.double()  # (m, b, b): R[k, i, l]
        m = Lb.shape[1]
        n = m * b
        # M[j*b+i, k*b+l] = L[i,j,k] R[k,i,l]
        M = t.einsum("ijk,kil->jikl", Lb, Rb).reshape(n, n)
        ref = M @ v.double()
        if recompute_rows > 0:
            ref[:recompute_rows] = self.dense_ref(q[:recompute_rows], k, v)
        return ref

    @staticmethod
    def err_vs(got, ref):
        diff = got.double() - ref
        max_abs = float(diff.abs().max().item()) if diff.numel() else 0.0
        den = float(ref.pow(2).sum().item())
        num = float(diff.pow(2).sum().item())
        rel = math.sqrt(num / den) if den > 0 else math.sqrt(num)
        return max_abs, rel

    # -------------------------------------------------------------- modes (bench_main.cpp:209-330)
    def run_mode(self):
        opt, vm, t = self.opt, self.vm, self.torch
        grid = resolve_grid(opt)
        n = grid[0] * grid[1] * grid[2] if grid else opt.n
        if n <= 0 and not opt.in_path:
            raise ValueError("sequence length missing: pass --n, --grid, --preset or --in")
        verify = opt.verify == "on"

        def cap(actual_n):
            if verify and actual_n > VERIFY_CAP:
                raise Refusal(f"verify requires N <= {VERIFY_CAP} (dense oracle memory cap); got N = {actual_n}")

        cap(n)
        out = {"n": n, "d": opt.d, "m": 0, "b": 0, "macs": 0, "cost": None, "err": None, "runs": []}
        if opt.mode in ("dense", "flash"):
            q, k, v = self.workload(n, 1)
            n, d = q.shape[1], q.shape[2]
            cap(n)
            out.update(n=n, d=d)
            if opt.mode == "dense":
                o, runs = self.timed(lambda: vm.dense_forward(q, k, v))
            else:
                qs = q * (1.0 / math.sqrt(d))
                o, runs = self.timed(lambda: vm.flash_entropy_fwd(qs, k, v, want_entropy=False)[0])
            out["runs"] = runs
            out["macs"] = 2 * n * n * d
            if verify:
                out["err"] = self.err_vs(o[0], self.dense_ref(q[0], k[0], v[0]))
            return out

        if opt.mode == "monarch":
            m, b = opt.m, opt.b
            if grid:
                m, b = vm.factorize(vm.TokenGrid(*grid, opt.d, 1, 1), self.vcfg())
            if m <= 0 or b <= 0:
                raise ValueError("monarch mode needs --m/--b or a grid/preset")
            q, k, v = self.workload(n, 1)
            n, d = q.shape[1], q.shape[2]
            if m * b != n:
                raise ValueError("dimension error: m*b must equal N")
            cap(n)
            out.update(n=n, d=d, m=m, b=b)
            pg = vm.TokenGrid(m, 1, b, d, 1, 1)  # monarch_attention == the grid path without recompute
            cfg = self.vcfg(recompute=False, override=False)
            factors = [] if verify else None
            o, runs = self.timed(lambda: vm.vmonarch_attention(q, k, v, pg, cfg, factors_out=factors))
            out["runs"] = runs
            rep = vm.flops_estimate(pg, cfg, d)
            out["cost"] = rep
            out["macs"] = rep.monarch_flops // 2
            if verify:
                L, R = factors[0]
                out["err"] = self.err_vs(o[0], self.monarch_ref(L, R, v[0], b, 0, q[0], k[0]))
            return out

        if opt.mode == "vmonarch":
            if not grid:
                raise ValueError("vmonarch mode needs --grid or --preset")
            g = vm.TokenGrid(*grid, opt.d, opt.heads, opt.batch)
            cfg = self.vcfg()
            m, b = vm.factorize(g, cfg)
            q, k, v = self.workload(n, g.units())
            out.update(m=m, b=b, n=n, d=opt.d)
            factors = [] if verify else None
            o, runs = self.timed(lambda: vm.vmonarch_attention(q, k, v, g, cfg, factors_out=factors))
            out["runs"] = runs
            rep = vm.flops_estimate(g, cfg, opt.d)
            out["cost"] = rep
            out["macs"] = g.units() * (rep.monarch_flops + rep.recompute_flops) // 2
            if verify:
                rr = g.h * g.w if cfg.recompute_first_frame else 0
                worst = (0.0, 0.0)
                for u in range(g.units()):
                    L, R = factors[u]
                    e = self.err_vs(o[u], self.monarch_ref(L, R, v[u], b, rr, q[u], k[u]))
                    worst = (max(worst[0], e[0]), max(worst[1], e[1]))
                out["err"] = worst
            return out
        raise ValueError(f"unknown mode '{opt.mode}'")

    def vcfg(self, recompute=None, override=True):
        """bench_main.cpp:109-122."""
        opt, vm = self.opt, self.vm
        om = None
        if override and (opt.m > 0 or opt.b > 0):
            if opt.m <= 0 or opt.b <= 0:
                raise ValueError("--m and --b must be given together")
            om = (opt.m, opt.b)
        return vm.VMonarchConfig(iters=opt.iters, clamp_min=opt.clamp_min, clamp_enabled=not opt.no_clamp,
                                 recompute_first_frame=(not opt.no_recompute) if recompute is None else recompute,
                                 override_m_b=om, tiles=(opt.br, opt.bc))

    # -------------------------------------------------------------- sweep (bench_main.cpp:404-474)
    def run_sweep(self):
        opt, vm = self.opt, self.vm
        try:
            parts = [int(x) for x in opt.sweep_spec.split(":")]
        except ValueError:
            raise ValueError("--sweep expects FROM:TO[:STEP]")
        if len(parts) not in (2, 3) or (len(parts) == 3 and parts[2] < 1):
            raise ValueError("--sweep expects FROM:TO[:STEP]")
        t_from, t_to = parts[0], parts[1]
        t_step = parts[2] if len(parts) == 3 else 4
        h, w = 8, 8
        g = resolve_grid(opt)
        if g:
            h, w = g[1], g[2]
        lines = [SWEEP_HEADER]
        for T in range(t_from, t_to + 1, t_step):
            n = T * h * w
            q, k, v = self.workload(n, 1)
            d = q.shape[2]
            od, druns = self.timed(lambda: vm.dense_forward(q, k, v))
            pg = vm.TokenGrid(T, 1, h * w, d, 1, 1)
            cfg = self.vcfg(recompute=False, override=False)
            factors = [] if opt.verify == "on" and n <= VERIFY_CAP else None
            om, mruns = self.timed(lambda: vm.vmonarch_attention(q, k, v, pg, cfg, factors_out=factors))
            dmed, mmed = sorted(druns)[len(druns) // 2], sorted(mruns)[len(mruns) // 2]
            rep = vm.flops_estimate(pg, cfg, d)
            status, err_field = "ok", ""
            if opt.verify == "on":
                if n > VERIFY_CAP:
                    status = "refused:verify-cap"
                else:
                    L, R = factors[0]
                    err_field = fmt_double(self.err_vs(om[0], self.monarch_ref(L, R, v[0], h * w, 0, q[0], k[0]))[0])
            lines.append(",".join(str(x) for x in [
                T, h, w, n, d, opt.iters, opt.precision, opt.seed, dmed, mmed, fmt_double(dmed / mmed),
                2 * n * n * d, rep.monarch_flops // 2, fmt_double(rep.sparsity), err_field, status]))
        return "\n".join(lines) + "\n"


def to_json(opt, oc, grid):
    """bench_main.cpp:332-371 key order."""
    j = {"mode": opt.mode, "precision": opt.precision, "seed": opt.seed, "n": oc["n"], "d": oc["d"], "m": oc["m"],
         "b": oc["b"], "iters": opt.iters, "heads": opt.heads, "batch": opt.batch, "clamp": not opt.no_clamp,
         "clamp_min": opt.clamp_min, "recompute": not opt.no_recompute, "br": opt.br, "bc": opt.bc,
         "dist": opt.dist, "threads": opt.threads, "repeats": opt.repeats,
         "grid": {"t": grid[0], "h": grid[1], "w": grid[2]} if grid else None, "macs": oc["macs"]}
    c = oc["cost"]
    j["cost"] = None if c is None else {
        "sparsity": c.sparsity, "sparsity_approx": c.sparsity_approx, "monarch_flops": c.monarch_flops,
        "full_attn_flops": c.full_attn_flops, "recompute_flops": c.recompute_flops,
        "reduction_ratio": c.reduction_ratio}
    if oc["err"] is not None:
        j["verify"] = {"max_abs_err": oc["err"][0], "rel_fro_err": oc["err"][1]}
    runs = oc["runs"]
    j["wall_ns"] = {"median": sorted(runs)[len(runs) // 2], "runs": runs}
    j["device"] = "B200 (libvmb, sm_100a)"  # extra key after the reference ones
    return json.dumps(j, indent=2) + "\n"


def to_csv(opt, oc):
    """bench_main.cpp:379-402 column order."""
    runs = oc["runs"]
    row = [opt.mode, opt.precision, opt.seed, oc["n"], oc["d"], oc["m"], oc["b"], opt.iters, opt.heads, opt.batch,
           0 if opt.no_clamp else 1, fmt_double(opt.clamp_min), 0 if opt.no_recompute else 1, opt.br, opt.bc,
           opt.dist, opt.threads, opt.repeats, sorted(runs)[len(runs) // 2], oc["macs"]]
    c = oc["cost"]
    row += ([fmt_double(c.sparsity), fmt_double(c.sparsity_approx), c.monarch_flops, c.full_attn_flops,
             c.recompute_flops, fmt_double(c.reduction_ratio)] if c else [""] * 6)
    row += [fmt_double(oc["err"][0]), fmt_double(oc["err"][1])] if oc["err"] else ["", ""]
    return CSV_HEADER + "\n" + ",".join(str(x) for x in row) + "\n"


def main(argv=None):
    try:
        opt = parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    if not opt.mode and not opt.sweep_spec:
        print("error: --mode is required (or use --sweep)", file=sys.stderr)
        return 1
    try:
        resolve_grid(opt)  # unknown presets / malformed grids fail before any device work
        if opt.in_path:
            from paper_2601_22275_b200.matn import read_matn
            read_matn(opt.in_path)
        r = Runner(opt)
        if opt.sweep_spec:
            text = r.run_sweep()
        else:
            oc = r.run_mode()
            text = to_csv(opt, oc) if opt.csv else to_json(opt, oc, resolve_grid(opt))
        if opt.out_path:
            try:
                with open(opt.out_path, "w") as f:
                    f.write(text)
            except OSError:
                raise RuntimeError(f"cannot open --out file '{opt.out_path}'")
        else:
            sys.stdout.write(text)
        return 0
    except Refusal as e:
        print(f"refused: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 -- the reference maps every other error to exit 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
