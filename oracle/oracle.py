"""ctypes/numpy bindings for the CPU checker.  TEST INFRASTRUCTURE ONLY.

Two libraries, same calling convention:

* ``Oracle("port")``      -> oracle/liboracle.so, the C restatement (vmonarch_oracle.c)
* ``Oracle("reference")`` -> oracle/_ref/libvmref.so, the unmodified reference library
  (/root/reference/proj) compiled from its own sources with oracle/ref_shim.cpp

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may import
this module.  The product (paper_2601_22275_b200, libvmb.so) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvmref.so")

ERR = {0: None, 1: ValueError, 2: ArithmeticError, 3: RuntimeError, 4: RuntimeError}
# status -> the reference exception class it stands for (check.hpp:10-20)
ERR_NAMES = {1: "dimension error", 2: "domain error", 3: "state error", 4: "error"}


class OracleError(Exception):
    def __init__(self, status: int, what: str):
        super().__init__(f"{ERR_NAMES.get(status, 'error')}: {what}")
        self.status = status


def build() -> None:
    """Compile liboracle.so (and _ref/libvmref.so when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_INT = C.c_int


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run oracle.build())")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = "vmo_" if kind == "port" else "vmr_"

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    @staticmethod
    def _check(st, what):
        if st != 0:
            raise OracleError(st, what)

    @staticmethod
    def _sfx(dtype):
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    # ---- index work ------------------------------------------------------------
    def make_perm(self, b: int, n: int) -> np.ndarray:
        out = np.zeros(max(n, 0), dtype=np.int64)
        f = self._fn("make_perm")
        f.argtypes = [_I64, _I64, _P]
        self._check(f(b, n, _ptr(out)), "permutation requires b >= 1, n >= 1, b | n")
        return out

    def to_blocked_permuted(self, x: np.ndarray, m: int, b: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        d = x.shape[1]
        out = np.zeros((b, m, d), dtype=np.float32)
        f = self._fn("to_blocked_permuted_f32")
        f.argtypes = [_P, _I64, _I64, _I64, _P]
        self._check(f(_ptr(x), m, b, d, _ptr(out)), "blocked view requires rows == m*b")
        return out

    # ---- half steps ------------------------------------------------------------
    def rstep(self, aR, cR, Kb, clamp_min=0.1, clamp_enabled=True, want_R=True):
        dt = aR.dtype
        m, b, d = aR.shape
        aL = np.zeros((b, m, d), dt)
        cL = np.zeros((b, m), dt)
        R = np.zeros((m, b, b), dt) if want_R else None
        f = self._fn("rstep_" + self._sfx(dt))
        f.argtypes = [_I64, _I64, _I64, _P, _P, _P, _D, _INT, _P, _P, _P]
        st = f(m, b, d, _ptr(np.ascontiguousarray(aR)), _ptr(np.ascontiguousarray(cR, dtype=dt)),
               _ptr(np.ascontiguousarray(Kb, dtype=dt)), clamp_min, int(clamp_enabled),
               _ptr(aL), _ptr(cL), _ptr(R))
        self._check(st, "r_update")
        return aL, cL, R

    def lstep(self, Qb, aL, cL, want_L=True):
        dt = Qb.dtype
        b, m, d = Qb.shape
        aR = np.zeros((m, b, d), dt)
        cR = np.zeros((m, b), dt)
        L = np.zeros((b, m, m), dt) if want_L else None
        f = self._fn("lstep_" + self._sfx(dt))
        f.argtypes = [_I64, _I64, _I64, _P, _P, _P, _P, _P, _P]
        st = f(m, b, d, _ptr(np.ascontiguousarray(Qb)), _ptr(np.ascontiguousarray(aL, dtype=dt)),
               _ptr(np.ascontiguousarray(cL, dtype=dt)), _ptr(aR), _ptr(cR), _ptr(L))
        self._check(st, "l_update")
        return aR, cR, L

    # ---- whole operators -------------------------------------------------------
    def monarch_attention(self, q, k, v, m, b, iters=2, clamp_min=0.1, clamp_enabled=True,
                          want_factors=False):
        dt = q.dtype
        n, d = q.shape
        out = np.zeros((n, d), dt)
        L = np.zeros((b, m, m), dt) if want_factors else None
        R = np.zeros((m, b, b), dt) if want_factors else None
        f = self._fn("monarch_attention_" + self._sfx(dt))
        f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I64, _D, _INT, _P, _P, _P]
        st = f(_ptr(np.ascontiguousarray(q)), _ptr(np.ascontiguousarray(k, dtype=dt)),
               _ptr(np.ascontiguousarray(v, dtype=dt)), m, b, d, iters, clamp_min,
               int(clamp_enabled), _ptr(out), _ptr(L), _ptr(R))
        self._check(st, "monarch_attention")
        return (out, L, R) if want_factors else out

    def flash_entropy_fwd(self, q, k, v, br=64, bc=64):
        dt = q.dtype
        nq, d = q.shape
        nk = k.shape[0]
        out = np.zeros((nq, d), dt)
        lse = np.zeros(nq, dt)
        ent = np.zeros(nq, dt)
        f = self._fn("flash_entropy_fwd_" + self._sfx(dt))
        f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P]
        st = f(_ptr(np.ascontiguousarray(q)), _ptr(np.ascontiguousarray(k, dtype=dt)),
               _ptr(np.ascontiguousarray(v, dtype=dt)), nq, nk, d, br, bc, _ptr(out), _ptr(lse),
               _ptr(ent))
        self._check(st, "flash_entropy_fwd")
        return out, lse, ent

    def flash_entropy_bwd(self, q, k, v, o, dout, lse, ent=None, dent=None, entropy_grad=False, br=64, bc=64):
        """flash_entropy.hpp:146-221 -> (dq, dk, dv)."""
        dt = q.dtype
        nq, d = q.shape
        nk = k.shape[0]
        dq = np.zeros((nq, d), dt)
        dk = np.zeros((nk, d), dt)
        dv = np.zeros((nk, d), dt)
        f = self._fn("flash_entropy_bwd_" + self._sfx(dt))
        f.argtypes = [_P] * 8 + [_I64, _I64, _I64, _INT, _I64, _I64, _P, _P, _P]
        c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=dt)  # noqa: E731
        ins = [c(q), c(k), c(v), c(o), c(dout), c(lse), c(ent), c(dent)]
        st = f(*[_ptr(a) for a in ins], nq, nk, d, int(entropy_grad), br, bc, _ptr(dq), _ptr(dk), _ptr(dv))
        self._check(st, "flash_entropy_bwd")
        return dq, dk, dv

    def vmonarch_attention(self, q, k, v, grid, iters=2, clamp_min=0.1, clamp_enabled=True,
                           recompute=True, override=(0, 0), threads=1, tiles=(64, 64)):
        """q,k,v: (units, N, d).  grid = (T, h, w).  Returns (units, N, d)."""
        dt = q.dtype
        units, n, d = q.shape
        tf, h, w = grid
        out = np.zeros_like(q)
        if self.kind == "reference":
            f = self._fn("vmonarch_attention_" + self._sfx(dt))
            f.argtypes = [_I64, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _D, _INT, _INT, _I64,
                          _I64, _INT, _P]
            st = f(units, _ptr(np.ascontiguousarray(q)), _ptr(np.ascontiguousarray(k, dtype=dt)),
                   _ptr(np.ascontiguousarray(v, dtype=dt)), tf, h, w, d, iters, clamp_min,
                   int(clamp_enabled), int(recompute), override[0], override[1], threads,
                   _ptr(out))
            self._check(st, "vmonarch_attention")
            return out
        f = self._fn("vmonarch_unit_" + self._sfx(dt))
        f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _D, _INT, _INT, _I64, _I64, _I64,
                      _I64, _P, _P, _P]
        q = np.ascontiguousarray(q)
        k = np.ascontiguousarray(k, dtype=dt)
        v = np.ascontiguousarray(v, dtype=dt)
        for u in range(units):
            o = np.zeros((n, d), dt)
            st = f(_ptr(q[u]), _ptr(k[u]), _ptr(v[u]), tf, h, w, d, iters, clamp_min,
                   int(clamp_enabled), int(recompute), override[0], override[1], tiles[0],
                   tiles[1], _ptr(o), None, None)
            self._check(st, "vmonarch_attention")
            out[u] = o
        return out

    def dense_attention_f64(self, q, k, v, scale=True, want_probs=False):
        q = np.ascontiguousarray(q, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        nq, d = q.shape
        nk = k.shape[0]
        out = np.zeros((nq, d))
        lse = np.zeros(nq)
        ent = np.zeros(nq)
        f = self._fn("dense_attention_f64")
        if self.kind == "port":
            probs = np.zeros((nq, nk)) if want_probs else None
            f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _INT, _P, _P, _P, _P]
            st = f(_ptr(q), _ptr(k), _ptr(v), nq, nk, d, int(scale), _ptr(out), _ptr(lse),
                   _ptr(ent), _ptr(probs))
            self._check(st, "dense_attention")
            return (out, lse, ent, probs) if want_probs else (out, lse, ent)
        f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _INT, _P, _P, _P]
        self._check(f(_ptr(q), _ptr(k), _ptr(v), nq, nk, d, int(scale), _ptr(out), _ptr(lse),
                      _ptr(ent)), "dense_attention")
        return out, lse, ent

    def materialize_monarch(self, L, R, b, n):
        out = np.zeros((n, n))
        f = self.lib.vmo_materialize_monarch_f64
        f.argtypes = [_P, _P, _I64, _I64, _P]
        self._check(f(_ptr(np.ascontiguousarray(L, dtype=np.float64)),
                      _ptr(np.ascontiguousarray(R, dtype=np.float64)), b, n, _ptr(out)),
                    "materialize")
        return out

    def monarch_objective(self, L, R, q, k, m, b, scale=True):
        res = C.c_double(0.0)
        f = self.lib.vmo_monarch_objective_f64
        f.argtypes = [_P, _P, _P, _P, _I64, _I64, _I64, _INT, C.POINTER(C.c_double)]
        q = np.ascontiguousarray(q, dtype=np.float64)
        self._check(f(_ptr(np.ascontiguousarray(L, dtype=np.float64)),
                      _ptr(np.ascontiguousarray(R, dtype=np.float64)), _ptr(q),
                      _ptr(np.ascontiguousarray(k, dtype=np.float64)), m, b, q.shape[1],
                      int(scale), C.byref(res)), "objective")
        return res.value

    def dense_forward(self, q, k, v, scale=True):
        dt = q.dtype
        nq, d = q.shape
        out = np.zeros((nq, d), dt)
        f = self.lib["vmo_dense_forward_" + self._sfx(dt)]
        f.argtypes = [_P, _P, _P, _I64, _I64, _I64, _INT, _P]
        self._check(f(_ptr(np.ascontiguousarray(q)), _ptr(np.ascontiguousarray(k, dtype=dt)),
                      _ptr(np.ascontiguousarray(v, dtype=dt)), nq, k.shape[0], d, int(scale),
                      _ptr(out)), "dense_forward")
        return out

    def flops_estimate(self, grid, d, iters=2, recompute=True, override=(0, 0)):
        tf, h, w = grid
        if self.kind == "port":

            class Rep(C.Structure):
                _fields_ = [("sparsity", C.c_double), ("sparsity_approx", C.c_double),
                            ("monarch_flops", C.c_uint64), ("full_attn_flops", C.c_uint64),
                            ("recompute_flops", C.c_uint64), ("reduction_ratio", C.c_double)]

            rep = Rep()
            f = self.lib.vmo_flops_estimate
            f.argtypes = [_I64, _I64, _I64, _I64, _I64, _I64, _INT, _I64, C.POINTER(Rep)]
            self._check(f(tf, h, w, override[0], override[1], iters, int(recompute), d,
                          C.byref(rep)), "flops_estimate")
            return {k: getattr(rep, k) for k, _ in Rep._fields_}
        vals = [C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_double()]
        f = self.lib.vmr_flops_estimate
        f.argtypes = [_I64] * 6 + [_INT, _I64] + [C.c_void_p] * 6
        self._check(f(tf, h, w, override[0], override[1], iters, int(recompute), d,
                      *[C.addressof(x) for x in vals]), "flops_estimate")
        keys = ["sparsity", "sparsity_approx", "monarch_flops", "full_attn_flops",
                "recompute_flops", "reduction_ratio"]
        return {k: x.value for k, x in zip(keys, vals)}


def randn(shape, seed: int, sigma: float = 1.0, dtype=np.float32) -> np.ndarray:
    """Reference-convention N(0, sigma) tensor (std::mt19937_64 + normal_distribution)."""
    lib = C.CDLL(PORT_SO)
    n = int(np.prod(shape))
    if np.dtype(dtype) == np.float32:
        out = np.zeros(n, np.float32)
        lib.vmo_randn_f32.argtypes = [_I64, C.c_uint64, _D, _P]
        lib.vmo_randn_f32(n, seed, sigma, _ptr(out))
    else:
        out = np.zeros(n, np.float64)
        lib.vmo_randn_f64.argtypes = [_I64, C.c_uint64, _D, _P]
        lib.vmo_randn_f64(n, seed, sigma, _ptr(out))
    return out.reshape(shape)


def workload(units: int, n: int, d: int, seed: int = 0, sigma: float = 1.0, dtype=np.float32):
    """bench_main.cpp:169-173 convention: Q, K, V of unit u use seeds s+3u, s+3u+1, s+3u+2."""
    q = np.stack([randn((n, d), seed + 3 * u, sigma, dtype) for u in range(units)])
    k = np.stack([randn((n, d), seed + 3 * u + 1, sigma, dtype) for u in range(units)])
    v = np.stack([randn((n, d), seed + 3 * u + 2, sigma, dtype) for u in range(units)])
    return q, k, v


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (the bf16 inputs' exact values)."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)
