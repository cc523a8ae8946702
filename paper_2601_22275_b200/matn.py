"""MATN binary tensors (matn_io.hpp:12-23, matn_io.cpp:39-90): the reference bench's `--in`
format and the golden-exchange format of this repo.

Layout: magic "MATN", u32 version = 1, u32 rank (1..8), rank x u64 dims, u8 dtype (0 = f32,
1 = f64), little-endian row-major payload, nothing after it.  Errors name the offending field
like the reference ("matn: field 'magic': expected \\"MATN\\"").
"""
from __future__ import annotations

import struct

import numpy as np


class MatnError(RuntimeError):
    pass


def _fail(field: str, what: str):
    raise MatnError(f"matn: field '{field}': {what}")


def read_matn(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise MatnError(f"matn: cannot open '{path}'")
    with f:
        data = f.read()
    pos = 0

    def take(n, field):
        nonlocal pos
        if pos + n > len(data):
            _fail(field, "unexpected end of file")
        out = data[pos:pos + n]
        pos += n
        return out

    if take(4, "magic") != b"MATN":
        _fail("magic", 'expected "MATN"')
    (version,) = struct.unpack("<I", take(4, "version"))
    if version != 1:
        _fail("version", f"unsupported version {version}")
    (rank,) = struct.unpack("<I", take(4, "rank"))
    if rank == 0 or rank > 8:
        _fail("rank", f"rank {rank} out of range [1,8]")
    dims = [struct.unpack("<Q", take(8, "dims"))[0] for _ in range(rank)]
    count = 1
    for d in dims:
        if d == 0:
            _fail("dims", "zero-sized dimension")
        count *= d
    (dtype,) = struct.unpack("<B", take(1, "dtype"))
    if dtype > 1:
        _fail("dtype", "expected 0 (f32) or 1 (f64)")
    np_dt = np.dtype("<f4") if dtype == 0 else np.dtype("<f8")
    payload = take(count * np_dt.itemsize, "payload")
    if pos != len(data):
        _fail("payload", "trailing bytes after payload")
    return np.frombuffer(payload, dtype=np_dt).reshape(dims).copy()


def write_matn(path: str, arr: np.ndarray) -> None:
    arr = np.ascontiguousarray(arr)
    if arr.dtype == np.float32:
        dtype = 0
    elif arr.dtype == np.float64:
        dtype = 1
    else:
        raise MatnError("matn: field 'dtype': expected float32 or float64")
    if not 1 <= arr.ndim <= 8:
        _fail("rank", f"rank {arr.ndim} out of range [1,8]")
    with open(path, "wb") as f:
        f.write(b"MATN")
        f.write(struct.pack("<II", 1, arr.ndim))
        for d in arr.shape:
            f.write(struct.pack("<Q", d))
        f.write(struct.pack("<B", dtype))
        f.write(arr.astype(arr.dtype.newbyteorder("<"), copy=False).tobytes())
