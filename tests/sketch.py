"""Seeded random-sign sketches of large images (full-image parity gates without full goldens).

``sketch(u, k)`` returns ``s_j = sum_i rho_j(i) u_i`` for ``j < k``, the signs ``rho_j(i)``
drawn from a splitmix64 hash of ``(i, j)``.  For two images ``E ||S(u - w)||^2 / k =
||u - w||^2`` (a Johnson-Lindenstrauss estimate; relative spread ``sqrt(2 / k)``), so a
committed ``k``-vector of the reference's image gates the L2 difference over EVERY pixel,
where a stored subsample only sees a fraction of them.  Used by ``tests/golden/make_golden.py``
(on the reference's outputs) and by the GPU parity tests (on the device's outputs).
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _signs(idx: np.ndarray, j: int) -> np.ndarray:
    z = idx + np.uint64(j + 1) * _GOLD
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    z = z ^ (z >> np.uint64(31))
    return 1.0 - 2.0 * (z >> np.uint64(63)).astype(np.float64)


def sketch(u, k: int = 32, chunk: int = 1 << 22) -> np.ndarray:
    """``k`` seeded random-sign projections of ``u`` (any shape, flattened C order)."""
    flat = np.ascontiguousarray(np.asarray(u, dtype=np.float64)).ravel()
    out = np.zeros(k)
    with np.errstate(over="ignore"):
        for c0 in range(0, flat.size, chunk):
            part = flat[c0:c0 + chunk]
            idx = np.arange(c0, c0 + part.size, dtype=np.uint64)
            for j in range(k):
                out[j] += float(np.dot(_signs(idx, j), part))
    return out


def sketch_rel_err(u, ref_sketch: np.ndarray, ref_norm: float) -> float:
    """JL estimate of ``||u - ref|| / ||ref||`` from the reference's sketch and norm."""
    s = sketch(u, len(ref_sketch))
    return float(np.linalg.norm(s - ref_sketch) / np.sqrt(len(ref_sketch)) / ref_norm)


def _signs_torch(idx, j: int):
    """``_signs`` on int64 torch tensors (same bit patterns: multiplication wraps mod 2^64,
    logical right shifts by masking)."""
    import torch

    def srl(z, s):
        return (z >> s) & ((1 << (64 - s)) - 1)

    def c64(v: int) -> int:  # a uint64 constant as the int64 with the same bits
        return v - (1 << 64) if v >= 1 << 63 else v

    z = idx + c64(((j + 1) * int(_GOLD)) % (1 << 64))
    z = (z ^ srl(z, 30)) * c64(int(_M1))
    z = (z ^ srl(z, 27)) * c64(int(_M2))
    z = z ^ srl(z, 31)
    return 1.0 - 2.0 * (z < 0).to(torch.float64)


def sketch_torch(t, k: int = 32, chunk: int = 1 << 24) -> np.ndarray:
    """:func:`sketch` of a torch tensor on its own device (the same projections)."""
    import torch

    flat = t.reshape(-1).to(torch.float64)
    out = np.zeros(k)
    for c0 in range(0, flat.numel(), chunk):
        part = flat[c0:c0 + chunk]
        idx = torch.arange(c0, c0 + part.numel(), dtype=torch.int64, device=part.device)
        for j in range(k):
            out[j] += float(torch.dot(_signs_torch(idx, j), part))
    return out
