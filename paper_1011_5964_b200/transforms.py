"""Fast trigonometric transforms on the GPU (mirror of reference transforms.py).

Same names and semantics as ``tvdeblur.transforms`` (transforms.py:29-171):
``dst1_apply`` (orthonormal DST-I, self-inverse), ``dct_apply`` (forward =
synthesis ``C v`` = DCT-III, ``inverse=True`` = analysis ``C^T v`` =
DCT-II), ``sinehat_apply`` (``diag(1, S_{n-2}, 1)``), ``apply_1d`` and
``tensor_apply_2d`` (axis 0 then axis 1).  Inputs may be numpy arrays (a
numpy array is returned) or CUDA tensors (a CUDA tensor is returned); every
transform runs in the sm_100a line-FFT kernels of ``csrc/tvd_lines.cu``.

The anti-reflective transform ``T = Shat (I + U)`` (transforms.py:84-140) feeds the P
preconditioner family and the transform-domain blur (blur.py:293-314).  ``ar_apply`` runs
``T``, ``T^-1``, ``T^T`` and ``T^-T`` over lines on the device (``tvd_ar_lines``: Shat line
passes plus the rank-2 factor as correction / projection kernels); ``tensor_apply_2d``
applies ``T (x) T`` and its inverse with the corrections fused into the pipelined DST row
passes (odd cores with the prime-factor engine) and the transposed forms axis by axis.
"""

from __future__ import annotations

from enum import Enum

import numpy as np
import torch

from . import _native as nat


class TransformKind(Enum):
    DCT = "dct"
    DST1 = "dst1"
    ANTI_REFLECTIVE = "anti_reflective"
    SINE_HAT = "sine_hat"


_CODES = {TransformKind.DST1: nat.T_DST1, TransformKind.SINE_HAT: nat.T_SINE_HAT,
          TransformKind.DCT: nat.T_DCT, TransformKind.ANTI_REFLECTIVE: nat.T_ANTI_REFLECTIVE}


def _lines(kind: TransformKind, v, inverse: bool, axis: int, transpose: bool = False):
    t, was_np = nat.to_device(v)
    if t.ndim == 0:
        raise ValueError("transform input must be at least 1D")
    axis = axis % t.ndim
    length = t.shape[axis]
    if length == 0:
        raise ValueError("transform input must be non-empty")
    if kind is TransformKind.SINE_HAT and length < 3:
        raise ValueError(f"Shat_n requires length >= 3, got {length}")
    if kind is TransformKind.ANTI_REFLECTIVE and length < 3:
        raise ValueError(f"T_n requires length >= 3, got {length}")
    moved = torch.movedim(t, axis, -1).contiguous()
    rows = moved.numel() // length
    flat = moved.reshape(rows, length)
    out = torch.empty_like(flat)
    ctx = nat.context(flat.device)
    if kind is TransformKind.ANTI_REFLECTIVE:
        nat.check(nat.load().tvd_ar_lines(ctx, rows, length, flat.data_ptr(), out.data_ptr(),
                                          1 if inverse else 0, 1 if transpose else 0))
    else:
        nat.check(nat.load().tvd_transform_lines(ctx, _CODES[kind], rows, length, 1,
                                                 flat.data_ptr(), out.data_ptr(),
                                                 1 if inverse else 0))
    res = torch.movedim(out.reshape(moved.shape), -1, axis)
    return nat.to_host_like(res.contiguous(), was_np)


def dst1_apply(v, axis: int = -1):
    """Symmetric, self-inverse type-I sine transform ``S_n`` (transforms.py:52-56)."""
    return _lines(TransformKind.DST1, v, False, axis)


def dct_apply(v, inverse: bool = False, axis: int = -1):
    """``C v`` (forward, synthesis) or ``C^T v`` (``inverse``, analysis) (transforms.py:59-69)."""
    return _lines(TransformKind.DCT, v, inverse, axis)


def sinehat_apply(v, axis: int = -1):
    """``Shat_n = diag(1, S_{n-2}, 1)`` (transforms.py:72-81)."""
    return _lines(TransformKind.SINE_HAT, v, False, axis)


def ar_apply(v, inverse: bool = False, transpose: bool = False, axis: int = -1):
    """``T_n``, ``T_n^-1``, ``T_n^T`` or ``T_n^-T`` along ``axis`` through the rank-2
    factorization ``T = Shat (I + U)`` (transforms.py:96-140)."""
    return _lines(TransformKind.ANTI_REFLECTIVE, v, inverse, axis, transpose)


def apply_1d(kind: TransformKind, v, inverse: bool = False, transpose: bool = False, axis: int = -1):
    """Dispatch a 1D transform along ``axis`` (transforms.py:143-156)."""
    if kind is TransformKind.DCT and transpose:
        inverse = not inverse
    if kind not in (TransformKind.DCT, TransformKind.DST1, TransformKind.SINE_HAT,
                    TransformKind.ANTI_REFLECTIVE):
        raise ValueError(f"unknown transform kind: {kind!r}")
    if kind is TransformKind.ANTI_REFLECTIVE:
        return ar_apply(v, inverse=inverse, transpose=transpose, axis=axis)
    return _lines(kind, v, inverse if kind is TransformKind.DCT else False, axis)


def tensor_apply_2d(kind: TransformKind, g, inverse: bool = False, transpose: bool = False):
    """``X G X^T`` on a square grid (transforms.py:159-171)."""
    t, was_np = nat.to_device(g)
    if t.ndim != 2 or t.shape[0] != t.shape[1]:
        raise ValueError(f"tensor transform needs a square grid, got shape {tuple(t.shape)}")
    if kind is TransformKind.ANTI_REFLECTIVE and transpose:
        # T^T (x) T^T / T^-T (x) T^-T: the 1D transposed form over axis 0, then axis 1
        out = ar_apply(t, inverse=inverse, transpose=True, axis=0)
        out = ar_apply(out, inverse=inverse, transpose=True, axis=1)
        return nat.to_host_like(out, was_np)
    if kind is TransformKind.DCT and transpose:
        inverse = not inverse
    n = t.shape[0]
    if kind is TransformKind.SINE_HAT and n < 3:
        raise ValueError(f"Shat_n requires length >= 3, got {n}")
    if kind is TransformKind.ANTI_REFLECTIVE and n < 3:
        raise ValueError(f"T_n requires length >= 3, got {n}")
    out = torch.empty_like(t)
    ctx = nat.context(t.device)
    nat.check(nat.load().tvd_transform_2d(ctx, _CODES[kind], n, t.data_ptr(), out.data_ptr(),
                                          1 if inverse else 0))
    return nat.to_host_like(out, was_np)


def dense_matrix(kind: TransformKind, n: int, inverse: bool = False) -> np.ndarray:
    """Transform matrix from its defining formula (transforms.py:174-212; oracle helper)."""
    if n < 1:
        raise ValueError("n must be positive")
    if kind is TransformKind.DCT:
        i = np.arange(n)[:, None]
        j = np.arange(n)[None, :]
        c = np.sqrt((2.0 - (j == 0)) / n) * np.cos((2 * i + 1) * j * np.pi / (2 * n))
        return c.T if inverse else c
    if kind is TransformKind.DST1:
        ij = np.outer(np.arange(1, n + 1), np.arange(1, n + 1))
        return np.sqrt(2.0 / (n + 1)) * np.sin(ij * np.pi / (n + 1))
    if kind is TransformKind.SINE_HAT:
        if n < 3:
            raise ValueError("sine_hat requires n >= 3")
        out = np.zeros((n, n))
        out[0, 0] = out[-1, -1] = 1.0
        out[1:-1, 1:-1] = dense_matrix(TransformKind.DST1, n - 2)
        return out
    if kind is TransformKind.ANTI_REFLECTIVE:
        # T = Shat (I + U): identity borders, S_{n-2} in the interior, and the two ramp columns
        # p_j = 1 - j / (n - 1) (forward) or -S p (inverse) under the border entries
        if n < 3:
            raise ValueError("anti_reflective requires n >= 3")
        core = dense_matrix(TransformKind.DST1, n - 2)
        ramp = 1.0 - np.arange(1, n - 1) / (n - 1)
        out = np.zeros((n, n))
        out[0, 0] = out[-1, -1] = 1.0
        out[1:-1, 1:-1] = core
        out[1:-1, 0] = -(core @ ramp) if inverse else ramp
        out[1:-1, -1] = -(core @ ramp[::-1]) if inverse else ramp[::-1]
        return out
    raise ValueError(f"unknown transform kind: {kind!r}")
