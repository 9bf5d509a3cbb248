"""ctypes binding of the C ABI in ``include/tvdeblur_b200.h``.

This is the only place the Python mirror touches native code.  There is no
CPU fallback: every operator in this package fails loudly (``RuntimeError``)
when the library or a CUDA device is missing.  Device memory is owned by
torch tensors; their raw pointers cross the ABI together with the current
torch stream of the device.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

import numpy as np
import torch

_LIB_PATH = pathlib.Path(__file__).resolve().parent / "libtvdeblur_b200.so"
_lib = None
_lock = threading.Lock()

TVD_OK, TVD_ERR_INVALID, TVD_ERR_DIVERGED, TVD_ERR_INDEFINITE = 0, 1, 2, 3
TVD_ERR_PRECOND, TVD_ERR_SCALING, TVD_ERR_CUDA, TVD_ERR_BREAKDOWN = 4, 5, 6, 7
BC_REFLECTIVE, BC_ANTI_REFLECTIVE = 2, 3
T_DST1, T_SINE_HAT, T_DCT, T_ANTI_REFLECTIVE = 0, 1, 2, 3
DBC_ZERO_NEUMANN, DBC_ANTI_REFLECTIVE = 0, 1
VARIANT_X, VARIANT_D_X, VARIANT_X_D = 0, 1, 2
PRE_NONE, PRE_DIAG, PRE_TRANSFORM = 0, 1, 2

_vp = ctypes.c_void_p
_i = ctypes.c_int
_d = ctypes.c_double
_ll = ctypes.c_longlong


class TvdSystem(ctypes.Structure):
    _fields_ = [("blur", _vp), ("alpha", _d), ("spacing", _d),
                ("a_h", _vp), ("a_v", _vp), ("s", _vp), ("bc_l", _i), ("reblur", _i)]


class TvdPrecond(ctypes.Structure):
    _fields_ = [("kind", _i), ("family", _i), ("inv_eig", _vp), ("d", _vp)]


_SIGNATURES = {
    "tvd_abi_version": ([], _i),
    "tvd_last_error": ([], ctypes.c_char_p),
    "tvd_ctx_create": ([_i, _vp, ctypes.POINTER(_vp)], _i),
    "tvd_ctx_set_stream": ([_vp, _vp], _i),
    "tvd_ctx_sync": ([_vp], _i),
    "tvd_ctx_destroy": ([_vp], _i),
    "tvd_ctx_set_option": ([_vp, _i, _i], _i),
    "tvd_ctx_get_option": ([_vp, _i, ctypes.POINTER(_i)], _i),
    "tvd_ctx_check_guards": ([_vp, ctypes.POINTER(_ll), ctypes.POINTER(_i)], _i),
    "tvd_diffusivity_rows": ([_vp, _i, _d, _d, _vp, _i, _i, _i, _i, _vp, _vp], _i),
    "tvd_diffusion_bands_rows": ([_vp, _i, _d, _vp, _vp, _i, _i, _vp, _vp, _vp], _i),
    "tvd_band_project_lines": ([_vp, _i, _i, _i, _vp, _vp, _i, _d, _i, _vp, _d, _vp,
                                ctypes.POINTER(_d)], _i),
    "tvd_ctx_counters": ([_vp, ctypes.POINTER(_ll)], _i),
    "tvd_ctx_profile": ([_vp, _i], _i),
    "tvd_ctx_profile_read": ([_vp, _i, ctypes.POINTER(_d), ctypes.POINTER(_ll)], _i),
    "tvd_profile_category": ([_i], ctypes.c_char_p),
    "tvd_blur_create": ([_vp, _i, _vp, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_i)], _i),
    "tvd_blur_destroy": ([_vp], _i),
    "tvd_blur_apply": ([_vp, _vp, _vp, _i], _i),
    "tvd_blur_normal_apply": ([_vp, _vp, _vp], _i),
    "tvd_blur_eigenvalues": ([_vp, _vp], _i),
    "tvd_diffusivity": ([_vp, _i, _d, _d, _vp, _vp, _vp], _i),
    "tvd_diffusion_apply": ([_vp, _i, _d, _vp, _vp, _vp, _vp], _i),
    "tvd_diffusion_bands": ([_vp, _i, _d, _vp, _vp, _vp, _vp, _vp], _i),
    "tvd_diffusivity_bc": ([_vp, _i, _d, _d, _i, _vp, _vp, _vp], _i),
    "tvd_diffusion_apply_bc": ([_vp, _i, _d, _i, _vp, _vp, _vp, _vp], _i),
    "tvd_diffusion_bands_bc": ([_vp, _i, _d, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "tvd_transform_lines": ([_vp, _i, _i, _i, _i, _vp, _vp, _i], _i),
    "tvd_transform_2d": ([_vp, _i, _i, _vp, _vp, _i], _i),
    "tvd_ar_lines": ([_vp, _i, _i, _vp, _vp, _i, _i], _i),
    "tvd_precond_assemble": ([_vp, _i, _i, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              ctypes.POINTER(_d), ctypes.POINTER(_d), ctypes.POINTER(_ll)], _i),
    "tvd_precond_assemble_async": ([_vp, _i, _i, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp], _i),
    "tvd_precond_apply_inverse": ([_vp, _i, _i, _vp, _vp, _vp, _vp], _i),
    "tvd_precond_apply": ([_vp, _i, _i, _vp, _vp, _vp, _vp], _i),
    "tvd_scaling": ([_vp, _ll, _d, _vp, _vp, _vp, _vp, ctypes.POINTER(_d)], _i),
    "tvd_system_apply": ([_vp, ctypes.POINTER(TvdSystem), _vp, _vp], _i),
    "tvd_pcg_solve": ([_vp, ctypes.POINTER(TvdSystem), ctypes.POINTER(TvdPrecond), _vp, _vp, _vp,
                       _d, _i, _vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i),
                       ctypes.POINTER(_d)], _i),
    "tvd_bicgstab_solve": ([_vp, ctypes.POINTER(TvdSystem), ctypes.POINTER(TvdPrecond), _vp, _vp,
                            _vp, _d, _i, _vp, ctypes.POINTER(_i), ctypes.POINTER(_i),
                            ctypes.POINTER(_i), ctypes.POINTER(_d)], _i),
    "tvd_valid_convolve": ([_vp, _vp, _i, _vp, _i, _vp, _vp, _vp], _i),
    "tvd_slab_create": ([_vp, ctypes.POINTER(TvdSystem), ctypes.POINTER(TvdPrecond), _i, _i,
                         ctypes.POINTER(_vp)], _i),
    "tvd_slab_destroy": ([_vp], _i),
    "tvd_slab_info": ([_vp, ctypes.POINTER(_i)], _i),
    "tvd_slab_buffer": ([_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_ll)], _i),
    "tvd_slab_start": ([_vp, _vp, _vp, _d, _i, _vp], _i),
    "tvd_slab_phase": ([_vp, _i], _i),
    "tvd_slab_status": ([_vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i),
                         ctypes.POINTER(_i), ctypes.POINTER(_d)], _i),
    "tvd_vec_dot": ([_vp, _ll, _vp, _vp, ctypes.POINTER(_d)], _i),
    "tvd_vec_axpby": ([_vp, _ll, _d, _vp, _d, _vp, _vp], _i),
    "tvd_vec_binary": ([_vp, _ll, _i, _vp, _vp, _vp], _i),
}

EXPORTED = tuple(_SIGNATURES)


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str) -> None:
        super().__init__(f"tvdeblur native error {code}: {message}")
        self.code = code
        self.message = message


def load(path: pathlib.Path | str | None = None):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path else _LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"native library {p} is missing; build it with "
                "`python -m paper_1011_5964_b200.build` (no CPU fallback exists)")
        lib = ctypes.CDLL(str(p))
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != TVD_OK:
        msg = load().tvd_last_error().decode(errors="replace")
        raise NativeError(rc, msg)


# ---------------------------------------------------------------- contexts
_tls = threading.local()


def _require_cuda(device: torch.device) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("tvdeblur B200 path needs a CUDA device (no CPU fallback)")


def context(device: torch.device | int | None = None) -> int:
    """Per-thread, per-device native context bound to torch's current stream."""
    lib = load()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       (device if isinstance(device, int) else (device.index or 0)))
    _require_cuda(dev)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    stream = torch.cuda.current_stream(dev).cuda_stream
    h = ctxs.get(dev.index)
    if h is None:
        out = _vp()
        check(lib.tvd_ctx_create(dev.index, _vp(stream), ctypes.byref(out)))
        h = ctxs[dev.index] = out.value
    else:
        check(lib.tvd_ctx_set_stream(h, _vp(stream)))
    return h


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("tvdeblur B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def to_device(x, device: torch.device | None = None) -> tuple[torch.Tensor, bool]:
    """``(float64 contiguous CUDA tensor, came_from_numpy)``."""
    if isinstance(x, torch.Tensor):
        dev = x.device if x.is_cuda else (device or default_device())
        t = x.to(device=dev, dtype=torch.float64)
        return t.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    dev = device or default_device()
    return torch.from_numpy(arr).to(dev), True


def to_host_like(t: torch.Tensor, was_numpy: bool):
    return t.cpu().numpy() if was_numpy else t


# ---------------------------------------------------------- instrumentation
def launch_count(device=None) -> int:
    out = _ll()
    check(load().tvd_ctx_counters(context(device), ctypes.byref(out)))
    return out.value


#: option ids of include/tvdeblur_b200.h (TVD_OPT_*)
OPTIONS = {"generic_fft": 1, "solver_graph": 2, "pdl": 3, "band_generic": 4, "band_slide": 5,
           "fin_fusion": 6, "p_fusion": 7, "pfa_stages": 8, "general_blur": 9,
           "band_prefetch": 10, "split_x": 11, "guard_slots": 12}


def set_option(name: str, value: int, device=None) -> None:
    """Set a library option (``generic_fft`` per context, the others process-wide)."""
    check(load().tvd_ctx_set_option(context(device), OPTIONS[name], int(value)))


def get_option(name: str, device=None) -> int:
    out = _i()
    check(load().tvd_ctx_get_option(context(device), OPTIONS[name], ctypes.byref(out)))
    return out.value


class option:
    """``with option("pdl", 1): ...`` -- set an option for a block, then restore it."""

    def __init__(self, name: str, value: int, device=None) -> None:
        self.name, self.value, self.device = name, int(value), device

    def __enter__(self):
        self.saved = get_option(self.name, self.device)
        set_option(self.name, self.value, self.device)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.saved, self.device)


def check_guards(device=None) -> tuple[int, int]:
    """``(corrupted guard bytes, guarded slots)`` of this thread's context (option
    ``guard_slots``)."""
    bad, slots = _ll(), _i()
    check(load().tvd_ctx_check_guards(context(device), ctypes.byref(bad), ctypes.byref(slots)))
    return bad.value, slots.value


def set_generic_fft(enable: bool, device=None) -> None:
    """Route DST passes through the generic mixed-radix FFT (parity tests of both engines)."""
    set_option("generic_fft", 1 if enable else 0, device)


def profile(enable: bool, device=None) -> None:
    check(load().tvd_ctx_profile(context(device), 1 if enable else 0))


def profile_read(device=None) -> dict[str, tuple[float, int]]:
    """``{category: (total_ms, launches)}`` recorded since ``profile(True)``."""
    lib = load()
    names = []
    while True:
        nm = lib.tvd_profile_category(len(names))
        if nm is None:
            break
        names.append(nm.decode())
    ms = (_d * len(names))()
    cnt = (_ll * len(names))()
    check(lib.tvd_ctx_profile_read(context(device), len(names), ms, cnt))
    return {nm: (ms[i], cnt[i]) for i, nm in enumerate(names) if cnt[i]}
