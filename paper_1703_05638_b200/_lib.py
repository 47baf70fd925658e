"""ctypes binding of the C ABI in include/lrk.h (liblrk.so, built for sm_100a).

This module is the only place Python touches native code.  It fails loudly:
a missing or stale shared library raises ImportError, and any device call on
a machine without CUDA raises RuntimeError — there is no CPU fallback.
Status codes map onto the reference's exceptions (errors.py:4-21).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, byref, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

from .errors import ConvergenceFailure, InvalidConfigError, NumericalError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblrk.so")

# status codes (include/lrk.h)
LRK_OK = 0
LRK_ERR_SHAPE = 1
LRK_ERR_CONFIG = 2
LRK_ERR_NUMERICAL = 3
LRK_ERR_CONVERGENCE = 4
LRK_ERR_CUDA = 5
LRK_ERR_UNSUPPORTED = 6

LRK_OP_HEAT = 0
LRK_OP_CONVDIFF = 1
LRK_OBS_FULL = 0
LRK_OBS_SUBGRID = 1
LRK_OBS_LIST = 2
LRK_MODE_IC = 0
LRK_MODE_SOURCE = 1
LRK_TRUNC_W1_ORTHO = 1
LRK_TRUNC_W2_ORTHOSCALED = 2
LRK_SOLVE_SWEEP = 0
LRK_SOLVE_GMRES = 1


class lrk_lr(Structure):
    _fields_ = [
        ("W1", c_void_p), ("W2", c_void_p), ("ld1", c_int64), ("ld2", c_int64),
        ("n_x", c_int), ("n_t", c_int), ("r", c_int), ("cap", c_int),
    ]


class lrk_operator_desc(Structure):
    _fields_ = [
        ("kind", c_int), ("dim", c_int), ("n_side", c_int), ("n_t", c_int),
        ("h", c_double), ("tau", c_double), ("m_scale", c_double), ("nu", c_double),
        ("wind", c_double * 3), ("stencil", c_int), ("wind_field", c_int),
    ]


class lrk_obs_desc(Structure):
    _fields_ = [
        ("kind", c_int), ("n1", c_int), ("n2", c_int),
        ("idx1", POINTER(c_int32)), ("idx2", POINTER(c_int32)),
        ("n_list", c_int), ("list", POINTER(c_int32)),
    ]


class lrk_solve_desc(Structure):
    _fields_ = [
        ("backend", c_int), ("eps0", c_double), ("r_max", c_int), ("compress_every", c_int),
        ("tol", c_double), ("max_iter", c_int),
    ]


class lrk_solve_info(Structure):
    _fields_ = [("achieved_residual", c_double), ("iterations", c_int), ("rank", c_int)]


class lrk_hessian_desc(Structure):
    _fields_ = [
        ("mode", c_int), ("gamma_prior", c_double), ("obs_weight", c_double),
        ("eps0", c_double), ("r_max", c_int), ("compress_every", c_int),
        ("prior_delta", c_double), ("prior_gamma", c_double), ("obs_every", c_int),
    ]


# exported symbols and their signatures (every entry point of include/lrk.h)
_SIGNATURES = {
    "lrk_version": (c_char_p, []),
    "lrk_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
    "lrk_ctx_destroy": (None, [c_void_p]),
    "lrk_last_error": (c_char_p, [c_void_p]),
    "lrk_launch_count": (c_int64, [c_void_p]),
    "lrk_profile_enable": (c_int, [c_void_p, c_int]),
    "lrk_set_emulated_shards": (c_int, [c_void_p, c_int]),
    "lrk_shard_setup": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "lrk_shard_connect": (c_int, [c_void_p, c_void_p]),
    "lrk_prior_apply": (c_int, [c_void_p, c_double, c_double, c_int, c_void_p, c_int64, c_int,
                                c_void_p, c_int64, c_void_p]),
    "lrk_prior_diag": (c_int, [c_void_p, c_double, c_double, c_int, c_void_p, c_void_p]),
    "lrk_profile_read": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int64), POINTER(c_double),
                                 c_int]),
    "lrk_last_traces": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int), c_int, POINTER(c_int),
                                POINTER(c_int), POINTER(c_int)]),
    "lrk_set_operator": (c_int, [c_void_p, POINTER(lrk_operator_desc)]),
    "lrk_set_observation": (c_int, [c_void_p, POINTER(lrk_obs_desc)]),
    "lrk_truncate": (c_int, [c_void_p, POINTER(lrk_lr), POINTER(lrk_lr), c_double, c_int, c_int,
                             POINTER(c_int), c_void_p]),
    "lrk_dot": (c_int, [c_void_p, POINTER(lrk_lr), POINTER(lrk_lr), POINTER(c_double), c_void_p]),
    "lrk_singular_values": (c_int, [c_void_p, POINTER(lrk_lr), POINTER(c_double), c_int,
                                    POINTER(c_int), c_void_p]),
    "lrk_step_solve": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_int64,
                               c_void_p]),
    "lrk_poisson_solve": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int64,
                                  c_void_p]),
    "lrk_operator_apply": (c_int, [c_void_p, POINTER(lrk_lr), c_int, POINTER(lrk_lr), c_void_p]),
    "lrk_st_solve_sweep": (c_int, [c_void_p, POINTER(lrk_lr), c_int, c_int, c_double, c_int,
                                   POINTER(lrk_lr), POINTER(c_int), c_int, POINTER(c_int),
                                   c_void_p]),
    "lrk_hessian_apply_ic": (c_int, [c_void_p, POINTER(lrk_hessian_desc), c_int, c_void_p,
                                     c_int64, c_void_p, c_int64, POINTER(c_int), c_void_p]),
    "lrk_hessian_apply_st": (c_int, [c_void_p, POINTER(lrk_hessian_desc), POINTER(lrk_lr),
                                     POINTER(lrk_lr), POINTER(c_int), c_void_p]),
    "lrk_add_truncate": (c_int, [c_void_p, c_int, POINTER(lrk_lr), POINTER(c_double), c_double,
                                 c_int, POINTER(lrk_lr), POINTER(c_int), c_void_p]),
    "lrk_lr_dots": (c_int, [c_void_p, POINTER(lrk_lr), POINTER(lrk_lr), c_int, POINTER(c_int),
                            POINTER(c_double), c_void_p]),
    "lrk_st_solve": (c_int, [c_void_p, POINTER(lrk_lr), c_int, POINTER(lrk_solve_desc),
                             POINTER(lrk_lr), POINTER(lrk_solve_info), POINTER(c_int), c_int,
                             POINTER(c_int), c_void_p]),
    "lrk_cgs2": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int, POINTER(c_double),
                         POINTER(c_double), c_void_p]),
    "lrk_combine": (c_int, [c_void_p, c_void_p, c_int64, c_int, POINTER(c_double), c_int,
                            c_void_p, c_void_p]),
}

_lib = None


def get_lib():
    """Load liblrk.so (no CUDA calls).  Raises ImportError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a).  There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGNATURES)


_cuda_seen = False


def require_cuda():
    """Fail loudly without a GPU.  torch.cuda.is_available() costs milliseconds
    (an NVML query) and sits on the per-apply path, so a positive answer is
    remembered; a negative one is re-checked every time."""
    global _cuda_seen
    if _cuda_seen:
        return
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1703_05638_b200 runs its hot path on a CUDA device (B200, sm_100a); "
            "no GPU is visible and there is no CPU fallback"
        )
    _cuda_seen = True


def stream_handle():
    import torch

    return c_void_p(torch.cuda.current_stream().cuda_stream)


def check(status, ctx=None, what="", info=None):
    """Map an lrk_status onto the reference's exceptions (errors.py:4-21);
    ``info`` (an lrk_solve_info) carries ConvergenceFailure's payload."""
    if status == LRK_OK:
        return
    msg = ""
    if ctx is not None:
        raw = get_lib().lrk_last_error(ctx)
        msg = raw.decode() if raw else ""
    msg = f"{what}: {msg}" if what else msg
    if status == LRK_ERR_SHAPE:
        raise ValueError(msg)
    if status == LRK_ERR_CONFIG:
        raise InvalidConfigError(msg)
    if status == LRK_ERR_CONVERGENCE:
        if info is not None:
            raise ConvergenceFailure(msg, achieved_residual=float(info.achieved_residual),
                                     iterations=int(info.iterations))
        raise ConvergenceFailure(msg)
    if status == LRK_ERR_NUMERICAL:
        raise NumericalError(msg)
    if status == LRK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA failure in liblrk: {msg}")


class Context:
    """Owns one lrk_ctx (workspace + optional operator/observation state)."""

    def __init__(self, device: int | None = None):
        import torch

        require_cuda()
        lib = get_lib()
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = c_void_p()
        check(lib.lrk_ctx_create(self.device, byref(h)), None, "lrk_ctx_create")
        self.handle = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.lrk_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None

    def launches(self) -> int:
        return int(self._lib.lrk_launch_count(self.handle))


_algebra_ctx: dict[int, Context] = {}


def algebra_context() -> Context:
    """Per-device context used by the free lr_* functions."""
    import torch

    require_cuda()
    dev = torch.cuda.current_device()
    ctx = _algebra_ctx.get(dev)
    if ctx is None:
        ctx = Context(dev)
        _algebra_ctx[dev] = ctx
    return ctx


def total_launches() -> int:
    return sum(c.launches() for c in _algebra_ctx.values())
