"""The C-ABI library loads on CPU and exports every symbol include/lrk.h declares
(no compute calls: this container has no GPU)."""

import os
import re

import numpy as np
import pytest

from paper_1703_05638_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lrk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lrk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("lrk_hessian_apply_ic", "lrk_hessian_apply_st", "lrk_st_solve_sweep",
                 "lrk_truncate", "lrk_dot", "lrk_operator_apply", "lrk_step_solve"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.get_lib()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib._SIGNATURES, f"{name} has no ctypes signature"


def test_version_string_without_gpu():
    assert b"sm_100a" in _lib.get_lib().lrk_version()


def test_compute_calls_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1703_05638_b200 as lp

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        lp.LowRankMat([[1.0]], [[1.0]])


def test_error_mapping():
    from paper_1703_05638_b200.errors import ConvergenceFailure, InvalidConfigError, NumericalError

    with pytest.raises(ValueError):
        _lib.check(_lib.LRK_ERR_SHAPE)
    with pytest.raises(InvalidConfigError):
        _lib.check(_lib.LRK_ERR_CONFIG)
    with pytest.raises(NumericalError):
        _lib.check(_lib.LRK_ERR_NUMERICAL)
    with pytest.raises(ConvergenceFailure):
        _lib.check(_lib.LRK_ERR_CONVERGENCE)
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.LRK_ERR_UNSUPPORTED)


def test_start_vector_matches_the_reference_rule():
    """cli.py:247-266: all-ones default, otherwise PCG64 standard_normal(seed), normalised."""
    import paper_1703_05638_b200 as lp

    v = lp.start_vector(50)
    np.testing.assert_array_equal(v, np.ones(50) / np.sqrt(50.0))
    w = lp.start_vector(50, start="random", seed=7)
    ref = np.random.default_rng(7).standard_normal(50)
    np.testing.assert_array_equal(w, ref / np.linalg.norm(ref))
    with pytest.raises(ValueError):
        lp.start_vector(5, start="zeros")
    with pytest.raises(ValueError):
        lp.start_vector(5, mode="source")
