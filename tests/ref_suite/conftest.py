"""Run the reference's own hot-path test suites against the B200 engine.

tests/ref_suite/test_amen.py, test_tt_core.py and test_cross.py are verbatim copies of the
reference's /root/reference/pkg/tests/ files of the same names (reference test vectors: test
infrastructure, not product code).  They import ``ttfem.tt``, ``ttfem.amen``, ``ttfem.cross``,
``ttfem.errors`` (and a few ``ttfem.grid`` index helpers); this conftest aliases those module
names to the engine's drop-in modules -- the INTEGRATION.md section 1 shim -- so every
``amen_solve``, ``tt_round``, ``tt_apply``, ``tt_norm``... call in the suites runs on the GPU
through libqtt.so.  All tests here are marked ``gpu``.

Deliberate deviations, marked xfail with the reason:
  * mode-size rejection: the engine's ``_ALLOWED_MODES`` also admits 3 (the 3D elasticity
    component core) and 9, so the reference's "mode 3 is rejected" checks cannot hold.
"""
import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2501_12151_b200 import amen as _amen  # noqa: E402
from paper_2501_12151_b200 import cross as _cross  # noqa: E402
from paper_2501_12151_b200 import errors as _errors  # noqa: E402
from paper_2501_12151_b200 import tt as _tt  # noqa: E402


def _fused_digit_matrix(m2, axis):
    """2x2 digit map lifted to the fused 2D digit 2*i + j (reference grid.py:120-126)."""
    return np.kron(m2, np.eye(2)) if axis == "i" else np.kron(np.eye(2), m2)


def build_shift_operator(axis, offset, d):
    """(S v)(n) = v(n - offset along axis), zero fill (reference grid.py:199-232), restated
    for the one reference test that needs a non-symmetric operator (2D grid assembly is out
    of this engine's scope)."""
    if axis not in ("i", "j"):
        raise ValueError(f"axis must be 'i' or 'j', got {axis!r}")
    if offset == 0:
        return _tt.TTLinearOperator([np.eye(4).reshape(1, 4, 4, 1)] * d)
    up = _fused_digit_matrix(np.array([[0.0, 0.0], [1.0, 0.0]]), axis)
    down = _fused_digit_matrix(np.array([[0.0, 1.0], [0.0, 0.0]]), axis)
    same = _fused_digit_matrix(np.eye(2), axis)
    if d == 1:
        return _tt.TTLinearOperator([up.reshape(1, 4, 4, 1)])
    first = np.zeros((1, 4, 4, 2))
    first[0, :, :, 0], first[0, :, :, 1] = same, up
    mids = []
    for _ in range(1, d - 1):
        mid = np.zeros((2, 4, 4, 2))
        mid[0, :, :, 0], mid[0, :, :, 1], mid[1, :, :, 1] = same, up, down
        mids.append(mid)
    last = np.zeros((2, 4, 4, 1))
    last[0, :, :, 0], last[1, :, :, 0] = up, down
    return _tt.TTLinearOperator([first] + mids + [last])


def interleave(i, j, d):
    """Fused digits 2*i_k + j_k, most significant first (reference grid.py:120-126)."""
    if not (0 <= i < 2 ** d and 0 <= j < 2 ** d):
        raise ValueError("axis index out of range")
    return tuple(2 * ((i >> (d - 1 - k)) & 1) + ((j >> (d - 1 - k)) & 1) for k in range(d))


def deinterleave(digits):
    """Inverse of interleave (reference grid.py:129-138)."""
    i = j = 0
    d = len(digits)
    for k, t in enumerate(digits):
        if t not in (0, 1, 2, 3):
            raise ValueError(f"fused digit {t} out of range")
        i += (t >> 1) << (d - 1 - k)
        j += (t & 1) << (d - 1 - k)
    return i, j


def morton_index(i, j, d):
    """Linear position of node (i, j) in the fused big-endian ordering (reference grid.py:141-146)."""
    out = 0
    for t in interleave(i, j, d):
        out = 4 * out + t
    return out


_grid = types.ModuleType("ttfem.grid")
_grid.build_shift_operator = build_shift_operator
_grid.interleave, _grid.deinterleave, _grid.morton_index = interleave, deinterleave, morton_index
_pkg = types.ModuleType("ttfem")
_pkg.__path__ = []
_pkg.tt, _pkg.amen, _pkg.errors, _pkg.grid, _pkg.cross = _tt, _amen, _errors, _grid, _cross
sys.modules.update({"ttfem": _pkg, "ttfem.tt": _tt, "ttfem.amen": _amen, "ttfem.errors": _errors,
                    "ttfem.grid": _grid, "ttfem.cross": _cross})

# (test-id substring -> reason): deliberate, documented deviations of the engine's API
XFAIL = {
    "test_rejects_bad_mode": "engine admits mode 3 (3D elasticity component core) and 9: _ALLOWED_MODES widened "
                             "on purpose (paper_2501_12151_b200/tt.py)",
}


def pytest_collection_modifyitems(config, items):
    here = os.path.dirname(os.path.abspath(__file__))
    for item in items:
        if str(item.fspath).startswith(here):
            item.add_marker(pytest.mark.gpu)
            for key, why in XFAIL.items():
                if key in item.nodeid:
                    item.add_marker(pytest.mark.xfail(reason=why, strict=True))
