"""Element-loop (scipy.sparse) assembly of the 3D Q1 cube problem -- TEST INFRASTRUCTURE.

Independent check of ``paper_2501_12151_b200.assembly3d`` (the builder's Kronecker/QTT
assembly of BASELINE's 3D configs; the reference itself only assembles 2D plane stress,
/root/reference/pkg/src/ttfem/elasticity.py:522-667, so SURVEY.md 8c asks for a
builder-written sparse oracle at L <= 3-4).  Nothing here shares code with the QTT
assembly: trilinear hexahedra on the 2^L-node grid (grid.py:63-77 node convention), element
stiffness B^T D B by 2x2x2 Gauss on each element -- split along z at a material interface so
a cut element is integrated exactly -- the consistent body load, an element-face quadrature
of the x = 1 patch traction (clipped to the patch), and the reference's symmetric clamp
P K P + (I - P), f <- P f, with the mean-diagonal scaling (elasticity.py:559-565, 612-667).

DOF order: (component, x, y, z) with index a*N^3 + i*N^2 + j*N + k, the dense layout of the
serial-binary QTT (component core first, big-endian digits per axis).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

_GP = (np.array([-1.0, 1.0]) / math.sqrt(3.0) + 1.0) / 2.0  # 2-pt Gauss on [0, 1]
_CORNERS = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]


def lame(E, nu):
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def element_stiffness(h, z0, z1, E, nu):
    """24 x 24 stiffness of the element [0,h]^3 restricted to local z in [z0, z1] (exact:
    the integrand is a polynomial of degree <= 2 per axis), dofs (corner, component)."""
    lam, mu = lame(E, nu)
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[3:, 3:] = mu * np.eye(3)
    ke = np.zeros((24, 24))
    for gx in _GP:
        for gy in _GP:
            for gz in _GP:
                x, y, z = gx * h, gy * h, z0 + gz * (z1 - z0)
                w = (h / 2.0) * (h / 2.0) * ((z1 - z0) / 2.0)
                B = np.zeros((6, 24))
                for c, (ix, iy, iz) in enumerate(_CORNERS):
                    fx, fy, fz = (x / h if ix else 1 - x / h), (y / h if iy else 1 - y / h), (z / h if iz else 1 - z / h)
                    dx = (1.0 if ix else -1.0) / h * fy * fz
                    dy = (1.0 if iy else -1.0) / h * fx * fz
                    dz = (1.0 if iz else -1.0) / h * fx * fy
                    B[0, 3 * c] = dx
                    B[1, 3 * c + 1] = dy
                    B[2, 3 * c + 2] = dz
                    B[3, 3 * c], B[3, 3 * c + 1] = dy, dx          # gamma_xy
                    B[4, 3 * c + 1], B[4, 3 * c + 2] = dz, dy      # gamma_yz
                    B[5, 3 * c], B[5, 3 * c + 2] = dz, dx          # gamma_xz
                ke += w * B.T @ D @ B
    return ke


def _dof(N, a, i, j, k):
    return a * N ** 3 + i * N * N + j * N + k


def stiffness(L, nu=0.3, E=1.0, layers=None):
    """Unclamped global stiffness (scipy.sparse CSR).  layers = (cut_z, E_lo, E_hi) with
    E = E_lo for z < cut_z, E_hi otherwise."""
    N = 2 ** L
    h = 1.0 / (N - 1)
    cache = {}

    def ke_for(ez):
        a, b = ez * h, (ez + 1) * h
        if layers is None:
            pieces = [(0.0, h, E)]
        else:
            cut, e_lo, e_hi = layers
            pts = [a] + ([cut] if a < cut < b else []) + [b]
            pieces = [(s0 - a, s1 - a, e_lo if (s0 + s1) / 2 < cut else e_hi) for s0, s1 in zip(pts[:-1], pts[1:])]
        key = tuple(pieces)
        if key not in cache:
            cache[key] = sum(element_stiffness(h, z0, z1, Ee, nu) for z0, z1, Ee in pieces)
        return cache[key]

    rows, cols, vals = [], [], []
    for ex in range(N - 1):
        for ey in range(N - 1):
            for ez in range(N - 1):
                ke = ke_for(ez)
                idx = np.array([_dof(N, comp, ex + a, ey + b, ez + c) for (a, b, c) in _CORNERS for comp in range(3)])
                rows.append(np.repeat(idx, 24))
                cols.append(np.tile(idx, 24))
                vals.append(ke.ravel())
    n = 3 * N ** 3
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()


def body_load(L, body=(0.0, 0.0, -1.0)):
    """f_i = int b . phi_i dV (consistent load): h^3/8 per element corner."""
    N = 2 ** L
    h = 1.0 / (N - 1)
    f = np.zeros(3 * N ** 3)
    for ex in range(N - 1):
        for ey in range(N - 1):
            for ez in range(N - 1):
                for (a, b, c) in _CORNERS:
                    for comp in range(3):
                        f[_dof(N, comp, ex + a, ey + b, ez + c)] += body[comp] * h ** 3 / 8.0
    return f


def patch_load(L, traction=(0.0, 0.0, -1.0), patch=(0.25, 0.75)):
    """Traction on the x = 1 face over y, z in patch: face elements clipped to the patch,
    2x2 Gauss on each clipped rectangle (exact for the bilinear face shape functions)."""
    N = 2 ** L
    h = 1.0 / (N - 1)
    lo, hi = patch
    f = np.zeros(3 * N ** 3)
    for ey in range(N - 1):
        for ez in range(N - 1):
            y0, y1 = max(ey * h, lo), min((ey + 1) * h, hi)
            z0, z1 = max(ez * h, lo), min((ez + 1) * h, hi)
            if y1 <= y0 or z1 <= z0:
                continue
            for gy in _GP:
                for gz in _GP:
                    y, z = y0 + gy * (y1 - y0), z0 + gz * (z1 - z0)
                    w = (y1 - y0) / 2.0 * (z1 - z0) / 2.0
                    ty, tz = (y - ey * h) / h, (z - ez * h) / h
                    for b in (0, 1):
                        for c in (0, 1):
                            phi = (ty if b else 1 - ty) * (tz if c else 1 - tz)
                            for comp in range(3):
                                f[_dof(N, comp, N - 1, ey + b, ez + c)] += w * phi * traction[comp]
    return f


def clamp_mask(L):
    """1 on free dofs, 0 on the clamped x = 0 face (all components)."""
    N = 2 ** L
    m = np.ones((3, N, N, N))
    m[:, 0, :, :] = 0.0
    return m.ravel()


def clamped_system(K, f, L):
    """The reference's symmetric clamp and mean-diagonal scaling (elasticity.py:559-565,
    612-620, 654-667): A = P K P / s + (I - P), rhs = P f / s, s = mean diag(P K P)."""
    p = clamp_mask(L)
    P = sp.diags(p)
    PKP = (P @ K @ P).tocsr()
    s = float(PKP.diagonal().mean())
    A = (PKP / s + sp.diags(1.0 - p)).tocsr()
    return A, p * f / s, s


def rigid_body_modes(L):
    """The six rigid motions of the cube (3 translations, 3 rotations) at the nodes."""
    N = 2 ** L
    t = np.linspace(0.0, 1.0, N)
    X, Y, Z = np.meshgrid(t, t, t, indexing="ij")
    zero, one = np.zeros_like(X), np.ones_like(X)
    modes = [(one, zero, zero), (zero, one, zero), (zero, zero, one),
             (-Y, X, zero), (zero, -Z, Y), (Z, zero, -X)]
    return np.array([np.stack(m).ravel() for m in modes])
