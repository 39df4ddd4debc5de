"""Cone projections (mirrors conic_pdhg.cones, /root/reference/pkg/src/conic_pdhg/
cones.py).  Every projection runs in libpdcs's segmented projection kernels
(warp/CTA per block, thread per exponential-cone block); these wrappers only
move host vectors to and from the GPU for the step-level API.  Inside the
solver the same device functions are fused into the PDHG half-steps.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .linalg import NumericalError
from .model import KIND_CODE, Cone

# PDCS_ERR_* codes of the projection kernels (include/pdcs.h)
_ERR_TEXT = {
    3: "exponential-cone projection of a non-finite point",
    4: "rescaled-soc projection failed to bracket the multiplier",
    6: "rescaled-soc root finding failed to converge within max_root_iters",
}


@dataclass(frozen=True)
class ProjectionSettings:
    """Root-finding controls (cones.py:24-32), honoured by the device kernels:
    root_tol is the exp-cone bisection width (cones.py:263), max_root_iters
    bounds the exp-cone Newton + bisection evaluations (cones.py:227, 256)
    and the rescaled-SOC brentq iterations (cones.py:421)."""

    root_tol: float = 1e-12
    max_root_iters: int = 100


DEFAULT_SETTINGS = ProjectionSettings()


def _seg(v, kind_code, smode=N.SCALE_NONE, scale=None, settings: ProjectionSettings = DEFAULT_SETTINGS):
    from .device import project_segments

    v = np.asarray(v, dtype=np.float64)
    out, err = project_segments(v, [(kind_code, 0, v.size, smode)], scale,
                                settings.root_tol, settings.max_root_iters)
    if err:
        raise NumericalError(_ERR_TEXT.get(err, f"projection failure {err}"))
    return out


def project_box(v: np.ndarray, l: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Componentwise clamp onto [l, u] (cones.py:46-51)."""
    from .device import project_box_dev

    both = np.isfinite(l) & np.isfinite(u)
    if np.any(l[both] > u[both]):
        raise ValueError("box projection requires l <= u componentwise")
    return project_box_dev(v, l, u)


def project_soc(v: np.ndarray) -> np.ndarray:
    """Projection onto {t >= ||xbar||} (cones.py:54-67)."""
    return _seg(v, N.SOC)


def in_exp(v, atol: float = 0.0) -> bool:
    """Membership in K_exp (cones.py:80-88)."""
    a, b, c = float(v[0]), float(v[1]), float(v[2])
    if b > 0.0:
        ratio = a / b
        if ratio < 709.0 and c >= -atol and c + atol >= b * math.exp(ratio):
            return True
    return -atol <= b <= atol and a <= atol and c >= -atol


def in_dual_exp(v, atol: float = 0.0) -> bool:
    """Membership in K_exp* (cones.py:91-99)."""
    u, vv, w = float(v[0]), float(v[1]), float(v[2])
    if u > atol:
        return False
    if u >= -atol:
        return vv >= -atol and w >= -atol
    if w <= 0.0:
        return False
    return u * math.log(-u / w) - u + vv >= -atol


def project_exp(v: np.ndarray, settings: ProjectionSettings = DEFAULT_SETTINGS) -> np.ndarray:
    """Exact Euclidean projection onto the exponential cone (cones.py:298-326)."""
    return _seg(v, N.EXP, settings=settings)


def project_dual_exp(v: np.ndarray, settings: ProjectionSettings = DEFAULT_SETTINGS) -> np.ndarray:
    """Moreau: P_{K*}(v) = v + P_K(-v) (cones.py:329-331)."""
    return _seg(v, N.DUAL_EXP, settings=settings)


def project_rescaled_soc(v: np.ndarray, d: np.ndarray,
                         settings: ProjectionSettings = DEFAULT_SETTINGS) -> np.ndarray:
    """Projection onto {z : diag(d) z in SOC} (cones.py:353-429)."""
    d = np.asarray(d, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if d.shape != v.shape:
        raise ValueError("scale vector must match the block dimension")
    if np.any(d <= 0) or not np.all(np.isfinite(d)):
        raise ValueError("scale entries must be strictly positive and finite")
    if np.all(d == d[0]):
        return project_soc(v)
    return _seg(v, N.SOC, N.SCALE_DIRECT, d, settings)


_DUAL_KIND = {
    Cone.ZERO: Cone.FREE,
    Cone.FREE: Cone.ZERO,
    Cone.NONNEG: Cone.NONNEG,
    Cone.SOC: Cone.SOC,
    Cone.EXP: Cone.DUAL_EXP,
    Cone.DUAL_EXP: Cone.EXP,
}


def dual_cone_kind(kind: Cone) -> Cone:
    if kind not in _DUAL_KIND:
        raise ValueError(f"no dual-cone mapping for {kind}")
    return _DUAL_KIND[kind]


def project_cone(v: np.ndarray, kind: Cone, scale: np.ndarray | None = None,
                 settings: ProjectionSettings = DEFAULT_SETTINGS) -> np.ndarray:
    """Project onto {z : diag(scale) z in K(kind)} (cones.py:452-478)."""
    uniform = scale is None or np.all(scale == scale[0])
    if kind is Cone.RSOC:
        raise ValueError("rotated blocks must be reformulated (rsoc_to_soc) before projection")
    if kind not in KIND_CODE:
        raise ValueError(f"unknown cone kind {kind}")
    if kind in (Cone.EXP, Cone.DUAL_EXP) and not uniform:
        raise ValueError(f"{kind.value} blocks support only block-uniform scaling; rebuild the scaling")
    if kind is Cone.SOC and not uniform:
        return _seg(v, N.SOC, N.SCALE_DIRECT, np.asarray(scale, dtype=np.float64), settings)
    return _seg(v, KIND_CODE[kind], settings=settings)


def project_cone_dual(v: np.ndarray, kind: Cone, scale: np.ndarray | None = None,
                      settings: ProjectionSettings = DEFAULT_SETTINGS) -> np.ndarray:
    """Projection onto the dual of {z : diag(scale) z in K} (cones.py:481-490)."""
    inv = None if scale is None else 1.0 / scale
    return project_cone(v, dual_cone_kind(kind), inv, settings)


def _set(problem, which, v, space_len, offset=0, settings: ProjectionSettings = DEFAULT_SETTINGS):
    from .device import engine_for

    e = engine_for(problem)
    v = np.asarray(v, dtype=np.float64)
    buf_in = e.px0 if which in (0, 3, 4) else e.py0
    buf_out = e.px1 if which in (0, 3, 4) else e.py1
    full = np.zeros(space_len)
    full[offset:offset + v.size] = v
    e.upload(buf_in, full)
    e.project_set(which, buf_in, buf_out, settings.root_tol, settings.max_root_iters)
    return e.host(buf_out, space_len)[offset:offset + v.size]


def project_primal_set(x: np.ndarray, problem, settings: ProjectionSettings = DEFAULT_SETTINGS):
    """Projection onto [l, u] x K_p (cones.py:498-506)."""
    return _set(problem, 0, x, problem.n, settings=settings)


def project_dual_set(y: np.ndarray, problem, settings: ProjectionSettings = DEFAULT_SETTINGS):
    """Projection of y onto K_d, the blockwise dual of the stored kinds (cones.py:509-520)."""
    return _set(problem, 1, y, problem.m, settings=settings)


def project_dual_residual_set(r: np.ndarray, problem, settings: ProjectionSettings = DEFAULT_SETTINGS):
    """Projection of Gx - h onto K_d* (cones.py:523-530)."""
    return _set(problem, 2, r, problem.m, settings=settings)


def project_primal_cone_part(v: np.ndarray, problem, settings: ProjectionSettings = DEFAULT_SETTINGS):
    """Projection of a length n - num_box vector onto K_p (cones.py:533-539)."""
    return _set(problem, 4, v, problem.n, problem.num_box, settings=settings)


def project_primal_cone_dual(lam: np.ndarray, problem, settings: ProjectionSettings = DEFAULT_SETTINGS):
    """Projection of lambda_2 onto K_p* (cones.py:542-549)."""
    return _set(problem, 3, lam, problem.n, problem.num_box, settings=settings)
