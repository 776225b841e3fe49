"""Shared test helpers: tolerance checks and device operators from the seeded inputs."""
from __future__ import annotations

import numpy as np

# North star: GPU vs oracle relative l2 error <= 1e-12 per right-hand side in
# fp64.  Elementwise: |dy_i| <= 1e-12 * max_i |y_ref_i|.
TOL = 1e-12


def assert_parity(y, ref, tol=TOL):
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.ndim == 1:
        y, ref = y[:, None], ref[:, None]
    assert y.shape == ref.shape, (y.shape, ref.shape)
    assert np.all(np.isfinite(y))
    for k in range(ref.shape[1]):
        d = y[:, k] - ref[:, k]
        nr = np.linalg.norm(ref[:, k])
        scale = np.abs(ref[:, k]).max() if ref.shape[0] else 0.0
        if nr == 0:
            assert np.all(d == 0)
            continue
        rel = np.linalg.norm(d) / nr
        assert rel <= tol, f"column {k}: rel l2 {rel:.3e} > {tol}"
        assert np.abs(d).max() <= tol * scale, f"column {k}: max abs {np.abs(d).max():.3e} > {tol} * {scale:.3e}"


def rel_err(y, ref):
    return float(np.linalg.norm(np.asarray(y) - np.asarray(ref)) / max(np.linalg.norm(ref), 1e-300))


def device_operator(cfg, hm, dist=None, stream=0):
    """hmat_create_uninit + in-place device generation of the seeded panels."""
    from gen import hgen
    create = hm.hmat_create_standard_uninit if cfg.adm else hm.hmat_create_uninit
    h = create(cfg.L, cfg.d, cfg.b, cfg.r, dist)
    r0, r1 = hm.hmat_local_rows(h)
    hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, stream)
    return h
