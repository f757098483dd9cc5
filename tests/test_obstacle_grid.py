"""The host-built nearest-cylinder candidate grid (mppi_obstacle_grid, HOST only,
no GPU): for points anywhere in the grid and its border band — including exactly on cell
boundaries — the minimum of |p - c|^2 over the cell's candidate list equals the minimum over all
cylinders, evaluated with the kernel's fp32 expression (dx = p + (-c), fma(dy, dy, dx * dx))."""
import ctypes as C

import numpy as np
import pytest

from mppi_inputs.forest import forest_4m, generate_forest


def _lib():
    from paper_1509_01149_b200 import _capi as A
    return A.lib(), A


def _grid(xy):
    L, A = _lib()
    xy = np.ascontiguousarray(xy, np.float32)
    geom = (C.c_float * 6)()
    st = L.mppi_obstacle_grid(xy.ctypes.data_as(C.POINTER(C.c_float)), len(xy), None, 0, geom)
    assert st == 0, A.status_string(st) if hasattr(A, "status_string") else st
    nx, ny = int(geom[0]), int(geom[1])
    words = (C.c_uint32 * (nx * ny))()
    st = L.mppi_obstacle_grid(xy.ctypes.data_as(C.POINTER(C.c_float)), len(xy), words, nx * ny, geom)
    assert st == 0
    return np.frombuffer(words, np.uint32).reshape(ny, nx), [float(g) for g in geom]


def _d2(px, py, cx, cy):
    """the kernel's fp32 squared distance (negated centres, fma), emulated in float64 then
    rounded; both sides of the comparison use the same emulation"""
    dx = (px + (-cx)).astype(np.float32)
    dy = (py + (-cy)).astype(np.float32)
    dxdx = (dx.astype(np.float64) * dx).astype(np.float32)
    return (dy.astype(np.float64) * dy + dxdx).astype(np.float32)


def _check(xy, pts, words, geom):
    nx, ny, ox, oy, inv_h, band = geom
    px, py = pts[:, 0].astype(np.float32), pts[:, 1].astype(np.float32)
    gx = (px.astype(np.float64) * np.float32(inv_h) + np.float32(ox)).astype(np.float32)
    gy = (py.astype(np.float64) * np.float32(inv_h) + np.float32(oy)).astype(np.float32)
    inband = (gx >= -band) & (gx < nx + band) & (gy >= -band) & (gy < ny + band)
    ix = np.clip(np.floor(gx).astype(np.int64), 0, int(nx) - 1)
    iy = np.clip(np.floor(gy).astype(np.int64), 0, int(ny) - 1)
    w = words[iy, ix]
    cnt = w >> 28
    ok = inband & (cnt > 0)
    cx, cy = xy[:, 0].astype(np.float32), xy[:, 1].astype(np.float32)
    full = np.min(_d2(px[:, None], py[:, None], cx[None, :], cy[None, :]), axis=1)
    cand = np.full(len(pts), np.inf, np.float32)
    for s in range(4):
        idx = ((w >> (7 * s)) & 127).astype(np.int64)
        cand = np.minimum(cand, _d2(px, py, cx[idx], cy[idx]))
    assert ok.mean() > 0.9, ok.mean()             # border (band) cells with > 4 candidates fall back
    bad = ok & (cand != full)
    assert not bad.any(), (np.nonzero(bad)[0][:10], pts[bad][:5])


def test_forest_4m_grid_random_and_boundary_points():
    xy = np.array(forest_4m()["centers"], np.float32)
    words, geom = _grid(xy)
    nx, ny, ox, oy, inv_h, band = geom
    rng = np.random.default_rng(0)
    h = 1.0 / inv_h
    x0, y0 = -ox * h, -oy * h                     # grid origin
    # uniform over the grid plus a 20-cell margin of the band
    pts = np.stack([rng.uniform(x0 - 20 * h, x0 + (nx + 20) * h, 200000),
                    rng.uniform(y0 - 20 * h, y0 + (ny + 20) * h, 200000)], axis=1)
    # exactly on (and 1 ulp around) cell boundaries and near the cylinders
    bx = x0 + h * rng.integers(0, int(nx), 20000)
    by = y0 + h * rng.integers(0, int(ny), 20000)
    edge = np.stack([np.nextafter(bx.astype(np.float32), np.float32(rng.choice([-1e9, 1e9]))),
                     by.astype(np.float32)], axis=1)
    near = xy[rng.integers(0, len(xy), 20000)] + rng.normal(scale=0.6, size=(20000, 2))
    _check(xy, np.concatenate([pts, edge, near]).astype(np.float32), words, geom)


@pytest.mark.parametrize("spacing,seed", [(3.0, 1), (5.0, 2), (4.0, 7)])
def test_other_forests(spacing, seed):
    xy = np.array(generate_forest(spacing=spacing, seed=seed)["centers"], np.float32)
    if len(xy) > 127:
        xy = xy[:127]
    words, geom = _grid(xy)
    nx, ny, ox, oy, inv_h, band = geom
    h = 1.0 / inv_h
    rng = np.random.default_rng(seed)
    pts = np.stack([rng.uniform(-ox * h, (nx - ox) * h, 100000),
                    rng.uniform(-oy * h, (ny - oy) * h, 100000)], axis=1).astype(np.float32)
    _check(xy, pts, words, geom)


def test_degenerate_inputs_refused():
    L, A = _lib()
    one = np.zeros((1, 2), np.float32)
    geom = (C.c_float * 6)()
    assert L.mppi_obstacle_grid(one.ctypes.data_as(C.POINTER(C.c_float)), 1, None, 0, geom) == A.MPPI_ERR_UNSUPPORTED
    same = np.ones((5, 2), np.float32)
    assert L.mppi_obstacle_grid(same.ctypes.data_as(C.POINTER(C.c_float)), 5, None, 0, geom) == A.MPPI_ERR_UNSUPPORTED
