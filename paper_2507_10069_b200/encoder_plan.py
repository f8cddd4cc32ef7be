"""Qwen2.5-VL vision-tower token order (pure numpy, no native code: bench.py's
CPU legs use it without loading libemm.so)."""
from __future__ import annotations

import numpy as np


def window_plan(gh: int, gw: int, merge: int, window: int) -> dict:
    """Token order of the Qwen2.5-VL vision tower for one gh x gw patch grid.

    Patches are grouped into merge x merge units (the merger's 2x2 groups),
    units into windows of (window/merge)^2 units, windows row-major; inside
    a window units are row-major and inside a unit patches are row-major
    (the processor's patch order permuted by the model's window index, so
    every attention window is one contiguous varlen segment).  Returns
    int32 arrays: row_patch (raster patch index of each row), pos_h / pos_w
    (patch row / column = the 2-D rotary positions), window_lens (patches
    per window, in row order) and unit_rows (for merged token u in raster
    order, the 4 rows of its patches: the merger's gather)."""
    m = merge
    mh, mw = gh // m, gw // m
    ws = max(1, window // m)
    nww = (mw + ws - 1) // ws
    ur, uc = np.divmod(np.arange(mh * mw, dtype=np.int64), mw)
    wid = (ur // ws) * nww + (uc // ws)
    order = np.lexsort((uc, ur, wid))          # units in window order
    dy, dx = np.divmod(np.arange(m * m, dtype=np.int64), m)
    py = (ur[order][:, None] * m + dy[None, :]).reshape(-1)
    px = (uc[order][:, None] * m + dx[None, :]).reshape(-1)
    counts = np.bincount(wid, minlength=int(wid.max()) + 1)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    unit_rows = (inv[:, None] * (m * m) + np.arange(m * m)[None, :]).reshape(-1)
    return {"row_patch": (py * gw + px).astype(np.int32), "pos_h": py.astype(np.int32),
            "pos_w": px.astype(np.int32),
            "window_lens": (counts[counts > 0] * m * m).astype(np.int64),
            "unit_rows": unit_rows.astype(np.int32)}


def window_lens(gh: int, gw: int, merge: int, window: int) -> np.ndarray:
    """Patches per attention window of a gh x gw grid, in row order."""
    if window <= 0:
        return np.array([gh * gw], np.int64)
    return window_plan(gh, gw, merge, window)["window_lens"]
