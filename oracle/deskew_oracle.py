"""CPU ORACLE (test infrastructure only) for the deskew + projection hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module.  It is the checker, never the product: the package
``paper_2211_00645_b200`` does not import it and has no CPU fallback.

It restates, in numpy, the reference ``skewstream`` algorithm for this path:

* canvas placement spans      ss/geometry.py:124-147, 236-255; ss/pipeline.py:274-281
* streaming linear rows       ss/pipeline.py:229-236  (fp64 (1-f)*a + f*b, rint half-even)
* streaming nearest rows      ss/pipeline.py:283-287  (a view of the frame)
* streaming max canvas        ss/pipeline.py:316-341  (np.maximum into the canvas)
* batch reference rows        ss/phantom.py:389-402   (np.interp per column; pile max; rint; clip)
* display warp                ss/pipeline.py:434-457
* rolling band recompute      ss/pipeline.py:345-398  (strict '>' first-max-wins contributor map)

and the north_star extensions that have no reference symbol: the full deskewed
volume V[i,u,x] (the reference's ``pile`` layout (N,U,W), ss/phantom.py:390,
rounded per voxel) and its projections along axis 0 (XY, = the reference's
canvas), axis 1 (XZ) and axis 2 (YZ), as max (uint16) or sum (uint32 of the
rounded voxels).

Pinning: ``tests/golden/make_golden.py`` generates fixtures by running the
reference itself (``ProjectionCanvas._slice_rows``, ``reference_deskew`` on
one-hot stacks, ``warp_projection``, rolling mode); ``tests/test_oracle.py``
checks this module against them bit for bit.

``np.interp`` is restated (numpy 2.3 ``arr_interp``: binary search for
xp[j] <= x < xp[j+1]; slope = (fp[j+1]-fp[j]) / (xp[j+1]-xp[j]);
value = slope*(x-xp[j]) + fp[j]; x < xp[0] -> fp[0]; x > xp[-1] or x == xp[-1]
-> fp[-1]; x == xp[j] -> fp[j]) in vectorised form, because the reference calls
it once per column (ss/phantom.py:399-400), which is too slow for the oracle.
"""

from __future__ import annotations

import math

import numpy as np

EPS = 1e-9  # ss/geometry.py:39
MAX_INTENSITY = 65535  # ss/phantom.py:34


# ---------------------------------------------------------------------------
# geometry restatement (ss/geometry.py)

def ceil_snapped(x: float) -> int:
    return math.ceil(x - EPS)  # ss/geometry.py:124-126


def canvas_height(n: int, h: int, shear: float) -> int:
    return h + ceil_snapped((n - 1) * shear)  # ss/geometry.py:141


def nearest_offset(i: int, shear: float) -> int:
    return math.floor(i * shear + 0.5)  # ss/geometry.py:243


def linear_span(i: int, shear: float, h: int) -> tuple[int, int]:
    off = i * shear  # ss/geometry.py:252-255
    return ceil_snapped(off), math.floor(off + h - 1 + EPS)


def span(i: int, shear: float, h: int, interp: str) -> tuple[int, int]:
    if interp == "nearest":  # ss/pipeline.py:274-281
        lo = nearest_offset(i, shear)
        return lo, lo + h - 1
    return linear_span(i, shear, h)


# ---------------------------------------------------------------------------
# per-slice row values

def canvas_rows(pixels: np.ndarray, lo: int, hi: int, off: float) -> np.ndarray:
    """ss/pipeline.py:229-236: fp64 lerp of two rows of the same frame, rint, uint16."""
    h = pixels.shape[0]
    j = np.arange(lo, hi + 1, dtype=np.float64) - off
    j0 = np.clip(np.floor(j).astype(np.int64), 0, h - 1)
    j1 = np.minimum(j0 + 1, h - 1)
    f = (j - j0)[:, None]
    a = pixels[j0].astype(np.float64)
    b = pixels[j1].astype(np.float64)
    return np.rint((1.0 - f) * a + f * b).astype(np.uint16)


def interp_rows_f64(pixels: np.ndarray, lo: int, hi: int, i: int, shear: float) -> np.ndarray:
    """Unrounded fp64 rows of ss/phantom.py:396-400 (np.interp per column), vectorised."""
    h, w = pixels.shape
    x = np.arange(lo, hi + 1, dtype=np.float64)
    xp = i * shear + np.arange(h)  # ss/phantom.py:398 (float + int64 array -> float64)
    fp = pixels.astype(np.float64)
    if h == 1:  # arr_interp's single-point branch: everything maps to fp[0]
        return np.repeat(fp[:1], x.size, axis=0)
    # j = largest k with xp[k] <= x  (searchsorted 'right' minus one)
    j = np.searchsorted(xp, x, side="right") - 1
    out = np.empty((x.size, w), dtype=np.float64)
    below = j < 0
    above = x > xp[-1]
    at_end = (j == h - 1) & ~above
    jj = np.clip(j, 0, h - 2)
    at_node = (~below) & (~above) & (~at_end) & (xp[jj] == x)
    mid = ~(below | above | at_end | at_node)
    out[below] = fp[0]
    out[above | at_end] = fp[h - 1]
    out[at_node] = fp[jj[at_node]]
    if mid.any():
        jm = jj[mid]
        dxp = (xp[jm + 1] - xp[jm])[:, None]
        slope = (fp[jm + 1] - fp[jm]) / dxp
        out[mid] = slope * (x[mid] - xp[jm])[:, None] + fp[jm]
    return out


def interp_rows(pixels: np.ndarray, lo: int, hi: int, i: int, shear: float) -> np.ndarray:
    """Rounded (rint, clip) per-voxel values of the batch reference."""
    v = interp_rows_f64(pixels, lo, hi, i, shear)
    return np.clip(np.rint(v), 0, MAX_INTENSITY).astype(np.uint16)


def slice_rows(pixels: np.ndarray, i: int, shear: float, interp: str,
               formula: str = "canvas") -> tuple[int, int, np.ndarray]:
    """(lo, hi, rows) that global slice ``i`` contributes to the canvas."""
    h = pixels.shape[0]
    lo, hi = span(i, shear, h, interp)
    if interp == "nearest":  # ss/pipeline.py:286-287 (a view), ss/phantom.py:393-394
        return lo, hi, pixels
    if formula == "canvas":
        return lo, hi, canvas_rows(pixels, lo, hi, i * shear)
    return lo, hi, interp_rows(pixels, lo, hi, i, shear)


# ---------------------------------------------------------------------------
# volume and projections

def deskew_volume(stack: np.ndarray, shear: float, interp: str = "linear",
                  formula: str = "canvas", first_slice: int = 0,
                  canvas_rows_total: int | None = None,
                  u_begin: int = 0, u_count: int | None = None) -> np.ndarray:
    """Deskewed volume V (n, u_count, W) uint16; zero outside each slice's span.

    Slice k of ``stack`` is global slice ``first_slice + k`` (scan-axis slabs use
    global indices). Rows are canvas rows ``u_begin .. u_begin+u_count-1``.
    """
    stack = np.asarray(stack)
    n, h, w = stack.shape
    if canvas_rows_total is None:
        canvas_rows_total = canvas_height(first_slice + n, h, shear)
    if u_count is None:
        u_count = canvas_rows_total - u_begin
    vol = np.zeros((n, u_count, w), dtype=np.uint16)
    for k in range(n):
        lo, hi, rows = slice_rows(stack[k], first_slice + k, shear, interp, formula)
        a, b = max(lo, u_begin), min(hi, u_begin + u_count - 1)
        if a > b:
            continue
        vol[k, a - u_begin:b - u_begin + 1] = rows[a - lo:b - lo + 1]
    return vol


def project(vol: np.ndarray, axis: int, reduce: str = "max") -> np.ndarray:
    """Projection of the (N,U,W) volume: max -> uint16, sum -> uint32 (exact)."""
    if reduce == "max":
        return vol.max(axis=axis)
    return vol.sum(axis=axis, dtype=np.uint64).astype(np.uint32)


def projections(vol: np.ndarray, axes=(0, 1, 2), reduce: str = "max") -> dict:
    return {ax: project(vol, ax, reduce) for ax in axes}


# ---------------------------------------------------------------------------
# streaming canvas (XY max) without materialising the volume

def canvas_max(stack: np.ndarray, shear: float, interp: str = "linear",
               first_slice: int = 0, canvas_rows_total: int | None = None) -> np.ndarray:
    """ss/pipeline.py:316-336: place() every slice then finalize_global()."""
    stack = np.asarray(stack)
    n, h, w = stack.shape
    if canvas_rows_total is None:
        canvas_rows_total = canvas_height(first_slice + n, h, shear)
    canvas = np.zeros((canvas_rows_total, w), dtype=np.uint16)
    for k in range(n):
        lo, hi, rows = slice_rows(stack[k], first_slice + k, shear, interp, "canvas")
        np.maximum(canvas[lo:hi + 1], rows, out=canvas[lo:hi + 1])
    return canvas


def reference_deskew(stack, shear: float, interp: str = "nearest") -> np.ndarray:
    """ss/phantom.py:359-402 restated (local slice indices, np.interp rows, pile max)."""
    stack = np.asarray(stack)
    n, h, w = stack.shape
    out = np.zeros((canvas_height(n, h, shear), w), dtype=np.float64)
    for i in range(n):
        lo, hi = span(i, shear, h, interp)
        if interp == "nearest":
            vals = stack[i].astype(np.float64)
        else:
            vals = interp_rows_f64(stack[i], lo, hi, i, shear)
        np.maximum(out[lo:hi + 1], vals, out=out[lo:hi + 1])
    return np.clip(np.rint(out), 0, MAX_INTENSITY).astype(np.uint16)


def reference_deskew_as_is(stack, shear: float, interp: str = "linear") -> np.ndarray:
    """ss/phantom.py:359-402 with the reference's own cost structure, for CPU timing only.

    Same result as ``reference_deskew``, but built the way the reference builds it: an
    (n, U, W) float64 pile of per-slice canvases (ss/phantom.py:390), one ``np.interp``
    call per frame column for linear slices (ss/phantom.py:396-400), then one max over the
    pile, rint and clip (ss/phantom.py:401-402).  ``bench.py --impl reference --config 1``
    times it beside the streaming path.
    """
    stack = np.asarray(stack)
    n, h, w = stack.shape
    pile = np.zeros((n, canvas_height(n, h, shear), w), dtype=np.float64)
    rows_in_frame = np.arange(h)
    for i in range(n):
        frame = stack[i]
        if interp == "nearest":
            top = nearest_offset(i, shear)
            pile[i, top:top + h] = frame
            continue
        lo, hi = linear_span(i, shear, h)
        targets = np.arange(lo, hi + 1, dtype=np.float64)
        sample_at = i * shear + rows_in_frame
        for col in range(w):
            pile[i, lo:hi + 1, col] = np.interp(targets, sample_at, frame[:, col].astype(np.float64))
    return np.clip(np.rint(pile.max(axis=0)), 0, MAX_INTENSITY).astype(np.uint16)


# ---------------------------------------------------------------------------
# display warp and rolling mode

def warp_projection(projection: np.ndarray, warp_scale: float) -> np.ndarray:
    """ss/pipeline.py:434-457 restated."""
    rows = projection.shape[0]
    out_rows = int(round(rows * warp_scale))
    if warp_scale == 1.0:
        return projection.copy()
    m = np.clip(np.arange(out_rows, dtype=np.float64) / warp_scale, 0, rows - 1)
    m0 = np.floor(m).astype(np.int64)
    m1 = np.minimum(m0 + 1, rows - 1)
    f = (m - m0)[:, None]
    vals = (1.0 - f) * projection[m0].astype(np.float64) + f * projection[m1].astype(np.float64)
    return np.rint(vals).astype(np.uint16)


def rolling_band(ring: list, shear: float, interp: str, h: int, w: int,
                 lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    """ss/pipeline.py:361-377: band max with first-max-wins contributor (ring order)."""
    band = np.zeros((hi - lo + 1, w), dtype=np.uint16)
    contrib = np.full((hi - lo + 1, w), -1, dtype=np.int16)
    for k, px in enumerate(ring):
        if px is None:
            continue
        klo, khi, rows = slice_rows(px, k, shear, interp, "canvas")
        olo, ohi = max(klo, lo), min(khi, hi)
        if olo > ohi:
            continue
        r = rows[olo - klo:ohi - klo + 1]
        seg = band[olo - lo:ohi - lo + 1]
        better = r > seg
        seg[better] = r[better]
        contrib[olo - lo:ohi - lo + 1][better] = k
    return band, contrib


# ---------------------------------------------------------------------------
# display encode

def encode_gray8(pixels: np.ndarray) -> tuple[np.ndarray, int, int]:
    """skewstream/server.py:83-91 restated: (payload uint8, g8_offset, g8_range)."""
    lo, hi = int(pixels.min()), int(pixels.max())
    rng = hi - lo
    if rng == 0:
        return np.zeros(pixels.shape, dtype=np.uint8), lo, 0
    scaled = (pixels.astype(np.float64) - lo) * (255.0 / rng)
    return np.rint(scaled).astype(np.uint8), lo, rng
