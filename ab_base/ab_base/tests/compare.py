"""Parity comparator: indices bit-exact, values per
(row-element, column-element) block in max-norm relative error, RHS per
element segment in max-norm relative error."""

from __future__ import annotations

import numpy as np

REL_TOL = 1e-12  # north star: values within 1e-12 relative, max-norm per block


def block_rel_errors(row_ptr, col_idx, vals, ref_vals, offsets, row_elements):
    """Max-norm relative error of every dense block of the given rows.

    Returns an array with one entry per (row element, neighbour) block.
    A block whose reference is exactly zero must be exactly zero too
    (error 0 if so, inf otherwise).
    """
    offsets = np.asarray(offsets)
    counts = np.diff(offsets)
    errs = []
    r = 0
    for e in row_elements:
        ne = int(counts[e])
        a, b = row_ptr[r], row_ptr[r + 1]
        cols = col_idx[a:b]
        L = b - a
        blk_v = vals[row_ptr[r]:row_ptr[r] + ne * L].reshape(ne, L)
        blk_r = ref_vals[row_ptr[r]:row_ptr[r] + ne * L].reshape(ne, L)
        col_el = np.searchsorted(offsets, cols, side="right") - 1
        starts = np.flatnonzero(np.r_[True, col_el[1:] != col_el[:-1]])
        ends = np.r_[starts[1:], L]
        for s, t in zip(starts, ends):
            ref = blk_r[:, s:t]
            diff = np.abs(blk_v[:, s:t] - ref).max()
            scale = np.abs(ref).max()
            errs.append(0.0 if diff == 0.0 else (diff / scale if scale > 0 else np.inf))
        r += ne
    return np.asarray(errs)


def rhs_rel_errors(rhs, ref, offsets, row_elements):
    out = []
    for e in row_elements:
        a, b = offsets[e], offsets[e + 1]
        d = np.abs(rhs[a:b] - ref[a:b]).max() if b > a else 0.0
        s = np.abs(ref[a:b]).max() if b > a else 0.0
        out.append(0.0 if d == 0.0 else (d / s if s > 0 else np.inf))
    return np.asarray(out)


def assert_parity(matrix, rhs, ref, offsets, row_elements=None, tol=REL_TOL):
    """``ref`` = (row_ptr, col_idx, values, rhs) from the oracle."""
    rp, ci, v, r = ref
    if row_elements is None:
        row_elements = np.arange(len(offsets) - 1)
    assert np.array_equal(np.asarray(matrix.row_ptr), rp), "row_ptr differs"
    assert np.array_equal(np.asarray(matrix.col_idx), ci), "col_idx differs"
    be = block_rel_errors(rp, ci, np.asarray(matrix.values), v, offsets, row_elements)
    re = rhs_rel_errors(np.asarray(rhs), r, offsets, row_elements)
    assert be.size == 0 or be.max() <= tol, f"block rel err {be.max():.3e} > {tol}"
    assert re.size == 0 or re.max() <= tol, f"rhs rel err {re.max():.3e} > {tol}"
    return (be.max() if be.size else 0.0), (re.max() if re.size else 0.0)
