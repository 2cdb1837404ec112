"""Independent brute-force restatement of the 27-point stencil in numpy / pure
Python ("dense brute-force oracle").  Shares no code with
oracle/spmvcomp_oracle.c; used to cross-check it on small grids."""
import itertools

import numpy as np


def dense_stencil(nx, ny, nz, diagonal=26.0, off_diagonal=-1.0):
    n = nx * ny * nz
    a = np.zeros((n, n))
    for iz, iy, ix in itertools.product(range(nz), range(ny), range(nx)):
        i = ix + nx * (iy + ny * iz)
        for dz, dy, dx in itertools.product((-1, 0, 1), repeat=3):
            x, y, z = ix + dx, iy + dy, iz + dz
            if 0 <= x < nx and 0 <= y < ny and 0 <= z < nz:
                j = x + nx * (y + ny * z)
                a[i, j] = diagonal if i == j else off_diagonal
    return a


def rel_err(y, ref, scale=None):
    """Element-wise relative deviation; where the reference is 0 the scale is
    sum_k |a_ik x_k| (unpinned choice 5)."""
    y = np.asarray(y)
    ref = np.asarray(ref)
    den = np.abs(ref) if scale is None else np.maximum(np.abs(ref), 0 * scale)
    if scale is not None:
        den = np.where(np.abs(ref) > 0, np.abs(ref), scale)
    den = np.where(den == 0, 1.0, den)
    return np.abs(y - ref) / den
