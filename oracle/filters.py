"""CPU restatement of the classical cone density filter (TEST INFRASTRUCTURE ONLY).

The reference package has only the Helmholtz filter (romtopt/filtering.py); SURVEY §8f rank 4
asks for the classical "linear hat" filter as an option.  Parity is unpinned against the
reference by construction; this restatement is the checker: an explicit sparse matrix
A[e, j] = w(e, j) / W_e with w(e, j) = max(0, R - |c_e - c_j|), element centres on the
structured grid, W_e = sum_j w(e, j).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def cone_matrix(nx: int, ny: int, nz: int, h: float, radius: float) -> sp.csr_matrix:
    dims = (nx, ny, nz if nz else 1)
    n = dims[0] * dims[1] * dims[2]
    idx = np.arange(n)
    i, j, k = idx % dims[0], (idx // dims[0]) % dims[1], idx // (dims[0] * dims[1])
    m = int(np.ceil(radius / h))
    rows, cols, vals = [], [], []
    for dz in range(-m, m + 1) if nz else [0]:
        for dy in range(-m, m + 1):
            for dx in range(-m, m + 1):
                w = radius - h * np.sqrt(dx * dx + dy * dy + dz * dz)
                if dx == dy == dz == 0 and w <= 0:
                    w = 1.0
                if w <= 0:
                    continue
                ii, jj, kk = i + dx, j + dy, k + dz
                ok = (ii >= 0) & (ii < dims[0]) & (jj >= 0) & (jj < dims[1]) & (kk >= 0) & (kk < dims[2])
                rows.append(idx[ok])
                cols.append((kk[ok] * dims[1] + jj[ok]) * dims[0] + ii[ok])
                vals.append(np.full(ok.sum(), w))
    a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    wsum = np.asarray(a.sum(axis=1)).ravel()
    return sp.diags(1.0 / wsum) @ a
