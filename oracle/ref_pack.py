"""Independent CPU CSR packer -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Writes the canonical CSR of the mode-1 matricised weights straight from the
definition, with NumPy, sharing nothing with the C++ packer in
paper_1608_01409_b200/csrc/plan.cpp.

Definition followed (Fig. 2 caption; Sec. 2.1):
  * one CSR row per output channel k ("rowptr[n] points to the first non-zero weight
    of the n-th output channel");
  * "For the j-th non-zero weight at (n,c,r,s), W.colidx[j] contains the offset to
    (c,r,s)-th element of tensor in, which is pre-computed by layout function as
    f(c,r,s)"; in CHW layout f(c,r,s) = (c*H_in + r)*W_in + s.
Build readings (R1-R3):
  * offsets are taken against the ZERO-PADDED input: Hp = H+2p, Wp = W+2p,
    colidx = ((g_k*(C/g) + c_local)*Hp + r)*Wp + s  (global input channel);
  * a nonzero is any w != 0.0f (+0 and -0 dropped); value bits copied unchanged;
  * within a row, nonzeros ascend in (c_local, r, s) == ascending colidx -- here by
    construction, because np.nonzero enumerates a C-ordered array in that order;
  * perm: within each group, channels by nnz DESCENDING, stable (ties by ascending k);
    groups in natural order (BASELINE.json north_star: "output channels sorted and
    binned by nnz").
"""
from __future__ import annotations

import numpy as np


def ref_pack(w: np.ndarray, H: int, W: int, pad: int, groups: int):
    """w: float32 [K, C/g, R, S].  Returns dict(rowptr int32[K+1], colidx int32[nnz],
    values float32[nnz], perm int32[K], nnz_per_row int64[K])."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    K, Cg, R, S = w.shape
    Hp, Wp = H + 2 * pad, W + 2 * pad
    Kg = K // groups
    rows_col, rows_val, counts = [], [], []
    for k in range(K):
        g = k // Kg
        cl, r, s = np.nonzero(w[k] != 0.0)          # C-order => ascending (cl, r, s)
        c = g * Cg + cl.astype(np.int64)
        col = (c * Hp + r) * Wp + s
        rows_col.append(col)
        rows_val.append(w[k][cl, r, s])
        counts.append(len(col))
    counts = np.asarray(counts, dtype=np.int64)
    rowptr = np.zeros(K + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    colidx = np.concatenate(rows_col) if K else np.zeros(0, np.int64)
    values = np.concatenate(rows_val) if K else np.zeros(0, np.float32)
    perm = []
    for g in range(groups):
        ks = np.arange(g * Kg, (g + 1) * Kg)
        # stable sort on -nnz keeps ascending k among equal counts
        order = np.argsort(-counts[ks], kind="stable")
        perm.extend(ks[order].tolist())
    return dict(
        rowptr=rowptr.astype(np.int32),
        colidx=colidx.astype(np.int32),
        values=values.astype(np.float32),
        perm=np.asarray(perm, dtype=np.int32),
        nnz_per_row=counts,
    )


def ref_densify(rowptr, colidx, values, K, C, R, S, H, W, pad, groups):
    """Inverse of ref_pack: decode colidx -> (c, r, s) and scatter values back into a
    dense [K, C/g, R, S] array (SPEC.md:79-83 'densify').  Used by the round-trip pin."""
    Hp, Wp = H + 2 * pad, W + 2 * pad
    Cg, Kg = C // groups, K // groups
    out = np.zeros((K, Cg, R, S), dtype=np.float32)
    for k in range(K):
        g = k // Kg
        for j in range(int(rowptr[k]), int(rowptr[k + 1])):
            off = int(colidx[j])
            c, rem = divmod(off, Hp * Wp)
            r, s = divmod(rem, Wp)
            out[k, c - g * Cg, r, s] = values[j]
    return out
