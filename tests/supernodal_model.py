"""Test-only numpy model of the device supernodal LDL' (csrc/ldl.cu).

Runs the same left-looking algorithm over the exported symbolic arrays so the
symbolic analysis (supernodes, update lists, scatter maps) can be validated on
CPU, without a GPU.  Never used by the product path.
"""
from __future__ import annotations

import numpy as np


def assemble(sym, n, P, A, hdiag, hblocks, delta_s):
    """Panel value array from the scatter maps (base image + −H), as the device does."""
    loff = sym.array("sn_loff")
    vals = np.zeros(int(loff[-1]))
    mp = sym.array("map_p")
    sel = mp >= 0
    vals[mp[sel]] = P.values[sel]
    vals[sym.array("map_a")] = A.values
    md = sym.array("map_diag")
    dim = len(md)
    sign = np.where(np.arange(dim) < n, 1.0, -1.0)
    vals[md] += sign * delta_s
    lin = len(hdiag)
    vals[md[n:n + lin]] += -hdiag
    mh = sym.array("map_hblk")
    vals[mh] += -hblocks
    return vals


def factor(sym, vals, sign_perm, delta_s, delta_d=0.0):
    col = sym.array("sn_col")
    rptr = sym.array("sn_rptr")
    rows = sym.array("sn_rows")
    loff = sym.array("sn_loff")
    uptr = sym.array("upd_ptr")
    usrc = sym.array("upd_src")
    up0 = sym.array("upd_p0")
    up1 = sym.array("upd_p1")
    order = sym.array("order")
    L = vals.copy()
    dim = int(col[-1])
    D = np.zeros(dim)
    ns = len(col) - 1
    for J in order:
        c0, w = col[J], col[J + 1] - col[J]
        r0, r = rptr[J], rptr[J + 1] - rptr[J]
        rowsJ = rows[r0:r0 + r]
        pan = L[loff[J]:loff[J] + w * r].reshape(w, r).T          # r x w view (column-major panel)
        for u in range(uptr[J], uptr[J + 1]):
            K = usrc[u]
            p0, p1 = up0[u], up1[u]
            kc0, wK = col[K], col[K + 1] - col[K]
            kr0, rK = rptr[K], rptr[K + 1] - rptr[K]
            LK = L[loff[K]:loff[K] + wK * rK].reshape(wK, rK).T
            DK = D[kc0:kc0 + wK]
            rowsK = rows[kr0:kr0 + rK]
            upd = (LK[p0:] * DK) @ LK[p0:p1].T                       # (rK-p0) x (p1-p0)
            tr = np.searchsorted(rowsJ, rowsK[p0:])
            tc = rowsK[p0:p1] - c0
            for cc in range(p1 - p0):
                sel = np.arange(p1 - p0 - cc) + cc if False else slice(cc, None)
                pan[tr[sel], tc[cc]] -= upd[sel, cc]
        for j in range(w):
            d = pan[j, j]
            if abs(d) < delta_s:
                d = delta_s if sign_perm[c0 + j] > 0 else -delta_s
            D[c0 + j] = d
            pan[j, j] = 1.0
            pan[j + 1:, j] /= d
            for c in range(j + 1, w):
                pan[c:, c] -= pan[c:, j] * d * pan[c, j]
        L[loff[J]:loff[J] + w * r] = pan.T.ravel()
    return L, D


def dense_factor(sym, L, D):
    """Dense unit-lower L (permuted order) from the panel storage."""
    col = sym.array("sn_col")
    rptr = sym.array("sn_rptr")
    rows = sym.array("sn_rows")
    loff = sym.array("sn_loff")
    dim = int(col[-1])
    Ld = np.eye(dim)
    for J in range(len(col) - 1):
        c0, w = col[J], col[J + 1] - col[J]
        r0, r = rptr[J], rptr[J + 1] - rptr[J]
        pan = L[loff[J]:loff[J] + w * r].reshape(w, r).T
        for j in range(w):
            Ld[rows[r0 + j + 1:r0 + r], c0 + j] = pan[j + 1:, j]
    return Ld


def factor_inbox(sym, vals, sign_perm, delta_s):
    """Model of the device push/pull factorisation (inbox maps of the symbolic analysis)."""
    col = sym.array("sn_col")
    rptr = sym.array("sn_rptr")
    loff = sym.array("sn_loff")
    order = sym.array("order")
    cb_off = sym.array("cb_off")
    push = sym.array("push_pos")
    irow = sym.array("irow_ptr")
    tgt = sym.array("inbox_tgt")
    inbox = np.zeros(int(cb_off[-1]))
    L = vals.copy()
    D = np.zeros(int(col[-1]))
    for J in order:
        c0, w = col[J], col[J + 1] - col[J]
        r0, r = rptr[J], rptr[J + 1] - rptr[J]
        flat = L[loff[J]:loff[J] + w * r].copy()            # column-major panel, flat index tc*r + tr
        for tr in range(r):
            for e in range(irow[r0 + tr], irow[r0 + tr + 1]):
                flat[tgt[e]] -= inbox[e]
        pan = flat.reshape(w, r).T
        for j in range(w):
            d = pan[j, j]
            if abs(d) < delta_s:
                d = delta_s if sign_perm[c0 + j] > 0 else -delta_s
            D[c0 + j] = d
            pan[j, j] = 1.0
            pan[j + 1:, j] /= d
            for c in range(j + 1, w):
                pan[c:, c] -= pan[c:, j] * d * pan[c, j]
        L[loff[J]:loff[J] + w * r] = pan.T.ravel()
        o = r - w
        if o:
            off = pan[w:, :]
            C = (off * D[c0:c0 + w]) @ off.T
            t = 0
            for b in range(o):
                for a in range(b, o):
                    inbox[push[cb_off[J] + t]] = C[a, b]
                    t += 1
    return L, D
