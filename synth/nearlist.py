"""Synthetic near-lists, standing in for the paper's sphere-union near
region N_Gamma_k and its Morton-sort search (§3.3), which are OUT of scope.

Rule: near(t) = { k : min_ij |x_t - y_ij^(k)| < 2 L_k }  U  {own panel of a node target},
L_k the panel's centerline arc length; optionally a forced list per row (config 1's
{k-1, k, k+1}).  Output: CSR over targets, panels ascending per row.

The exact node-min test is pruned with two bounds that need no approximation: a
panel bounding sphere (KD-tree pair search) and, per GL ring i (nodes at distance rho_i
from the ring centre x_c(s_i)), |x - x_c(s_i)| -/+ rho_i bracketing the ring's node
distances.  Only pairs inside that bracket get the exact min over the panel's nodes.
"""
import numpy as np
from scipy.spatial import cKDTree

_CHUNK = 1 << 21


def build_near_csr(x_trg, y_panels, ring_xc, rho_ring, L, own_panel, forced_rows=None):
    T = x_trg.shape[0]
    Ptot, Nn, _ = y_panels.shape
    cent = y_panels.mean(axis=1)
    Rk = np.sqrt(np.max(np.sum((y_panels - cent[:, None, :]) ** 2, axis=-1), axis=1))
    rad = 2 * L + Rk * 1.0000001 + 1e-12
    pairs = cKDTree(cent).sparse_distance_matrix(cKDTree(x_trg), float(rad.max()),
                                                 output_type="ndarray")
    K = pairs["i"].astype(np.int64)
    Tt = pairs["j"].astype(np.int64)
    keep = pairs["v"] <= rad[K]
    K, Tt = K[keep], Tt[keep]
    forced_n = 0 if forced_rows is None else forced_rows.shape[0]
    if forced_n:
        keep = Tt >= forced_n
        K, Tt = K[keep], Tt[keep]
    near = np.zeros(K.shape[0], bool)
    for a in range(0, K.shape[0], _CHUNK):
        k = K[a:a + _CHUNK]
        X = x_trg[Tt[a:a + _CHUNK]]
        rc = ring_xc[k]                        # [c, Ns, 3]
        d = np.sqrt((X[:, None, 0] - rc[:, :, 0]) ** 2 + (X[:, None, 1] - rc[:, :, 1]) ** 2
                    + (X[:, None, 2] - rc[:, :, 2]) ** 2)
        rr = rho_ring[k]
        lim = 2 * L[k]
        hi = np.min(d + rr, axis=1)
        lo = np.min(d - rr, axis=1)
        # shortcuts only where the bound clears the threshold by a relative 1e-9, so every decision
        # equals the exact rule  sqrt(min_j ((dx^2 + dy^2) + dz^2)) < 2 L_k  evaluated in fp64
        sure = hi < lim * (1 - 1e-9)
        maybe = np.nonzero((~sure) & (lo < lim * (1 + 1e-9)))[0]
        res = sure
        if maybe.size:
            Y = y_panels[k[maybe]]             # [m, Nn, 3]
            Xm = X[maybe]
            dm = np.min((Xm[:, None, 0] - Y[:, :, 0]) ** 2 + (Xm[:, None, 1] - Y[:, :, 1]) ** 2
                        + (Xm[:, None, 2] - Y[:, :, 2]) ** 2, axis=1)
            res[maybe] = np.sqrt(dm) < lim[maybe]
        near[a:a + _CHUNK] = res
    t_l = [Tt[near]]
    k_l = [K[near]]
    own_t = np.nonzero(own_panel >= 0)[0]
    if forced_n:
        own_t = own_t[own_t >= forced_n]
        t_l.append(np.repeat(np.arange(forced_n), forced_rows.shape[1]))
        k_l.append(forced_rows.reshape(-1).astype(np.int64))
    t_l.append(own_t)
    k_l.append(own_panel[own_t])
    key = np.sort(np.concatenate(t_l) * Ptot + np.concatenate(k_l), kind="stable")
    first = np.ones(key.shape[0], bool)
    first[1:] = key[1:] != key[:-1]
    key = key[first]
    t_u = key // Ptot
    k_u = key % Ptot
    counts = np.bincount(t_u, minlength=T)
    row_ptr = np.zeros(T + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, k_u.astype(np.int32)
