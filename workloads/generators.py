"""Seeded synthetic matrix generators (inputs only; no method arithmetic).

Recipes (BASELINE.json configs):

* grid_gmrf(N, theta): J = I - theta*Adj(N x N 4-neighbour grid, free boundary),
  natural ordering i = r*N + c.  Stands in for the paper's 5000x5000 GMRF
  (§5.2; reading G15).
* torus_laplacian(N): Laplacian of the N x N torus (periodic 4-neighbour grid),
  diag 4, off-diagonal -1 (BASELINE.json configs[1]).
* random_nonsingular(d, seed): diag 3.0 + 8 distinct off-diagonal columns per
  row drawn uniformly, values U(-0.1, 0.1) (BASELINE.json configs[4]; reading G19).
* random_spd(d, seed): the paper's §5.1 generator: 5 U[-1,1]
  off-diagonals per row, symmetrised, diagonal = abs row sum + 1e-3 (reading G23).
* triangular_b / complete_graph_laplacian: pin inputs with closed-form answers.
"""
import numpy as np

from .csr import CSR, from_coo

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_at(seed, counter):
    """SplitMix64 output at position `counter` (>=1) of the stream seeded `seed`.

    Vectorised over numpy uint64 arrays (wrap-around arithmetic).  Used here only
    to draw *matrix* entries for random_nonsingular / random_spd.
    """
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.asarray(counter, dtype=np.uint64) * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _unit_double(z):
    """Top 53 bits -> float64 in [0, 1)."""
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def grid_gmrf(N: int, theta: float, M: int = None) -> CSR:
    """J = I - theta*Adj on an N x M grid (M defaults to N), free boundary.

    Each row i=r*M+c holds, in ascending column order, i-M, i-1, i, i+1, i+M
    (those inside the grid).  Diagonal 1.0, off-diagonal -theta.
    """
    M = N if M is None else M
    d = N * M
    i = np.arange(d, dtype=np.int64)
    r, c = i // M, i % M
    cand = np.stack([i - M, i - 1, i, i + 1, i + M], axis=1)
    ok = np.stack([r > 0, c > 0, np.ones(d, bool), c < M - 1, r < N - 1], axis=1)
    vals = np.full((d, 5), -float(theta))
    vals[:, 2] = 1.0
    counts = ok.sum(axis=1)
    rp = np.zeros(d + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    col = cand[ok].astype(np.int32)
    val = vals[ok]
    return CSR(d, d, rp, col, val)


def torus_laplacian(N: int) -> CSR:
    """Laplacian of the N x N torus C_N x C_N (N >= 3): 4 on the diagonal, -1 to
    the four periodic neighbours; columns sorted ascending."""
    if N < 3:
        raise ValueError("torus needs N >= 3 for a simple graph")
    d = N * N
    i = np.arange(d, dtype=np.int64)
    r, c = i // N, i % N
    cand = np.stack([((r - 1) % N) * N + c, r * N + (c - 1) % N, i,
                     r * N + (c + 1) % N, ((r + 1) % N) * N + c], axis=1)
    vals = np.tile(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), (d, 1))
    order = np.argsort(cand, axis=1, kind="stable")
    cand = np.take_along_axis(cand, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    rp = np.arange(0, 5 * d + 1, 5, dtype=np.int64)
    return CSR(d, d, rp, cand.reshape(-1).astype(np.int32), vals.reshape(-1))


def complete_graph_laplacian(n: int) -> CSR:
    """Laplacian of K_n: n-1 on the diagonal, -1 elsewhere (dense CSR)."""
    rows = np.repeat(np.arange(n), n)
    cols = np.tile(np.arange(n), n)
    vals = np.where(rows == cols, float(n - 1), -1.0)
    return from_coo(n, n, rows, cols, vals)


def random_nonsingular(d: int, seed: int = 1, per_row: int = 8,
                       diag: float = 3.0, scale: float = 0.1) -> CSR:
    """BASELINE configs[4] generator, reading G19.

    Row i draws `per_row` distinct off-diagonal columns by rejection from the
    counter stream splitmix64_at(seed, 1 + i*64 + t), t = attempt index,
    column = (z >> 32) * d >> 32 (multiply-shift, d < 2^32).  Values
    U(-scale, scale) from splitmix64_at(seed ^ 0xD1B54A32D192ED03, 1 + i*per_row + s).
    """
    if d < per_row + 1:
        raise ValueError("d too small")
    chosen = np.full((d, per_row), -1, dtype=np.int64)
    count = np.zeros(d, dtype=np.int64)
    rows = np.arange(d, dtype=np.int64)
    dd = np.uint64(d)
    for t in range(64):
        act = rows[count < per_row]
        if act.size == 0:
            break
        z = splitmix64_at(seed, 1 + act.astype(np.uint64) * np.uint64(64) + np.uint64(t))
        col = ((z >> np.uint64(32)) * dd >> np.uint64(32)).astype(np.int64)
        dup = (chosen[act] == col[:, None]).any(axis=1) | (col == act)
        acc = act[~dup]
        chosen[acc, count[acc]] = col[~dup]
        count[acc] += 1
    if np.any(count < per_row):
        raise RuntimeError("rejection sampling did not converge")
    vseed = np.uint64(seed) ^ np.uint64(0xD1B54A32D192ED03)
    ctr = 1 + np.arange(d * per_row, dtype=np.uint64)
    u = _unit_double(splitmix64_at(vseed, ctr)).reshape(d, per_row)
    offv = -scale + 2.0 * scale * u
    r = np.concatenate([np.repeat(rows, per_row), rows])
    c = np.concatenate([chosen.reshape(-1), rows])
    v = np.concatenate([offv.reshape(-1), np.full(d, float(diag))])
    return from_coo(d, d, r, c, v)


def random_spd(d: int, seed: int = 1, per_row: int = 5, shift: float = 1e-3,
               device: str = "cpu") -> CSR:
    """Paper §5.1 generator, reading G23: every row draws `per_row`
    off-diagonal columns uniformly (splitmix64_at(seed, 1+t), multiply-shift) with
    values U[-1,1] (second stream); each draw (i,j,v) also sets the transposed entry
    (j,i) = v; coinciding draws are summed; self-draws are dropped; the diagonal is the
    absolute off-diagonal row sum (numpy add.reduceat over the row) + `shift`, which
    makes C strictly diagonally dominant, hence SPD.

    The sort/dedupe runs in torch on `device` (a CUDA device makes d = 3e7 take
    seconds); the arrays returned are numpy.
    """
    import torch
    dev = torch.device(device)
    n = d * per_row
    ctr = 1 + np.arange(n, dtype=np.uint64)
    cols = ((splitmix64_at(seed, ctr) >> np.uint64(32)) * np.uint64(d) >> np.uint64(32)).astype(np.int64)
    vals = -1.0 + 2.0 * _unit_double(splitmix64_at(np.uint64(seed) ^ np.uint64(0xA0761D6478BD642F), ctr))
    del ctr
    rows = torch.arange(d, dtype=torch.int64, device=dev).repeat_interleave(per_row)
    cols_t = torch.from_numpy(cols).to(dev)
    vals_t = torch.from_numpy(vals).to(dev)
    del cols, vals
    keep = rows != cols_t
    rows, cols_t, vals_t = rows[keep], cols_t[keep], vals_t[keep]
    # both orientations + a zero placeholder for every diagonal entry
    diag = torch.arange(d, dtype=torch.int64, device=dev)
    keys = torch.cat([rows * d + cols_t, cols_t * d + rows, diag * d + diag])
    v = torch.cat([vals_t, vals_t, torch.zeros(d, dtype=torch.float64, device=dev)])
    del rows, cols_t, vals_t
    keys, order = torch.sort(keys, stable=True)
    v = v[order]
    del order
    ukeys, inv = torch.unique_consecutive(keys, return_inverse=True)
    del keys
    sv = torch.zeros(ukeys.numel(), dtype=torch.float64, device=dev).index_add_(0, inv, v)
    del inv, v
    r = (ukeys // d).cpu().numpy()
    c = (ukeys % d).cpu().numpy().astype(np.int32)
    sv = sv.cpu().numpy()
    del ukeys
    counts = np.bincount(r, minlength=d)
    rp = np.zeros(d + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    rowsum = np.add.reduceat(np.abs(sv), rp[:-1])  # sequential left-to-right per row
    isdiag = c == r
    sv[isdiag] = rowsum + shift
    return CSR(d, d, rp, c, sv)


def triangular_b(d: int, diag: float = 3.0, seed: int = 7, per_row: int = 3,
                 scale: float = 0.1) -> CSR:
    """Lower-triangular B: constant diagonal `diag` plus up to `per_row` random
    strictly-lower entries per row.  log|det B| = d*log|diag| exactly."""
    rows, cols, vals = [np.arange(d)], [np.arange(d)], [np.full(d, float(diag))]
    r = np.repeat(np.arange(d, dtype=np.int64), per_row)
    ctr = 1 + np.arange(d * per_row, dtype=np.uint64)
    z = splitmix64_at(seed, ctr)
    # column in [0, r): multiply-shift on r (rows 0 get none)
    c = ((z >> np.uint64(32)) * r.astype(np.uint64) >> np.uint64(32)).astype(np.int64)
    v = -scale + 2 * scale * _unit_double(splitmix64_at(seed + 1, ctr))
    keep = r > 0
    r, c, v = r[keep], c[keep], v[keep]
    key = r * d + c
    _, first = np.unique(key, return_index=True)
    rows.append(r[first]); cols.append(c[first]); vals.append(v[first])
    return from_coo(d, d, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
