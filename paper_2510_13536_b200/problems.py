"""Seeded synthetic problems for the BASELINE.json configurations.

The reference has generators only for 2-D problems (sparse.py:259-342); the
3-D / banded / random configurations are new code pinned here (SURVEY.md
§8(d) "Synthetic inputs").  Right-hand sides built as b = A x use
`spmv_fp64_host`, which reproduces the reference's unfused, row-sequential
FP64 SpMV (_fast.py:284-290) so b is bit-identical to what the reference
would compute.
"""
import numpy as np

from .sparse import CsrMatrix, laplacian_2d

__all__ = ["spmv_fp64_host", "stencil_matrix", "poisson_3d", "config1", "config2",
           "config3", "config4", "config5", "config5_style", "random_irregular_spd",
           "matrix_digest", "CONFIGS"]


def spmv_fp64_host(A, x):
    """y_i = (((0 + a_i0 x_c0) + a_i1 x_c1) + ...) in FP64, no FMA: the
    reference's spmv_fp64 order, vectorised over rows (one pass per entry
    position)."""
    rp = A.row_ptr
    lens = np.diff(rp)
    y = np.zeros(A.n_rows)
    if A.nnz == 0:
        return y
    for k in range(int(lens.max())):
        rows = np.nonzero(lens > k)[0]
        idx = rp[rows] + k
        prod = A.values[idx] * x[A.col_idx[idx]]
        y[rows] = y[rows] + prod
    return y


def matrix_digest(A):
    """SHA-256 over (n, row_ptr, col_idx as int64, values): pins a generated
    problem so a golden recorded against it cannot silently drift."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.int64(A.n_rows).tobytes())
    h.update(np.ascontiguousarray(A.row_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(A.col_idx, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(A.values, dtype=np.float64).tobytes())
    return h.hexdigest()


def stencil_matrix(dims, offsets, diag_value, off_value=-1.0):
    """Constant-coefficient stencil on a lexicographic grid (x fastest).
    offsets: list of (dz, dy, dx) excluding (0,0,0); columns ascending."""
    nz, ny, nx = dims
    n = nz * ny * nx
    idx = np.arange(n, dtype=np.int64)
    z, rem = np.divmod(idx, ny * nx)
    y, x = np.divmod(rem, nx)
    allo = sorted(list(offsets) + [(0, 0, 0)], key=lambda o: o[0] * ny * nx + o[1] * nx + o[2])
    cols, masks, vals = [], [], []
    for dz, dy, dx in allo:
        m = ((z + dz >= 0) & (z + dz < nz) & (y + dy >= 0) & (y + dy < ny)
             & (x + dx >= 0) & (x + dx < nx))
        cols.append(idx + dz * ny * nx + dy * nx + dx)
        masks.append(m)
        vals.append(diag_value if (dz, dy, dx) == (0, 0, 0) else off_value)
    cols = np.stack(cols, axis=1)
    mask = np.stack(masks, axis=1)
    vv = np.broadcast_to(np.array(vals), cols.shape)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=rp[1:])
    return CsrMatrix(n, n, rp, cols[mask], vv[mask].copy())


def poisson_3d(k):
    """7-point 3-D Poisson, diag 6, off -1 on a k^3 grid."""
    offs = [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 1), (0, 1, 0), (1, 0, 0)]
    return stencil_matrix((k, k, k), offs, 6.0)


def config1():
    """C1: 2-D 5-point Poisson 256x256; x_true ~ U(-1,1) seed 0; b = A x_true
    (unfused sequential); eps 1e-12, max 10,000."""
    A = laplacian_2d(256)
    x_true = np.random.default_rng(0).uniform(-1.0, 1.0, A.n_rows)
    b = spmv_fp64_host(A, x_true)
    return dict(name="C1", A=A, b=b, x_star=x_true, epsilon=1e-12, max_iterations=10000)


def config2(k=128):
    """C2: 3-D 7-point Poisson k^3 (k=128: n=2,097,152, nnz=14,581,760);
    b = A ones (exact); eps 1e-12, max 20,000."""
    A = poisson_3d(k)
    ones = np.ones(A.n_rows)
    b = spmv_fp64_host(A, ones)
    return dict(name="C2", A=A, b=b, x_star=ones, epsilon=1e-12, max_iterations=20000)


def config3(k=160, seed=1):
    """C3: 3-D 27-point stencil k^3.  Off-diagonals -(1 + 0.1 U(-1,1)), one
    draw per unordered pair (upper triangle, CSR order) from
    default_rng(seed), mirrored; a_ii = max(26, sum_j |a_ij|) + 1e-3 (pinned,
    BASELINE leaves it open); x_true = the same rng's standard_normal(n);
    b = A x_true; eps 1e-12."""
    offs = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
            if (dz, dy, dx) != (0, 0, 0)]
    S = stencil_matrix((k, k, k), offs, 0.0)
    n = S.n_rows
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(S.row_ptr))
    upper = S.col_idx > rows
    rng = np.random.default_rng(seed)
    vals = np.zeros(S.nnz)
    vals[upper] = -(1.0 + 0.1 * rng.uniform(-1.0, 1.0, int(upper.sum())))
    # mirror: entry (i,j) with j<i takes the value drawn for (j,i)
    lower = S.col_idx < rows
    key_up = rows[upper] * n + S.col_idx[upper]
    key_lo = S.col_idx[lower] * n + rows[lower]
    pos = np.searchsorted(key_up, key_lo)  # upper entries are in ascending (row, col) order
    vals[lower] = vals[upper][pos]
    diag = rows == S.col_idx
    absrow = np.zeros(n)
    np.add.at(absrow, rows[~diag], np.abs(vals[~diag]))
    vals[diag] = np.maximum(26.0, absrow) + 1e-3
    A = CsrMatrix(n, n, S.row_ptr, S.col_idx, vals)
    x_true = rng.standard_normal(n)
    b = spmv_fp64_host(A, x_true)
    return dict(name="C3", A=A, b=b, x_star=x_true, epsilon=1e-12, max_iterations=20000)


def config4(n=1_000_000, half_band=9, delta=1e-3, seed=2):
    """C4: ill-conditioned banded SPD, A = D^1/2 L D^1/2.  L: off-diagonals
    U(-1,0), one draw per upper pair (offset-major), mirrored; L_ii =
    sum_j |L_ij| + delta (delta pinned at 1e-3); D_ii =
    10^U(0,6).  The scaled value is computed once per upper pair and
    mirrored.  b = fl(A ones); eps 1e-10, max 200,000."""
    rng = np.random.default_rng(seed)
    up = {}
    for o in range(1, half_band + 1):
        up[o] = rng.uniform(-1.0, 0.0, n - o)       # L[i, i+o], i = 0..n-o-1
    d = 10.0 ** rng.uniform(0.0, 6.0, n)
    s = np.sqrt(d)
    absrow = np.zeros(n)
    for o, v in up.items():
        absrow[:n - o] += np.abs(v)
        absrow[o:] += np.abs(v)
    ldiag = absrow + delta
    cols, vals, masks = [], [], []
    idx = np.arange(n, dtype=np.int64)
    for o in range(-half_band, half_band + 1):
        c = idx + o
        m = (c >= 0) & (c < n)
        v = np.zeros(n)
        if o == 0:
            v = (s * ldiag) * s
        elif o > 0:
            v[:n - o] = (s[:n - o] * up[o]) * s[o:]
        else:
            v[-o:] = (s[:n + o] * up[-o]) * s[-o:]   # mirror of (i+o, i)
        cols.append(c)
        vals.append(v)
        masks.append(m)
    cols = np.stack(cols, 1)
    vals = np.stack(vals, 1)
    mask = np.stack(masks, 1)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    A = CsrMatrix(n, n, rp, cols[mask], vals[mask])
    ones = np.ones(n)
    b = spmv_fp64_host(A, ones)
    return dict(name="C4", A=A, b=b, x_star=ones, epsilon=1e-10, max_iterations=200000)


def random_irregular_spd(n, seed=3, device="cuda", near_width=1024, cmin=16, cmax=64):
    """BASELINE config 5 generator, on the GPU (torch, seeded Philox).

    Row i draws c ~ U{cmin..cmax} off-diagonal entries: ceil(c/2) columns
    uniform over [i - near_width, i + near_width] clipped to [0, n), minus i;
    the rest uniform in [0, n); values U(-1, 0); far draws landing on the
    diagonal are dropped.  The pattern is
    symmetrised by adding (i, j, v) and (j, i, v) and summing duplicates (in
    sorted order, deterministic), then a_ii = 1.01 * sum_j |a_ij| (strictly
    diagonally dominant -> SPD).  Returns a DeviceCsrMatrix (int32 indices).
    """
    import torch
    from .sparse import DeviceCsrMatrix
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    cnt = torch.randint(cmin, cmax + 1, (n,), generator=g, device=dev)
    T = int(cnt.sum())
    rows = torch.repeat_interleave(torch.arange(n, device=dev), cnt)
    start = torch.cumsum(cnt, 0) - cnt
    k = torch.arange(T, device=dev) - torch.repeat_interleave(start, cnt)
    near = k < torch.repeat_interleave((cnt + 1) // 2, cnt)
    del k, start
    # near: uniform over [i - W, i + W] clipped to [0, n), excluding i
    lo = (rows - near_width).clamp(min=0)
    m = (rows + near_width).clamp(max=n - 1) - lo          # candidates (i excluded)
    u = (torch.rand(T, generator=g, device=dev, dtype=torch.float64) * m).floor().to(torch.int64)
    u = torch.minimum(u, m - 1)
    cn = lo + u
    cn = cn + (cn >= rows).to(torch.int64)
    del lo, m, u
    far = torch.randint(0, n, (T,), generator=g, device=dev)
    cols = torch.where(near, cn, far)
    del cn, far, near
    vals = -torch.rand(T, generator=g, device=dev, dtype=torch.float64)
    keep = cols != rows
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    del keep
    # duplicates are summed per UNORDERED pair (canonical key min*n + max, in
    # draw order, deterministic) and the sum is mirrored, so A is exactly
    # symmetric
    lo = torch.minimum(rows, cols)
    hi = torch.maximum(rows, cols)
    del rows, cols
    key, order = torch.sort(lo * n + hi, stable=True)
    del lo, hi
    v = vals[order]
    del vals, order
    first = torch.ones_like(key, dtype=torch.bool)
    first[1:] = key[1:] != key[:-1]
    run = torch.cumsum(first, 0) - 1
    out = v[first].clone()
    pos = torch.arange(key.numel(), device=dev) - torch.nonzero(first).squeeze(1)[run]
    r = 1
    while True:  # head + 2nd + 3rd ... of each run, in draw order
        sel = pos == r
        if not bool(sel.any()):
            break
        out.index_add_(0, run[sel], v[sel])
        r += 1
    pkey = key[first]
    del key, v, first, run, pos
    pa, pb = pkey // n, pkey % n
    del pkey
    key2, order = torch.sort(torch.cat([pa * n + pb, pb * n + pa]))
    out = torch.cat([out, out])[order]
    del pa, pb, order
    nu = key2.numel()
    urow = key2 // n
    ucol = key2 % n
    del key2
    counts = torch.bincount(urow, minlength=n)
    rp_u = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp_u[1:] = torch.cumsum(counts, 0)
    cs = torch.zeros(nu + 1, dtype=torch.float64, device=dev)
    cs[1:] = torch.cumsum(out.abs(), 0)
    rowsum = cs[rp_u[1:]] - cs[rp_u[:-1]]
    del cs
    diag = 1.01 * rowsum
    nnz = nu + n
    # final index: off-diagonal entry e of row r -> e + r + [col > r]; diagonal
    # of row r -> rp_u[r] + (#entries of row r with col < r) + r
    e = torch.arange(nu, device=dev)
    fidx = e + urow + (ucol > urow).to(torch.int64)
    del e
    col_f = torch.empty(nnz, dtype=torch.int32, device=dev)
    val_f = torch.empty(nnz, dtype=torch.float64, device=dev)
    col_f[fidx] = ucol.to(torch.int32)
    val_f[fidx] = out
    below = torch.bincount(urow[ucol < urow], minlength=n)
    didx = rp_u[:-1] + below + torch.arange(n, device=dev)
    col_f[didx] = torch.arange(n, device=dev, dtype=torch.int32)
    val_f[didx] = diag
    rp_f = (rp_u + torch.arange(n + 1, device=dev)).to(torch.int32)
    del urow, ucol, out, fidx, didx, rp_u, below
    torch.cuda.empty_cache() if dev.type == "cuda" else None
    return DeviceCsrMatrix(n, n, rp_f, col_f, val_f) if dev.type == "cuda" else \
        (rp_f, col_f, val_f)


def config5(n=16_000_000, seed=3):
    """C5: random irregular SPD (multi-GPU config), n = 16M, ~1.3e9 nnz, built
    on the GPU; b ~ U(-1,1) from default_rng(seed); eps 1e-12 (DW, QTW)."""
    A = random_irregular_spd(n, seed=seed)
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    return dict(name="C5", A=A, b=b, x_star=None, epsilon=1e-12, max_iterations=20000)


def config5_style(n=1_000_000, seed=3):
    """A C5-style instance small enough for a CPU solve of the reference order
    (parity at scale, tests/golden/scale.json): the config-5 generator run on the host (torch
    CPU generator -- deterministic, but a different stream from the CUDA
    one, so this is a different matrix from a device-built C5 of the same
    n), b ~ U(-1,1) from default_rng(seed); eps 1e-12."""
    rp, col, val = random_irregular_spd(n, seed=seed, device="cpu")
    A = CsrMatrix(n, n, rp.numpy().astype(np.int64), col.numpy().astype(np.int64), val.numpy())
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    return dict(name="C5s", A=A, b=b, x_star=None, epsilon=1e-12, max_iterations=20000)


def config4_style(n=100_000):
    """A C4-style instance (the config-4 generator at n = 1e5: same band, same
    10^U(0,6) diagonal scaling, so precision still moves the iteration count)
    small enough for host solves of the reference order in every arithmetic
    (parity at scale, tests/golden/scale.json)."""
    c = config4(n=n)
    c["name"] = "C4s"
    return c


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5,
           "C5s": config5_style, "C4s": config4_style}
