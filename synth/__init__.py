"""Seeded synthetic instance generators (0-1 ILPs) shared by tests, bench and smoke.

This module holds NONE of the method's arithmetic: it only draws costs and
writes linear constraint rows (the input of Def. "Binary Program" P:555-565 in
the row form of Example "ILP" P:567-577).  Both the oracle (oracle/) and the
product (paper_2111_10270_b200/) consume its output; neither is imported here.

Workload shapes follow SURVEY.md §8(d) / DESIGN.md §4 (synthetic look-alikes
of the paper's datasets P:474-485, sizes P:383-385).
"""
from __future__ import annotations

import dataclasses

import numpy as np

LE, EQ, GE = -1, 0, 1


@dataclasses.dataclass
class Problem:
    """CSR rows: row j is sum_p col_coef[p]*x[col_var[p]] rel[j] rhs[j], p in row j."""
    n_vars: int
    cost: np.ndarray      # float64 [n_vars]
    row_ptr: np.ndarray   # int64 [n_cons+1]
    col_var: np.ndarray   # int32, strictly ascending within a row
    col_coef: np.ndarray  # int32, nonzero
    rel: np.ndarray       # int8: -1 <=, 0 ==, +1 >=
    rhs: np.ndarray       # int64
    name: str = ""

    @property
    def n_cons(self) -> int:
        return int(self.row_ptr.size - 1)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def row(self, j):
        a, b = int(self.row_ptr[j]), int(self.row_ptr[j + 1])
        return self.col_var[a:b], self.col_coef[a:b], int(self.rel[j]), int(self.rhs[j])


class RowBuilder:
    """Accumulates families of equal-length rows (2-D var/coef arrays)."""

    def __init__(self):
        self.fams = []

    def add(self, vars2d, coefs2d, rel, rhs):
        v = np.asarray(vars2d, dtype=np.int64)
        c = np.asarray(coefs2d, dtype=np.int64)
        if v.ndim == 1:
            v = v[None, :]
            c = c[None, :]
        if v.shape[0] == 0:
            return
        c = np.broadcast_to(c, v.shape)
        rel = np.broadcast_to(np.asarray(rel, dtype=np.int8), (v.shape[0],))
        rhs = np.broadcast_to(np.asarray(rhs, dtype=np.int64), (v.shape[0],))
        order = np.argsort(v, axis=1, kind="stable")
        v = np.take_along_axis(v, order, axis=1)
        c = np.take_along_axis(c, order, axis=1)
        self.fams.append((v, c, rel.copy(), rhs.copy()))

    def add_row(self, vars_, coefs, rel, rhs):
        self.add(np.asarray(vars_)[None, :], np.asarray(coefs)[None, :], [rel], [rhs])

    def build(self, n_vars, cost, name="") -> Problem:
        lens = [np.full(f[0].shape[0], f[0].shape[1], dtype=np.int64) for f in self.fams]
        lens = np.concatenate(lens) if lens else np.zeros(0, np.int64)
        row_ptr = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=row_ptr[1:])
        col_var = np.concatenate([f[0].ravel() for f in self.fams]) if self.fams else np.zeros(0)
        col_coef = np.concatenate([f[1].ravel() for f in self.fams]) if self.fams else np.zeros(0)
        rel = np.concatenate([f[2] for f in self.fams]) if self.fams else np.zeros(0)
        rhs = np.concatenate([f[3] for f in self.fams]) if self.fams else np.zeros(0)
        p = Problem(int(n_vars), np.ascontiguousarray(cost, dtype=np.float64), row_ptr,
                    col_var.astype(np.int32), col_coef.astype(np.int32), rel.astype(np.int8),
                    rhs.astype(np.int64), name)
        return p


def from_rows(n_vars, cost, rows, name="") -> Problem:
    """rows: iterable of (vars, coefs, rel, rhs); vars need not be sorted."""
    rb = RowBuilder()
    for v, c, r, b in rows:
        rb.add_row(v, c, r, b)
    return rb.build(n_vars, cost, name)


# --------------------------------------------------------------------------
# Paper / SPEC fixed examples


def figure_bdd_problem():
    """The weighted-BDD example of P:303: a+b-c-d = 0 with costs (2,3,1,4)."""
    return from_rows(4, [2.0, 3.0, 1.0, 4.0], [([0, 1, 2, 3], [1, 1, -1, -1], EQ, 0)], "figure")


def spec_two_constraint():
    """{min 2a+3b+c+4d; a+b-c-d=0; b+c>=1}."""
    return from_rows(4, [2.0, 3.0, 1.0, 4.0],
                     [([0, 1, 2, 3], [1, 1, -1, -1], EQ, 0), ([1, 2], [1, 1], GE, 1)], "spec2")


LAP4_LITERAL = np.array([[7, 2, 9, 4], [3, 8, 1, 6], [5, 4, 7, 2], [8, 1, 3, 9]], dtype=np.float64)


def lap(cmat) -> Problem:
    """Linear assignment: x_ab (index a*n+b), one-hot rows and one-hot columns."""
    cmat = np.asarray(cmat, dtype=np.float64)
    n = cmat.shape[0]
    idx = np.arange(n * n).reshape(n, n)
    rb = RowBuilder()
    rb.add(idx, np.ones((n, n)), EQ, 1)        # rows: sum_b x_ab = 1
    rb.add(idx.T.copy(), np.ones((n, n)), EQ, 1)  # columns: sum_a x_ab = 1
    return rb.build(n * n, cmat.ravel(), f"lap{n}")


def lap_random(n, seed) -> Problem:
    """BASELINE configs[0]: c_ab ~ U{0..9}."""
    rng = np.random.default_rng(seed)
    return lap(rng.integers(0, 10, size=(n, n)).astype(np.float64))


# --------------------------------------------------------------------------
# Random tiny ILPs (property tests; SPEC acceptance 1, 3-6)


def random_ilp(seed, n=8, m=4, kmax=5, coef=3, forced_ok=False, max_tries=1000) -> Problem:
    """Random feasible rows with |I_j| <= kmax, coefficients in [-coef, coef]\\{0}.

    Each row is drawn until it admits a satisfying assignment.  Unless
    forced_ok, rows that fix a variable (some x_i takes only one value on the
    row's feasible set) are rejected so all min-marginals are finite.
    """
    rng = np.random.default_rng(seed)
    rows = []
    tries = 0
    while len(rows) < m and tries < max_tries:
        tries += 1
        k = int(rng.integers(1, min(kmax, n) + 1))
        vars_ = np.sort(rng.choice(n, size=k, replace=False))
        a = rng.integers(1, coef + 1, size=k) * rng.choice([-1, 1], size=k)
        rel = int(rng.choice([LE, EQ, GE]))
        # rhs near the middle of the achievable range
        lo, hi = int(np.minimum(a, 0).sum()), int(np.maximum(a, 0).sum())
        b = int(rng.integers(lo, hi + 1))
        xs = ((np.arange(2 ** k)[:, None] >> np.arange(k)[None, :]) & 1)
        s = xs @ a
        ok = (s <= b) if rel == LE else (s >= b) if rel == GE else (s == b)
        if not ok.any():
            continue
        if not forced_ok:
            feas = xs[ok]
            if (feas.min(axis=0) == feas.max(axis=0)).any():
                continue
        rows.append((vars_, a, rel, b))
    cost = rng.uniform(-5, 5, size=n).round(3)
    return from_rows(n, cost, rows, f"rand{seed}")


# --------------------------------------------------------------------------
# Workload look-alikes


def gm_worms_like(seed=0, n_src=500, k_cand=10, knn=30) -> Problem:
    """Graph matching shaped like 'worms' (n_max 1.5M, m_max 0.2M).

    x_{ia}: source i takes candidate label a in {K nearest targets} + dummy.
    Rows: one-hot per source; at-most-one per target over its candidate
    x's; per edge (i,j) and label a: sum_b y_{ia,jb} - x_ia = 0, and per
    label b: sum_a y_{ia,jb} - x_jb = 0.
    """
    rng = np.random.default_rng(seed)
    L = k_cand + 1
    p = rng.uniform(0, 1, size=(n_src, 3))
    perm = rng.permutation(n_src)
    q = (p + rng.normal(0, 0.01, size=p.shape))[perm]
    dpq = np.linalg.norm(p[:, None, :] - q[None, :, :], axis=2)
    cand = np.argsort(dpq, axis=1, kind="stable")[:, :k_cand]          # target ids
    unary = 10.0 * np.take_along_axis(dpq, cand, axis=1) + rng.uniform(0, 1, size=cand.shape)
    xcost = np.concatenate([unary, np.full((n_src, 1), 5.0)], axis=1)  # dummy = 5
    xidx = np.arange(n_src * L).reshape(n_src, L)
    # symmetrised kNN graph of the sources
    dpp = np.linalg.norm(p[:, None, :] - p[None, :, :], axis=2)
    np.fill_diagonal(dpp, np.inf)
    nn = np.argsort(dpp, axis=1, kind="stable")[:, :knn]
    a = np.repeat(np.arange(n_src), knn)
    b = nn.ravel()
    e = np.unique(np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1), axis=0)
    E = e.shape[0]
    ei, ej = e[:, 0], e[:, 1]
    # y_{e, a, b}, index base + e*L*L + a*L + b
    ybase = n_src * L
    yidx = ybase + np.arange(E * L * L).reshape(E, L, L)
    # pairwise cost 10 * | |p_i - p_j| - |q_a - q_b| |, 0 if either label is dummy
    dq = np.linalg.norm(q[:, None, :] - q[None, :, :], axis=2)
    ca = cand[ei]  # [E, K]
    cb = cand[ej]
    qq = dq[ca[:, :, None], cb[:, None, :]]                     # [E, K, K]
    ycost = np.zeros((E, L, L))
    ycost[:, :k_cand, :k_cand] = 10.0 * np.abs(dpp[ei, ej][:, None, None] - qq)
    cost = np.concatenate([xcost.ravel(), ycost.ravel()])
    rb = RowBuilder()
    rb.add(xidx, np.ones((n_src, L)), EQ, 1)                    # one-hot per source
    # at-most-one per target over all x_{ia} with cand[i,a] == t
    order = np.argsort(cand.ravel(), kind="stable")
    tgt_sorted = cand.ravel()[order]
    xs_sorted = xidx[:, :k_cand].ravel()[order]
    bounds = np.flatnonzero(np.diff(tgt_sorted)) + 1
    groups = np.split(xs_sorted, bounds)
    by_len = {}
    for g in groups:
        if g.size >= 2:
            by_len.setdefault(g.size, []).append(np.sort(g))
    for ln, gs in sorted(by_len.items()):
        rb.add(np.stack(gs), np.ones((len(gs), ln)), LE, 1)
    # marginalisation rows
    coefs = np.concatenate([np.ones(L), [-1]])
    for lab in range(L):
        v = np.concatenate([yidx[:, lab, :], xidx[ei, lab][:, None]], axis=1)   # sum_b y_{ia,jb} - x_ia
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
        v = np.concatenate([yidx[:, :, lab], xidx[ej, lab][:, None]], axis=1)   # sum_a y_{ia,jb} - x_jb
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
    return rb.build(ybase + E * L * L, cost, f"gm_worms_like(seed={seed},n={n_src},K={k_cand},knn={knn})")


def mrf_potts(seed=0, H=300, W=400, L=8, conn8=True) -> Problem:
    """Potts MRF shaped like 'color-seg-n8' (local polytope, marginalisation rows)."""
    rng = np.random.default_rng(seed)
    npx = H * W
    xidx = np.arange(npx * L).reshape(npx, L)
    pix = np.arange(npx).reshape(H, W)
    edges = [np.stack([pix[:, :-1].ravel(), pix[:, 1:].ravel()], 1),
             np.stack([pix[:-1, :].ravel(), pix[1:, :].ravel()], 1)]
    if conn8:
        edges += [np.stack([pix[:-1, :-1].ravel(), pix[1:, 1:].ravel()], 1),
                  np.stack([pix[:-1, 1:].ravel(), pix[1:, :-1].ravel()], 1)]
    e = np.concatenate(edges)
    E = e.shape[0]
    unary = rng.uniform(0, 10, size=(npx, L))
    w = rng.uniform(0.5, 2.0, size=E)
    ybase = npx * L
    yidx = ybase + np.arange(E * L * L).reshape(E, L, L)
    ycost = w[:, None, None] * (1.0 - np.eye(L))[None]
    cost = np.concatenate([unary.ravel(), ycost.ravel()])
    rb = RowBuilder()
    rb.add(xidx, np.ones((npx, L)), EQ, 1)
    coefs = np.concatenate([np.ones(L), [-1]])
    ei, ej = e[:, 0], e[:, 1]
    for lab in range(L):
        v = np.concatenate([yidx[:, lab, :], xidx[ei, lab][:, None]], axis=1)
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
        v = np.concatenate([yidx[:, :, lab], xidx[ej, lab][:, None]], axis=1)
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
    return rb.build(ybase + E * L * L, cost, f"mrf_potts(seed={seed},{H}x{W}x{L},{'8' if conn8 else '4'}-conn)")


def mrf_potts_cut(seed=0, H=300, W=400, L=8, conn8=True) -> Problem:
    """Potts MRF in the cut form ('Potts-cut variant'):
    the same grid, unaries and Potts weights as mrf_potts, but one z_e per edge
    (cost w_e) with rows x_il - x_jl - z_e <= 0 and x_jl - x_il - z_e <= 0 for
    every label l, plus the per-pixel simplex.  n = H*W*L + E (1.44 M at full
    size, the paper's n_max 1.4 M for color-seg-n8)."""
    rng = np.random.default_rng(seed)
    npx = H * W
    xidx = np.arange(npx * L).reshape(npx, L)
    pix = np.arange(npx).reshape(H, W)
    edges = [np.stack([pix[:, :-1].ravel(), pix[:, 1:].ravel()], 1),
             np.stack([pix[:-1, :].ravel(), pix[1:, :].ravel()], 1)]
    if conn8:
        edges += [np.stack([pix[:-1, :-1].ravel(), pix[1:, 1:].ravel()], 1),
                  np.stack([pix[:-1, 1:].ravel(), pix[1:, :-1].ravel()], 1)]
    e = np.concatenate(edges)
    E = e.shape[0]
    unary = rng.uniform(0, 10, size=(npx, L))
    w = rng.uniform(0.5, 2.0, size=E)
    zbase = npx * L
    zidx = zbase + np.arange(E)
    cost = np.concatenate([unary.ravel(), w])
    rb = RowBuilder()
    rb.add(xidx, np.ones((npx, L)), EQ, 1)
    ei, ej = e[:, 0], e[:, 1]
    for lab in range(L):
        v = np.stack([xidx[ei, lab], xidx[ej, lab], zidx], axis=1)
        rb.add(v, np.broadcast_to(np.array([1, -1, -1]), v.shape), LE, 0)
        rb.add(v, np.broadcast_to(np.array([-1, 1, -1]), v.shape), LE, 0)
    return rb.build(zbase + E, cost, f"mrf_potts_cut(seed={seed},{H}x{W}x{L},{'8' if conn8 else '4'}-conn)")


def qap(seed=0, n=50) -> Problem:
    """QAPLib-like (tai-a): x_ik plus y_{ik,jl} (i<j, k!=l), assignment + product rows."""
    rng = np.random.default_rng(seed)
    F = rng.integers(0, 100, size=(n, n)); F = np.triu(F, 1); F = F + F.T
    D = rng.integers(0, 100, size=(n, n)); D = np.triu(D, 1); D = D + D.T
    xidx = np.arange(n * n).reshape(n, n)
    I, J = np.triu_indices(n, 1)
    P = I.size
    # y index for pair p, k, l (k != l): base + p*n*(n-1) + k*(n-1) + (l if l<k else l-1)
    ybase = n * n
    kk, ll = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    off = np.where(ll < kk, ll, ll - 1)
    mask = kk != ll
    yid = np.full((P, n, n), -1, dtype=np.int64)
    yid[:, mask] = ybase + np.arange(P * n * (n - 1)).reshape(P, n * (n - 1))
    ycost = (F[I, J][:, None, None] * D[None, :, :] + F[J, I][:, None, None] * D.T[None, :, :])
    ycost = ycost[:, mask].astype(np.float64)  # [P, n*(n-1)] in (k, l) row-major order
    cost = np.concatenate([np.zeros(n * n), ycost.ravel()])
    rb = RowBuilder()
    rb.add(xidx, np.ones((n, n)), EQ, 1)
    rb.add(xidx.T.copy(), np.ones((n, n)), EQ, 1)
    coefs = np.concatenate([np.ones(n - 1), [-1]])
    for k in range(n):
        ls = np.array([l for l in range(n) if l != k])
        v = np.concatenate([yid[:, k, ls], xidx[I, k][:, None]], axis=1)  # sum_{l!=k} y_{ik,jl} - x_ik
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
    for l in range(n):
        ks = np.array([k for k in range(n) if k != l])
        v = np.concatenate([yid[:, ks, l], xidx[J, l][:, None]], axis=1)  # sum_{k!=l} y_{ik,jl} - x_jl
        rb.add(v, np.broadcast_to(coefs, v.shape), EQ, 0)
    return rb.build(ybase + P * n * (n - 1), cost, f"qap(seed={seed},n={n})")


def _grouped_rows(rb, det, var, extra_vars, extra_coefs, rel, rhs):
    """One row per detection: its incident variables (coef 1) plus extra columns."""
    order = np.lexsort((var, det))
    det, var = det[order], var[order]
    nd = extra_vars.shape[0]
    counts = np.bincount(det, minlength=nd)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    for ln in np.unique(counts):
        dets = np.flatnonzero(counts == ln)
        if ln:
            pos = starts[dets][:, None] + np.arange(ln)[None, :]
            inc = var[pos]
        else:
            inc = np.zeros((dets.size, 0), dtype=np.int64)
        v = np.concatenate([inc, extra_vars[dets]], axis=1)
        c = np.concatenate([np.ones((dets.size, ln)), np.broadcast_to(extra_coefs, (dets.size, extra_coefs.size))], axis=1)
        rb.add(v, c, rel, rhs)


def celltrack(seed=0, frames=100, dets=2150, n_trans=5, n_div=3, excl_pairs=None) -> Problem:
    """Cell tracking shaped like 'Cell tracking - large' (detection / conservation / exclusion).

    Per detection d: x_d (cost U[-10,1)), appearance a_d and disappearance e_d
    (U[5,20)); per detection and frame, transitions to its n_trans nearest
    detections of the next frame (cost 5*dist/max + U[0,4)) and divisions into
    pairs of those (U[2,8)).  Rows: incoming sum(in) + a_d - x_d = 0, outgoing
    sum(out) + e_d - x_d = 0, and x_u + x_w <= 1 on random pairs per frame.
    """
    rng = np.random.default_rng(seed)
    if excl_pairs is None:
        excl_pairs = dets // 2
    T, Dn = frames, dets
    pos = rng.uniform(0, 1, size=(T, Dn, 2))
    nd = T * Dn
    did = np.arange(nd).reshape(T, Dn)
    x0, a0, e0 = 0, nd, 2 * nd
    nv = 3 * nd
    cost = [rng.uniform(-10, 1, size=nd), rng.uniform(5, 20, size=nd), rng.uniform(5, 20, size=nd)]
    pairs = [(0, 1), (0, 2), (1, 2)][:n_div]
    in_det, in_var, out_det, out_var = [], [], [], []
    for t in range(T - 1):
        d = np.sqrt(((pos[t][:, None, :] - pos[t + 1][None, :, :]) ** 2).sum(-1))
        sel = np.argpartition(d, n_trans, axis=1)[:, :n_trans]
        sel.sort(axis=1)  # ties in distance are broken by index (deterministic)
        nbr = np.take_along_axis(sel, np.argsort(np.take_along_axis(d, sel, axis=1), axis=1, kind="stable"), axis=1)
        tc = 5.0 * np.take_along_axis(d, nbr, axis=1) / max(d.max(), 1e-9) + rng.uniform(0, 4, size=nbr.shape)
        tv = nv + np.arange(Dn * n_trans).reshape(Dn, n_trans)
        nv += Dn * n_trans
        cost.append(tc.ravel())
        dv = nv + np.arange(Dn * len(pairs)).reshape(Dn, len(pairs))
        nv += Dn * len(pairs)
        cost.append(rng.uniform(2, 8, size=Dn * len(pairs)))
        src = np.repeat(did[t], n_trans)
        out_det.append(src); out_var.append(tv.ravel())
        in_det.append(did[t + 1][nbr].ravel()); in_var.append(tv.ravel())
        out_det.append(np.repeat(did[t], len(pairs))); out_var.append(dv.ravel())
        for q, (u, w) in enumerate(pairs):
            in_det.append(did[t + 1][nbr[:, u]]); in_var.append(dv[:, q])
            in_det.append(did[t + 1][nbr[:, w]]); in_var.append(dv[:, q])
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
    rb = RowBuilder()
    xd = np.arange(nd)
    _grouped_rows(rb, cat(in_det), cat(in_var), np.stack([a0 + xd, x0 + xd], 1), np.array([1, -1]), EQ, 0)
    _grouped_rows(rb, cat(out_det), cat(out_var), np.stack([e0 + xd, x0 + xd], 1), np.array([1, -1]), EQ, 0)
    ex = []
    for t in range(T):
        pr = rng.choice(Dn, size=(excl_pairs, 2))
        pr = pr[pr[:, 0] != pr[:, 1]]
        ex.append(did[t][pr])
    ex = np.concatenate(ex)
    rb.add(ex, np.ones(ex.shape), LE, 1)
    return rb.build(nv, np.concatenate(cost), f"celltrack(seed={seed},{frames}x{dets})")


def gap(seed=0, jobs=300, agents=20, wmax=100, load=0.6) -> Problem:
    """Knapsack-style workload (a single constraint may itself be a
    Knapsack): a generalized assignment problem.  x_ja = 1 if job j goes to
    agent a, cost U[0, 20); every job on exactly one agent (one-hot rows over the
    agents) and every agent within capacity, sum_j w_ja x_ja <= C_a with
    w_ja ~ U{5..wmax} and C_a = load * (jobs / agents) * E[w].  The capacity
    rows have `jobs` variables and partitions of up to C_a + 1 nodes (hundreds
    at the defaults): the wide-BDD case of the sweep."""
    rng = np.random.default_rng(seed)
    x = np.arange(jobs * agents).reshape(jobs, agents)
    w = rng.integers(5, wmax + 1, size=(jobs, agents))
    cap = int(load * jobs / agents * (5 + wmax) / 2)
    cost = rng.uniform(0, 20, size=jobs * agents)
    rb = RowBuilder()
    rb.add(x, np.ones((jobs, agents)), EQ, 1)
    rb.add(x.T.copy(), w.T.copy(), LE, cap)
    return rb.build(jobs * agents, cost, f"gap(seed={seed},{jobs}x{agents},w<={wmax},cap={cap})")


def mckp(seed=0, classes=20_000, items=8, knaps=1200, k=40, wmax=100, frac=0.35) -> Problem:
    """Multiple-choice multi-knapsack (knapsack-style, many wide BDDs): items in
    classes of `items`, exactly one item per class (one-hot rows), and `knaps`
    capacity rows sum_t w_t x_t <= frac * sum_t w_t over k items of k distinct
    random classes, w ~ U{1..wmax}.  Item cost U[-10, 0) (a profit).  Capacity
    rows have partitions of up to ~frac * k * E[w] nodes (hundreds)."""
    rng = np.random.default_rng(seed)
    n = classes * items
    cost = rng.uniform(-10, 0, size=n)
    rb = RowBuilder()
    rb.add(np.arange(n).reshape(classes, items), np.ones((classes, items)), EQ, 1)
    cls = np.stack([rng.choice(classes, size=k, replace=False) for _ in range(knaps)])
    var = cls * items + rng.integers(0, items, size=(knaps, k))
    w = rng.integers(1, wmax + 1, size=(knaps, k))
    cap = np.floor(frac * w.sum(axis=1)).astype(np.int64)
    rb.add(var, w, LE, cap)
    return rb.build(n, cost, f"mckp(seed={seed},{classes}x{items},{knaps}x{k},w<={wmax})")


def thin_hop(seed=0, k=10_000) -> Problem:
    """Thin-hop microbench: one at-most-one row over k variables, c ~ U[-1,1)."""
    rng = np.random.default_rng(seed)
    return from_rows(k, rng.uniform(-1, 1, size=k), [(np.arange(k), np.ones(k), LE, 1)], f"thin_hop({k})")


WORKLOADS = {
    "lap4": lambda seed=0: lap_random(4, seed),
    "gm_worms_like": gm_worms_like,
    "mrf_potts": mrf_potts,
    "mrf_potts_cut": mrf_potts_cut,
    "celltrack": celltrack,
    "qap50": lambda seed=0: qap(seed, 50),
}
