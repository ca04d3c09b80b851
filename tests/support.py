"""Shared test fixtures: numpy restatements of the reference's ground-truth
property oracles (tests/support.hpp:211-337, test_solvers.cpp:60-188,
test_lbfgs.cpp:17-27). They share no code with either the CPU oracle or the
CUDA product, which is what makes them useful as a second opinion.

Flat problems are dicts of numpy arrays (see oracle/oracle.py).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def node_mat(flat, key, i, rows, cols):
    sz = rows * cols
    return flat[key][i * sz:(i + 1) * sz].reshape((rows, cols), order="F")


def node_vec(flat, key, i, n):
    return flat[key][i * n:(i + 1) * n]


def con_F(flat, lay, i):
    nx = flat["nx"]
    m = int(flat["stage_rows"][i])
    off = int(lay["dual_offset"][i])
    return flat["F"][off * nx:(off + m) * nx].reshape((m, nx), order="F")


def con_G(flat, lay, i):
    nu = flat["nu"]
    m = int(flat["stage_rows"][i])
    off = int(lay["dual_offset"][i])
    return flat["G"][off * nu:(off + m) * nu].reshape((m, nu), order="F")


def term_F(flat, lay, l):
    nx = flat["nx"]
    m = int(flat["terminal_rows"][l])
    off = int(lay["tdual_offset"][l]) - lay["stage_total"]
    return flat["FN"][off * nx:(off + m) * nx].reshape((m, nx), order="F")


def dense_H(flat):
    """tests/support.hpp:213-233: H over [all u; all x incl. root]."""
    lay = orc.layout(flat)
    nx, nu, n = flat["nx"], flat["nu"], lay["n"]
    nu_cols = lay["first_leaf"] * nu
    H = np.zeros((lay["dual_dim"], nu_cols + n * nx))
    anc = flat["ancestor"]
    for i in range(1, n):
        a = int(anc[i])
        o = int(lay["dual_offset"][i])
        F, G = con_F(flat, lay, i), con_G(flat, lay, i)
        H[o:o + F.shape[0], nu_cols + a * nx:nu_cols + (a + 1) * nx] = F
        H[o:o + F.shape[0], a * nu:(a + 1) * nu] = G
    for l in range(lay["L"]):
        i = lay["first_leaf"] + l
        o = int(lay["tdual_offset"][l])
        F = term_F(flat, lay, l)
        H[o:o + F.shape[0], nu_cols + i * nx:nu_cols + (i + 1) * nx] = F
    return H


def kkt_dual_grad(flat, y):
    """tests/support.hpp:238-317: dense KKT solve of min <z,H'y> + f(z) s.t. dynamics."""
    lay = orc.layout(flat)
    nx, nu, n = flat["nx"], flat["nu"], lay["n"]
    fl = lay["first_leaf"]
    nu_cols = fl * nu
    dim = nu_cols + (n - 1) * nx
    neq = (n - 1) * nx
    uo = lambda i: i * nu  # noqa: E731
    xo = lambda i: nu_cols + (i - 1) * nx  # noqa: E731
    M = np.zeros((dim, dim))
    lin = np.zeros(dim)
    p = flat["root_state"]
    anc = flat["ancestor"]
    prob = flat["probability"]
    for i in range(1, n):
        a = int(anc[i])
        pi = prob[i]
        Q = node_mat(flat, "Q", i, nx, nx)
        R = node_mat(flat, "R", i, nu, nu)
        S = node_mat(flat, "S", i, nu, nx)
        q = node_vec(flat, "q", i, nx)
        r = node_vec(flat, "r", i, nu)
        M[uo(a):uo(a) + nu, uo(a):uo(a) + nu] += pi * R
        lin[uo(a):uo(a) + nu] += pi * r
        if a == 0:
            lin[uo(a):uo(a) + nu] += 2.0 * pi * (S @ p)
        else:
            M[xo(a):xo(a) + nx, xo(a):xo(a) + nx] += pi * Q
            M[uo(a):uo(a) + nu, xo(a):xo(a) + nx] += pi * S
            M[xo(a):xo(a) + nx, uo(a):uo(a) + nu] += pi * S.T
            lin[xo(a):xo(a) + nx] += pi * q
        F, G = con_F(flat, lay, i), con_G(flat, lay, i)
        o = int(lay["dual_offset"][i])
        yi = y[o:o + F.shape[0]]
        lin[uo(a):uo(a) + nu] += G.T @ yi
        if a != 0:
            lin[xo(a):xo(a) + nx] += F.T @ yi
    for l in range(lay["L"]):
        i = fl + l
        pi = prob[i]
        P = node_mat(flat, "P", l, nx, nx)
        pv = node_vec(flat, "p", l, nx)
        M[xo(i):xo(i) + nx, xo(i):xo(i) + nx] += pi * P
        lin[xo(i):xo(i) + nx] += pi * pv
        F = term_F(flat, lay, l)
        o = int(lay["tdual_offset"][l])
        lin[xo(i):xo(i) + nx] += F.T @ y[o:o + F.shape[0]]
    E = np.zeros((neq, dim))
    rhs = np.zeros(neq)
    for i in range(1, n):
        a = int(anc[i])
        row = (i - 1) * nx
        A = node_mat(flat, "A", i, nx, nx)
        B = node_mat(flat, "B", i, nx, nu)
        c = node_vec(flat, "c", i, nx)
        E[row:row + nx, xo(i):xo(i) + nx] = np.eye(nx)
        E[row:row + nx, uo(a):uo(a) + nu] = -B
        rhs[row:row + nx] = c
        if a == 0:
            rhs[row:row + nx] += A @ p
        else:
            E[row:row + nx, xo(a):xo(a) + nx] = -A
    K = np.zeros((dim + neq, dim + neq))
    K[:dim, :dim] = 2.0 * M
    K[:dim, dim:] = E.T
    K[dim:, :dim] = E
    b = np.concatenate([-lin, rhs])
    sol = np.linalg.solve(K, b)
    x = np.zeros((nx, n))
    u = np.zeros((nu, fl))
    x[:, 0] = p
    for i in range(fl):
        u[:, i] = sol[uo(i):uo(i) + nu]
    for i in range(1, n):
        x[:, i] = sol[xo(i):xo(i) + nx]
    return x.ravel(order="F"), u.ravel(order="F")


def rel_gap(ax, au, bx, bu):
    """test_tree_oracles.cpp:13-19."""
    scale = 1.0 + max(np.abs(ax).max(), np.abs(au).max() if au.size else 0.0)
    gap = max(np.abs(ax - bx).max(), np.abs(au - bu).max() if au.size else 0.0)
    return gap / scale


def dense_dual_hessian(fac: orc.Factor):
    """tests/support.hpp:320-331."""
    prob = fac.prob
    m = prob.dual_dim
    H = np.zeros((m, m))
    for j in range(m):
        e = np.zeros(m)
        e[j] = 1.0
        x, u = fac.hessian_vec(e)
        H[:, j] = -orc.apply_H(prob, x, u)
    return 0.5 * (H + H.T)


def dual_lipschitz_dense(fac: orc.Factor) -> float:
    return float(np.linalg.eigvalsh(dense_dual_hessian(fac)).max())


def dense_bfgs_inverse(pairs, dim, gamma0):
    """test_lbfgs.cpp:17-27."""
    inv = gamma0 * np.eye(dim)
    eye = np.eye(dim)
    for s, q in pairs:
        rho = 1.0 / s.dot(q)
        left = eye - rho * np.outer(s, q)
        inv = left @ inv @ left.T + rho * np.outer(s, s)
    return inv


def reduce_dense(flat):
    """test_solvers.cpp:69-133: dynamics-eliminated dense QP in u."""
    lay = orc.layout(flat)
    nx, nu, n = flat["nx"], flat["nu"], lay["n"]
    udim = lay["first_leaf"] * nu
    anc = flat["ancestor"]
    prob = flat["probability"]
    Xm = [np.zeros((nx, udim)) for _ in range(n)]
    bo = [np.zeros(nx) for _ in range(n)]
    bo[0] = flat["root_state"].copy()
    for i in range(1, n):
        a = int(anc[i])
        A = node_mat(flat, "A", i, nx, nx)
        B = node_mat(flat, "B", i, nx, nu)
        Xm[i] = A @ Xm[a]
        Xm[i][:, a * nu:(a + 1) * nu] += B
        bo[i] = A @ bo[a] + node_vec(flat, "c", i, nx)
    quad = np.zeros((udim, udim))
    lin = np.zeros(udim)
    con = np.zeros((lay["dual_dim"], udim))
    shift = np.zeros(lay["dual_dim"])
    for i in range(1, n):
        a = int(anc[i])
        pi = prob[i]
        X, b = Xm[a], bo[a]
        Q = node_mat(flat, "Q", i, nx, nx)
        R = node_mat(flat, "R", i, nu, nu)
        S = node_mat(flat, "S", i, nu, nx)
        q = node_vec(flat, "q", i, nx)
        r = node_vec(flat, "r", i, nu)
        usel = np.zeros((nu, udim))
        usel[:, a * nu:(a + 1) * nu] = np.eye(nu)
        quad += pi * (X.T @ Q @ X + usel.T @ R @ usel + usel.T @ S @ X + X.T @ S.T @ usel)
        lin += pi * (2.0 * X.T @ (Q @ b) + 2.0 * usel.T @ (S @ b) + X.T @ q + usel.T @ r)
        F, G = con_F(flat, lay, i), con_G(flat, lay, i)
        o = int(lay["dual_offset"][i])
        con[o:o + F.shape[0]] = F @ X + G @ usel
        shift[o:o + F.shape[0]] = F @ b
    for l in range(lay["L"]):
        i = lay["first_leaf"] + l
        pi = prob[i]
        X, b = Xm[i], bo[i]
        P = node_mat(flat, "P", l, nx, nx)
        pv = node_vec(flat, "p", l, nx)
        quad += pi * (X.T @ P @ X)
        lin += pi * (2.0 * X.T @ (P @ b) + X.T @ pv)
        F = term_F(flat, lay, l)
        o = int(lay["tdual_offset"][l])
        con[o:o + F.shape[0]] = F @ X
        shift[o:o + F.shape[0]] = F @ b
    return dict(quad=quad, lin=lin, con=con, shift=shift, X=Xm, b=bo)


def admm_reference(flat, blocks, rho=1.0, iters=60000, tol=1e-11):
    """test_solvers.cpp:138-188 (blocks: list of (offset,size,weight,kind,gamma,zmin,zmax))."""
    red = reduce_dense(flat)
    lay = orc.layout(flat)
    normal = 2.0 * red["quad"] + rho * red["con"].T @ red["con"]
    Linv = np.linalg.inv(normal)
    udim = red["quad"].shape[0]
    u = np.zeros(udim)
    z = red["shift"].copy()
    w = np.zeros(lay["dual_dim"])
    for _ in range(iters):
        u = Linv @ (-red["lin"] - rho * red["con"].T @ (red["shift"] - z + w))
        v = red["con"] @ u + red["shift"]
        target = v + w
        for b in blocks:
            sl = slice(b["offset"], b["offset"] + b["size"])
            if b["kind"] == 1:
                target[sl] = np.minimum(np.maximum(target[sl], b["zmin"]), b["zmax"])
            elif b["kind"] == 2:
                thr = b["weight"] * b["gamma"] / rho
                t = target[sl]
                target[sl] = np.maximum(np.abs(t) - thr, 0.0) * np.where(t > 0, 1.0, -1.0)
        pg = np.abs(v - target).max()
        dg = rho * np.abs(target - z).max()
        z = target
        w += v - z
        if pg < tol and dg < tol:
            break
    nx, nu, n = flat["nx"], flat["nu"], lay["n"]
    x = np.zeros((nx, n))
    for i in range(n):
        x[:, i] = red["X"][i] @ u + red["b"][i]
    return x.ravel(order="F"), u.copy()


def blocks_of(flat):
    """make_nonsmooth (prox.hpp:30-52) as a list of python dicts."""
    lay = orc.layout(flat)
    out = []
    for i in range(1, lay["n"]):
        o = int(lay["dual_offset"][i])
        m = int(flat["stage_rows"][i])
        out.append(dict(offset=o, size=m, weight=float(flat["probability"][i]),
                        kind=int(flat["g_kind"][i]), gamma=float(flat["g_gamma"][i]),
                        zmin=flat["zmin"][o:o + m], zmax=flat["zmax"][o:o + m]))
    for l in range(lay["L"]):
        i = lay["first_leaf"] + l
        o = int(lay["tdual_offset"][l])
        m = int(flat["terminal_rows"][l])
        out.append(dict(offset=o, size=m, weight=float(flat["probability"][i]),
                        kind=int(flat["tg_kind"][l]), gamma=float(flat["tg_gamma"][l]),
                        zmin=flat["zmin"][o:o + m], zmax=flat["zmax"][o:o + m]))
    return out
