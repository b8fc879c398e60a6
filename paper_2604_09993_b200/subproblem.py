"""GPU assembly of the whole SCP convex subproblem.

Replaces `cito.scp.build_subproblem` + `cito.conic.canonicalize`
(/root/reference/pkg/src/cito/scp.py:160-351, conic.py:99-125, 209-269) for the
iteration loop: every row of A (equalities) and G (orthant rows, then SOC
blocks) is laid out once per (scenario, SCP config) as a *superset* CSC pattern
whose entries carry a value recipe -- a constant (computed on the host exactly
as the reference computes it) or `(sign * LIN[src][idx]) * sigma[col]` for the
linearized rows (dynamics, impulse map, impact complementarity Theta, integral
complementarity Psi).  Per iteration the device evaluates the recipes, drops
exact zeros (the reference's `keep = vals != 0` and `eliminate_zeros`) and
compacts to the final CSC (sorted rows, int32 indices), and forms b/h of the
linearized rows; c depends on z_j only.  The pattern therefore moves with the
data exactly as the reference's does (node rows change with Phi, §0.5).

Row order (scp.py:226-337): A = [dynamics (k, r)], per node k [impulse (n_q),
copy (n_q + n_y), Theta-eq (2 n_c)], [x_init (2 n_q), y_init (n_y), masked
x_final, fixed time]; G = per node k [Theta-ineq (4 n_c), impulse boxes (3 per
contact)], per interval [Psi (n_psi), accumulator increments (5 n_c)], control
boxes per (k, side), dilation boxes, slack nonnegativity, then SOC blocks in
add_soc order (node impulse cones inside the node loop, control cones).
"""

import os
import sys
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["SubproblemPattern", "SubproblemAssembler", "LIN_SOURCES", "build_subproblem", "precondition", "GpuSCPStep"]

# value sources (device pointer table order)
LIN_SOURCES = ["jx", "ju", "js", "imp_jac", "theta_jac", "psi_jac", "ends", "imp_v", "theta", "psi"]
SRC = {k: i for i, k in enumerate(LIN_SOURCES)}


class _Rows:
    """Append-only COO with recipes: const entries (src = -1, val = value) or
    linearized entries (src >= 0, idx = flat index, val = sign)."""

    def __init__(self):
        self.row, self.col, self.src, self.idx, self.val = [], [], [], [], []
        self.rhs = []  # constant rhs per row (np.nan where the device computes it)
        self.n = 0

    def add(self, cols, src, idx, val, rhs):
        cols = np.asarray(cols, dtype=np.int64)
        m = cols.size
        self.row.append(np.full(m, self.n, dtype=np.int64))
        self.col.append(cols)
        self.src.append(np.broadcast_to(np.asarray(src, dtype=np.int8), (m,)).copy())
        self.idx.append(np.broadcast_to(np.asarray(idx, dtype=np.int64), (m,)).copy())
        self.val.append(np.broadcast_to(np.asarray(val, dtype=np.float64), (m,)).copy())
        self.rhs.append(rhs)
        self.n += 1
        return self.n - 1

    def arrays(self):
        cat = lambda L, dt: np.concatenate(L).astype(dt) if L else np.zeros(0, dt)
        return (cat(self.row, np.int64), cat(self.col, np.int64), cat(self.src, np.int8), cat(self.idx, np.int64),
                cat(self.val, np.float64), np.asarray(self.rhs, dtype=np.float64))


class SubproblemPattern:
    """Superset CSC + recipes of A and G, constant rhs, P, cones (host, once)."""

    def __init__(self, scenario, lay, scale_v, w_prox=2000.0, w_ep=50000.0):
        sc = scenario
        model = sc.model
        self.lay = lay
        N, n_q, n_c, n_y, n_xt, n_u, n_a = lay.N, lay.n_q, lay.n_c, lay.n_y, lay.n_xt, lay.n_u, lay.n_a
        self.n_psi = n_psi = 3 * n_c + lay.n_g_out
        sigma = np.asarray(scale_v, dtype=float)
        self.sigma = sigma
        self.n_eq_slack = n_eq = (N - 1) * n_xt + N * (n_q + 2 * n_c)
        self.n_in_slack = n_in = (N - 1) * n_psi + N * 4 * n_c
        dim = lay.dim
        self.n = n = dim + 2 * n_eq + n_in
        sp0, sm0, t0 = dim, dim + n_eq, dim + 2 * n_eq
        self.z_idx = np.arange(0, dim)
        self.sp_idx = np.arange(sp0, sp0 + n_eq)
        self.sm_idx = np.arange(sm0, sm0 + n_eq)
        self.t_idx = np.arange(t0, t0 + n_in)
        A, G, S = _Rows(), _Rows(), _Rows()
        lin_rows_A, lin_rows_G = [], []  # (row, form, segments[(src, off, len, cols)], vsrc, voff)
        state = lambda idx: idx  # noqa: E731
        nu2 = 2 * n_u
        eq_s = 0
        in_s = 0
        # -- multiple-shooting defects (scp.py:226-236)
        for k in range(N - 1):
            xp_k, xm_n, u_k, s_k = lay.xp(k), lay.xm(k + 1), lay.u(k), lay.s(k)
            for r in range(n_xt):
                cols = np.concatenate([[xm_n[r]], xp_k, u_k, s_k, [sp0 + eq_s, sm0 + eq_s]])
                src = np.concatenate([[-1], np.full(n_xt, SRC["jx"]), np.full(nu2, SRC["ju"]), [SRC["js"]], [-1, -1]])
                idx = np.concatenate([[0], (k * n_xt + r) * n_xt + np.arange(n_xt),
                                      (k * n_xt + r) * nu2 + np.arange(nu2), [k * n_xt + r], [0, 0]])
                val = np.concatenate([[1.0 * sigma[xm_n[r]]], -np.ones(n_xt + nu2 + 1), [-1.0, 1.0]])
                row = A.add(cols, src, idx, val, np.nan)
                lin_rows_A.append((row, 0, [(SRC["jx"], (k * n_xt + r) * n_xt, n_xt, xp_k),
                                            (SRC["ju"], (k * n_xt + r) * nu2, nu2, u_k),
                                            (SRC["js"], k * n_xt + r, 1, s_k)], SRC["ends"], k * n_xt + r))
                eq_s += 1
        # -- node relations (scp.py:239-282)
        _, imp_hi = _impulse_bounds(sc, lay)
        n_vec = 3 * n_q + 3 * n_c
        n_imp = 3 * n_q + 2 * n_c
        for k in range(N):
            xm_k, xp_k, phi_k, gam_k = lay.xm(k), lay.xp(k), lay.phi(k), lay.gam(k)
            vec_cols = np.concatenate([xm_k[:n_q], xm_k[n_q: 2 * n_q], xp_k[n_q: 2 * n_q], phi_k, gam_k])
            imp_cols = vec_cols[:n_imp]
            for r in range(n_q):  # impulse-map velocity rows
                cols = np.concatenate([imp_cols, [sp0 + eq_s, sm0 + eq_s]])
                src = np.concatenate([np.full(n_imp, SRC["imp_jac"]), [-1, -1]])
                idx = np.concatenate([(k * n_q + r) * n_imp + np.arange(n_imp), [0, 0]])
                val = np.concatenate([np.ones(n_imp), [-1.0, 1.0]])
                row = A.add(cols, src, idx, val, np.nan)
                lin_rows_A.append((row, 1, [(SRC["imp_jac"], (k * n_q + r) * n_imp, n_imp, imp_cols)],
                                   SRC["imp_v"], k * n_q + r))
                eq_s += 1
            for r in list(range(n_q)) + list(range(2 * n_q, n_xt)):  # copy rows
                cols = np.array([xp_k[r], xm_k[r]])
                vals = np.array([1.0, -1.0]) * sigma[cols]
                A.add(cols, -1, 0, vals, 0.0)
            for r in range(2 * n_c):  # Theta equality rows
                cols = np.concatenate([vec_cols, [sp0 + eq_s, sm0 + eq_s]])
                src = np.concatenate([np.full(n_vec, SRC["theta_jac"]), [-1, -1]])
                idx = np.concatenate([(k * 6 * n_c + r) * n_vec + np.arange(n_vec), [0, 0]])
                val = np.concatenate([np.ones(n_vec), [-1.0, 1.0]])
                row = A.add(cols, src, idx, val, np.nan)
                lin_rows_A.append((row, 1, [(SRC["theta_jac"], (k * 6 * n_c + r) * n_vec, n_vec, vec_cols)],
                                   SRC["theta"], k * 6 * n_c + r))
                eq_s += 1
            for r in range(2 * n_c, 6 * n_c):  # Theta inequality rows
                cols = np.concatenate([vec_cols, [t0 + in_s]])
                src = np.concatenate([np.full(n_vec, SRC["theta_jac"]), [-1]])
                idx = np.concatenate([(k * 6 * n_c + r) * n_vec + np.arange(n_vec), [0]])
                val = np.concatenate([np.ones(n_vec), [-1.0]])
                row = G.add(cols, src, idx, val, np.nan)
                lin_rows_G.append((row, 1, [(SRC["theta_jac"], (k * 6 * n_c + r) * n_vec, n_vec, vec_cols)],
                                   SRC["theta"], k * 6 * n_c + r))
                in_s += 1
            for i in range(n_c):  # impulse boxes
                G.add([phi_k[2 * i + 1]], -1, 0, [1.0 * sigma[phi_k[2 * i + 1]]], float(imp_hi[2 * i + 1]))
                G.add([gam_k[i]], -1, 0, [1.0 * sigma[gam_k[i]]], float(imp_hi[2 * n_c + i]))
                G.add([gam_k[i]], -1, 0, [-1.0 * sigma[gam_k[i]]], 0.0)
            for i in range(n_c):  # impulse friction cones (SOC)
                mu = model.contacts[i].friction_mu
                self._soc(S, ((phi_k[2 * i + 1], -mu), (phi_k[2 * i], -1.0)), sigma)
        # -- integral complementarity rows (scp.py:285-301)
        for k in range(N - 1):
            pair_cols = np.concatenate([lay.y_of_xp(k), lay.y_of_xm(k + 1)])
            for r in range(n_psi):
                cols = np.concatenate([pair_cols, [t0 + in_s]])
                src = np.concatenate([np.full(2 * n_y, SRC["psi_jac"]), [-1]])
                idx = np.concatenate([(k * n_psi + r) * 2 * n_y + np.arange(2 * n_y), [0]])
                val = np.concatenate([np.ones(2 * n_y), [-1.0]])
                row = G.add(cols, src, idx, val, np.nan)
                lin_rows_G.append((row, 1, [(SRC["psi_jac"], (k * n_psi + r) * 2 * n_y, 2 * n_y, pair_cols)],
                                   SRC["psi"], k * n_psi + r))
                in_s += 1
            for i in range(5 * n_c):
                margin = 2.0 * sc.ctcs_epsilon if i % 5 == 4 else 0.0
                cols = np.array([pair_cols[n_y + i], pair_cols[i]])
                G.add(cols, -1, 0, np.array([-1.0, 1.0]) * sigma[cols], margin)
        # -- control boxes, cones, dilation boxes (scp.py:304-324)
        lo_u, hi_u = _control_bounds(sc, lay)
        for k in range(N - 1):
            u_k, s_k = lay.u(k), lay.s(k)
            for side in range(2):
                base = side * n_u
                for i in range(n_a):
                    c = u_k[base + i]
                    G.add([c], -1, 0, [1.0 * sigma[c]], float(hi_u[i]))
                    G.add([c], -1, 0, [-1.0 * sigma[c]], float(-lo_u[i]))
                for i in range(n_c):
                    c = u_k[base + n_a + 2 * i + 1]
                    G.add([c], -1, 0, [1.0 * sigma[c]], float(hi_u[n_a + 2 * i + 1]))
                    gi = n_a + 2 * n_c + i
                    c = u_k[base + gi]
                    G.add([c], -1, 0, [1.0 * sigma[c]], float(hi_u[gi]))
                    G.add([c], -1, 0, [-1.0 * sigma[c]], 0.0)
                for i in range(n_c):
                    mu = model.contacts[i].friction_mu
                    fn = u_k[base + n_a + 2 * i + 1]
                    ft = u_k[base + n_a + 2 * i]
                    self._soc(S, ((fn, -mu), (ft, -1.0)), sigma)
            G.add(s_k, -1, 0, [1.0 * sigma[s_k[0]]], float(sc.s_bounds[1]))
            G.add(s_k, -1, 0, [-1.0 * sigma[s_k[0]]], float(-sc.s_bounds[0]))
        # -- boundary conditions (scp.py:327-337)
        x_dim = 2 * n_q
        for r in range(x_dim):
            c = lay.xm(0)[r]
            A.add([c], -1, 0, [1.0 * sigma[c]], float(sc.x_init[r]))
        for r in range(n_y):
            c = lay.y_of_xm(0)[r]
            A.add([c], -1, 0, [1.0 * sigma[c]], 0.0)
        for r in range(x_dim):
            if sc.mask_final[r]:
                c = lay.xp(N - 1)[r]
                A.add([c], -1, 0, [1.0 * sigma[c]], float(sc.x_final[r]))
        if sc.fixed_time:
            cols = np.concatenate([lay.s(k) for k in range(N - 1)])
            A.add(cols, -1, 0, np.ones(N - 1) * sigma[cols], float(sc.t_f))
        # -- slack nonnegativity (scp.py:345-348)
        for idx_set in (self.sp_idx, self.sm_idx, self.t_idx):
            for i in idx_set:
                G.add([i], -1, 0, [-1.0], 0.0)
        if eq_s != n_eq or in_s != n_in:
            raise RuntimeError(f"row count mismatch: eq {eq_s} vs {n_eq}, ineq {in_s} vs {n_in}")
        self.n_orthant = G.n
        # SOC rows follow the orthant rows (conic.py:250-258)
        g_rows = G.arrays()
        s_rows = S.arrays()
        s_rows = (s_rows[0] + G.n,) + s_rows[1:]
        G_all = tuple(np.concatenate([a, b]) for a, b in zip(g_rows, s_rows))
        self.soc_dims = tuple([2] * (S.n // 2))
        self.A = self._csc(A.arrays(), A.n, n)
        self.G = self._csc(G_all, G.n + S.n, n)
        self.lin_rows_A = lin_rows_A
        self.lin_rows_G = lin_rows_G
        # objective (scp.py:340-348 + conic.py:214-232): P diagonal, c
        P_cost, c_cost = _cost_quadratic(sc, lay)
        pdiag = np.zeros(n)
        v1 = P_cost * sigma[:dim] ** 2
        pdiag[:dim] = np.where(v1 != 0.0, v1, 0.0)
        pdiag[:dim] = pdiag[:dim] + 2.0 * w_prox
        self.P_diag = pdiag
        self.c_fixed = np.zeros(n)
        lin0 = sigma[:dim] * (P_cost * 0.0 + c_cost)
        self.c_fixed[:dim] = np.where(lin0 != 0.0, lin0, 0.0)
        for idx_set in (self.sp_idx, self.sm_idx, self.t_idx):
            self.c_fixed[idx_set] += w_ep
        self.w_prox = w_prox

    def sigma_full(self):
        """Per-column scale of the whole variable vector (slacks are unscaled)."""
        return np.concatenate([self.sigma, np.ones(self.n - self.lay.dim)])

    def objective_c(self, z_j):
        """c of the subproblem at iterate z_j (scp.py:341-346, conic.py:227-229).
        Same floating-point operations as ``c[:dim] + (-2 w) * ((z - 0) / sigma)``
        (z - 0.0 is z for every z, -0.0 included), with fewer temporaries."""
        dim = self.lay.dim
        c = self.c_fixed.copy()
        add = np.divide(np.asarray(z_j, dtype=float), self.sigma[:dim])
        add *= -2.0 * self.w_prox
        c[:dim] += add
        return c

    @staticmethod
    def _soc(S, entries, sigma):
        for (c, v) in entries:  # soc_entry: vals * sigma[cols], offset 0 (scp.py:218-221)
            S.add([c], -1, 0, [np.float64(v) * sigma[c]], 0.0)

    def _csc(self, arrs, nrows, ncols):
        row, col, src, idx, val, rhs = arrs
        order = np.lexsort((row, col))
        key = col[order] * (nrows + 1) + row[order]
        if not np.all(np.diff(key) > 0):
            raise RuntimeError("duplicate (row, col) in the superset pattern")
        counts = np.bincount(col, minlength=ncols)
        return dict(indptr=np.concatenate([[0], np.cumsum(counts)]).astype(np.int64), row=row[order].astype(np.int32),
                    col=col[order], src=src[order], idx=idx[order], val=val[order], rhs=rhs, nrows=nrows)


def _impulse_bounds(sc, lay):  # ocp.py:443-457
    n_c = lay.n_c
    lo = np.empty(3 * n_c)
    hi = np.empty(3 * n_c)
    for i in range(n_c):
        mu = sc.model.contacts[i].friction_mu
        lo[2 * i] = -mu * sc.impulse_max
        hi[2 * i] = mu * sc.impulse_max
        lo[2 * i + 1] = 0.0
        hi[2 * i + 1] = sc.impulse_max
    lo[2 * n_c:] = 0.0
    hi[2 * n_c:] = sc.gamma_max
    return lo, hi


def _control_bounds(sc, lay):  # ocp.py:419-441
    model = sc.model
    lo = np.empty(lay.n_u)
    hi = np.empty(lay.n_u)
    for a, j in enumerate(model.actuated_joints):
        lo[a] = model.joints[j].torque_min
        hi[a] = model.joints[j].torque_max
    for i in range(lay.n_c):
        mu = model.contacts[i].friction_mu
        lo[lay.n_a + 2 * i] = -mu * sc.force_max
        hi[lay.n_a + 2 * i] = mu * sc.force_max
        lo[lay.n_a + 2 * i + 1] = 0.0
        hi[lay.n_a + 2 * i + 1] = sc.force_max
    lo[lay.n_a + 2 * lay.n_c:] = 0.0
    hi[lay.n_a + 2 * lay.n_c:] = sc.gamma_max
    return lo, hi


def _cost_quadratic(sc, lay):  # ocp.py:380-390
    P = np.zeros(lay.dim)
    c = np.zeros(lay.dim)
    for k in range(lay.N - 1):
        tq = np.concatenate([lay.u(k)[: lay.n_a], lay.u(k)[lay.n_u: lay.n_u + lay.n_a]])
        P[tq] += sc.torque_weight
        if sc.s_reg:
            P[lay.s(k)] += sc.s_reg
            c[lay.s(k)] += -sc.s_reg * sc.s_nominal
    return P, c


@dataclass
class _Meta:
    """Same interface as cito.scp._SubproblemMeta (scp.py:138-157)."""

    z_idx: np.ndarray
    sp_idx: np.ndarray
    sm_idx: np.ndarray
    t_idx: np.ndarray

    def step_scaled(self, sol, z_j_scaled):
        return sol.x[self.z_idx] - z_j_scaled

    def j_px(self, sol, z_j_scaled):
        d = self.step_scaled(sol, z_j_scaled)
        return float(d @ d)

    def j_ep(self, sol):
        return float(np.sum(sol.x[self.sp_idx]) + np.sum(sol.x[self.sm_idx]) + np.sum(sol.x[self.t_idx]))


@dataclass
class Preconditioner:
    """Same fields as cito.conic.Preconditioner (conic.py:270-277)."""

    row_scale_A: np.ndarray
    row_scale_G: np.ndarray
    var_scale: np.ndarray
    cost_scale: float = 1.0


def _preconditioner_type():
    mod = sys.modules.get("cito.conic")
    return getattr(mod, "Preconditioner", Preconditioner) if mod is not None else Preconditioner


def soc_tables(n_nonneg, soc_dims, device):
    """Device int32 (start row, dim) of every SOC block of G (G rows: orthant, then SOC blocks)."""
    import torch

    dims = np.asarray(soc_dims, dtype=np.int32).reshape(-1)
    start = (n_nonneg + np.concatenate([[0], np.cumsum(dims)[:-1]])).astype(np.int32) if dims.size else dims
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a if a.size else np.zeros(1, np.int32)), device=device)  # noqa
    return t(start), t(dims)


def precondition_device(ncols, out, nA, nG, n_nonneg, n_soc, soc_start, soc_dim, rowmax, max_nnz, stream):
    """Row scaling of a device program in place (cito_precondition_dev); returns
    the device row scales (A, G).  rowmax = (A, G) zeroed int64 workspaces that
    already hold the fused norms, or None (computed here)."""
    import torch

    dev = out["A_data"].device
    ready = rowmax is not None
    if not ready:
        rm = torch.empty(max(1, nA + nG), dtype=torch.int64, device=dev)
        rowmax = (rm[:nA], rm[nA:])
    sA = torch.empty(max(1, nA), dtype=torch.float64, device=dev)
    sG = torch.empty(max(1, nG), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().cito_precondition_dev(
        int(ncols), out["A_indptr"].data_ptr(), out["A_indices"].data_ptr(), out["A_data"].data_ptr(), int(nA),
        out["b"].data_ptr(), out["G_indptr"].data_ptr(), out["G_indices"].data_ptr(), out["G_data"].data_ptr(),
        int(nG), out["h"].data_ptr(), int(n_nonneg), int(n_soc), soc_start.data_ptr(), soc_dim.data_ptr(),
        rowmax[0].data_ptr(), rowmax[1].data_ptr(), int(ready), int(max_nnz), sA.data_ptr(), sG.data_ptr(),
        None, None, None, None, 0, stream),
        "precondition")
    return sA[:nA], sG[:nG]


def precondition(prog):
    """Drop-in for cito.conic.precondition (conic.py:290-338), computed on the GPU.

    A program produced by this package's build_subproblem is scaled where it
    already lives (device copy of the last assembly); any other program is
    uploaded, scaled by the same kernels and copied back.  The sparsity pattern
    does not change, so only the scaled values, b, h and the row scales come
    back (pinned, one synchronization).  Returns (scaled ConicProgram,
    Preconditioner) with the reference's types when cito.conic is loaded; A/G
    values and row scales are bit-identical to the reference's, b/h scale the
    GPU's own b/h by the same factors."""
    import scipy.sparse as sp
    import torch

    ConicProgram, ConeSpec = _conic_types()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    cones = prog.cones
    n = int(prog.A.shape[1])
    nA, nG = int(prog.A.shape[0]), int(prog.G.shape[0])
    A = sp.csc_matrix(prog.A)
    G = sp.csc_matrix(prog.G)
    A.sort_indices()
    G.sort_indices()
    own = None
    for asm in _assemblers.values():
        last = getattr(asm, "last", None)
        if last is not None and last[0] is prog:
            own = last[1]
            break
    if own is not None:  # device copy of exactly these values (to_program copied it out unchanged)
        out = {k: own[k] for k in ("A_indptr", "A_indices", "G_indptr", "G_indices")}
        out.update({k: own[k].clone() for k in ("A_data", "b", "G_data", "h")})
    else:
        i32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32) if a.size else np.zeros(1, np.int32),  # noqa
                                        device=dev)
        f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).reshape(-1) if np.size(a)  # noqa
                                        else np.zeros(1), device=dev)
        out = {"A_indptr": i32(A.indptr), "A_indices": i32(A.indices), "A_data": f64(A.data),
               "G_indptr": i32(G.indptr), "G_indices": i32(G.indices), "G_data": f64(G.data),
               "b": f64(prog.b), "h": f64(prog.h)}
    start, dim = soc_tables(int(cones.nonneg), tuple(cones.soc), dev)
    sA, sG = precondition_device(n, out, nA, nG, int(cones.nonneg), len(cones.soc), start, dim, None,
                                 max(A.nnz, G.nnz), stream.cuda_stream)
    # values come back into fresh pinned buffers: nnz prefixes only (pattern unchanged)
    back = {"A": out["A_data"][: A.nnz], "G": out["G_data"][: G.nnz], "b": out["b"][:nA], "h": out["h"][:nG],
            "sA": sA, "sG": sG}
    pin = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in back.items()}
    for k, v in back.items():
        pin[k].copy_(v, non_blocking=True)
    stream.synchronize()
    h = {k: v.numpy() for k, v in pin.items()}
    mats = {"A": sp.csc_matrix((h["A"], A.indices.copy(), A.indptr.copy()), shape=A.shape),
            "G": sp.csc_matrix((h["G"], G.indices.copy(), G.indptr.copy()), shape=G.shape)}
    omega = max(1.0, float(np.max(np.abs(prog.c))) if prog.c.size else 0.0)
    if prog.P.nnz:
        omega = max(omega, float(np.max(np.abs(prog.P.data))))
    P = sp.csc_matrix(prog.P / omega)
    P.sort_indices()
    scaled = ConicProgram(P=P, c=prog.c / omega, A=mats["A"], b=h["b"], G=mats["G"], h=h["h"], cones=cones)
    prec = _preconditioner_type()(row_scale_A=h["sA"], row_scale_G=h["sG"], var_scale=np.ones(n), cost_scale=omega)
    return scaled, prec


@dataclass(frozen=True)
class ConeSpec:
    """Same fields as cito.conic.ConeSpec (conic.py:37-51)."""

    nonneg: int = 0
    soc: tuple = ()


@dataclass
class ConicProgram:
    """Same fields as cito.conic.ConicProgram (conic.py:54-84)."""

    P: object
    c: np.ndarray
    A: object
    b: np.ndarray
    G: object
    h: np.ndarray
    cones: ConeSpec


_CSC_FAST = None  # None: not probed yet; else (maxprint,) when the direct construction is valid
_CSC_CHECK = os.environ.get("CITO_CHECK_CSC", "0") == "1"
_CSC_RECIPES = os.environ.get("CITO_CSC_RECIPES", "0") == "1"  # A/B switch: warp-per-column compaction
# A/B switch CITO_Z_HOST=1: z read straight from the pinned buffer by K1 / K3 / the
# compaction (no H2D node before K1): -6 us on one box of the pool, +17 us on another
# (host-memory read latency differs between boxes), so the default copies z first
_Z_HOST = os.environ.get("CITO_Z_HOST", "0") == "1"
_SKIP_CONSTS = os.environ.get("CITO_SKIP_CONSTS", "1") == "1"  # A/B: constant CSC entries not re-sent
_Z_UPLOAD_KERNEL = os.environ.get("CITO_Z_UPLOAD", "kernel") != "dma"  # A/B: "dma" = copy-engine H2D


def packed_entries(csc, sigma):
    """16-byte records {w, key, row} of a superset CSC for k_csc_flat (include/cito_b200.h,
    cito_csc_assemble_packed_dev) and the first column owned by each 2048-entry tile."""
    src = csc["src"].astype(np.int64)
    idx = np.asarray(csc["idx"], dtype=np.int64)
    val = np.asarray(csc["val"], dtype=np.float64)
    col = np.asarray(csc["col"], dtype=np.int64)
    lin = src >= 0
    if np.any(np.abs(val[lin]) != 1.0):
        raise RuntimeError("packed CSC records need sign-only recipes for the linearized entries")
    if idx.size and (idx.max() >= (1 << 27) or idx.min() < 0):
        raise RuntimeError("lin index outside the 27-bit key range")
    rec = np.zeros(src.size, dtype=np.dtype([("w", "<f8"), ("key", "<u4"), ("row", "<i4")]))
    rec["w"] = np.where(lin, val * sigma[col], val)
    rec["key"] = (((src + 1) << 27) | np.where(lin, idx, 0)).astype(np.uint32)
    rec["row"] = csc["row"]
    ntile = max(1, -(-src.size // 2048))
    tcol = np.searchsorted(csc["indptr"], np.arange(ntile, dtype=np.int64) * 2048, side="left")
    return rec, np.concatenate([tcol, [len(csc["indptr"])]]).astype(np.int32)


def _csc_direct(data, indices, indptr, shape, check=True):
    """scipy.sparse.csc_matrix over arrays already in canonical form (int32 indices,
    float64 data, len == nnz; sorted, no duplicates -- the device compaction's
    output), without the constructor's per-call dtype/format checks (~20 us per
    matrix).  Probed once against the regular constructor: if this scipy's matrix
    carries attributes the direct form does not set, the regular one is used.
    Every call keeps the O(1) invariants (int32/float64 dtypes, indptr[0] == 0,
    indptr[-1] == nnz, len(indptr) == ncols + 1; check=False leaves the two that
    read indptr's contents to the caller, for a matrix built before the device
    result arrived); CITO_CHECK_CSC=1 adds scipy's full format check (sorted,
    in-range indices) for debugging."""
    global _CSC_FAST
    import scipy.sparse as sp

    if (indices.dtype != np.int32 or indptr.dtype != np.int32 or data.dtype != np.float64
            or len(indptr) != shape[1] + 1 or len(data) != len(indices)
            or (check and (indptr[0] != 0 or indptr[-1] != len(indices)))):
        raise RuntimeError("device CSC compaction returned an inconsistent matrix "
                           f"(indptr[0]={indptr[0]}, indptr[-1]={indptr[-1]}, nnz={len(indices)})")
    if _CSC_CHECK:
        m = sp.csc_matrix((data, indices, indptr), shape=shape, copy=False)
        m.check_format(full_check=True)
        return m
    if _CSC_FAST is None:
        ref = sp.csc_matrix((data, indices, indptr), shape=shape, copy=False)
        keys = set(vars(ref))
        _CSC_FAST = (ref.maxprint,) if keys == {"_shape", "maxprint", "indices", "indptr", "data"} else False
        return ref
    if _CSC_FAST is False:
        return sp.csc_matrix((data, indices, indptr), shape=shape, copy=False)
    m = sp.csc_matrix.__new__(sp.csc_matrix)
    m._shape = (int(shape[0]), int(shape[1]))
    m.maxprint = _CSC_FAST[0]
    m.indices = indices
    m.indptr = indptr
    m.data = data
    return m


def _conic_types():
    """The reference's own program types when cito.conic is loaded (so its IPM and
    validate() accept the result), else the local mirrors."""
    mod = sys.modules.get("cito.conic")
    if mod is not None and hasattr(mod, "ConicProgram"):
        return mod.ConicProgram, mod.ConeSpec
    return ConicProgram, ConeSpec


class SubproblemAssembler:
    """Device-side assembly of the whole subproblem from a device linearization."""

    def __init__(self, pattern, device):
        import torch

        self.pat = pattern
        self.device = device
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=device)  # noqa: E731
        self.sigma_dev = t(pattern.sigma_full(), np.float64)
        self._mats = {}
        for M, rows in (("A", pattern.lin_rows_A), ("G", pattern.lin_rows_G)):
            csc = getattr(pattern, M)
            d = dict(sp_ptr=t(csc["indptr"], np.int64), row=t(csc["row"], np.int32), src=t(csc["src"], np.int8),
                     idx=t(csc["idx"], np.int64), val=t(csc["val"], np.float64), nrows=csc["nrows"],
                     nsup=int(csc["row"].size), rhs_const=t(np.nan_to_num(csc["rhs"]), np.float64))
            # block totals / per-column counts; the one-pass compaction keeps tagged block
            # totals and its launch epoch here across calls, so it starts zeroed
            d["counts"] = torch.zeros(pattern.n + 64, dtype=torch.int32, device=device)
            # packed 16-byte records of the entry-parallel compaction (k_csc_flat)
            rec, tcol = packed_entries(csc, pattern.sigma_full())
            d.update(ent=t(rec.view(np.uint8), np.uint8), tcol=t(tcol, np.int32), ntile=len(tcol) - 1)
            # rhs descriptors of the linearized rows
            nr = len(rows)
            r_row = np.array([r[0] for r in rows], dtype=np.int32)
            r_form = np.array([r[1] for r in rows], dtype=np.int8)
            r_vsrc = np.array([r[3] for r in rows], dtype=np.int8)
            r_voff = np.array([r[4] for r in rows], dtype=np.int64)
            seg_src = np.full((nr, 3), -1, dtype=np.int8)
            seg_off = np.zeros((nr, 3), dtype=np.int64)
            seg_len = np.zeros((nr, 3), dtype=np.int32)
            seg_cb = np.zeros((nr, 3), dtype=np.int64)
            cols, cache = [], {}
            total = 0
            for i, (_, _, segs, _, _) in enumerate(rows):
                for j, (s, off, ln, cz) in enumerate(segs):
                    key = (int(cz[0]), int(len(cz)))
                    if key not in cache:
                        cache[key] = total
                        cols.append(np.asarray(cz, dtype=np.int64))
                        total += len(cz)
                    seg_src[i, j], seg_off[i, j], seg_len[i, j], seg_cb[i, j] = s, off, ln, cache[key]
            d.update(nlin=nr, r_row=t(r_row, np.int32), r_form=t(r_form, np.int8), r_vsrc=t(r_vsrc, np.int8),
                     r_voff=t(r_voff, np.int64), seg_src=t(seg_src, np.int8), seg_off=t(seg_off, np.int64),
                     seg_len=t(seg_len, np.int32), seg_cb=t(seg_cb, np.int64),
                     cols=t(np.concatenate(cols) if cols else np.zeros(1), np.int64))
            self._mats[M] = d

    def packed_args(self, lin_ptrs, outs, rowmax, arr, stamp=None, mirror=None):
        """Argument tuple of cito_csc_assemble_packed_dev for A and G (without the
        stream); `outs` = [(indptr, indices, data)] per matrix, `arr` builds a
        ctypes pointer table from tensors, `stamp` = optional (stamp_in, changed_at)
        device pointers of the pattern-change stamp, `mirror` = optional
        (host_vals, host_rows, rows_wanted, consts_wanted) of the host mirror."""
        import ctypes

        import torch

        mats = [self._mats["A"], self._mats["G"]]
        if getattr(self, "_ws", None) is None:
            tiles = sum(d["ntile"] for d in mats)
            self._ws = torch.zeros(4 + 2 * tiles, dtype=torch.int32, device=self.device)
            self._nsup = (ctypes.c_int64 * 2)(*[d["nsup"] for d in mats])
            self._ntile = (ctypes.c_int32 * 2)(*[d["ntile"] for d in mats])
        return (2, self.pat.n, arr([d["ent"] for d in mats]), ctypes.cast(self._nsup, ctypes.c_void_p),
                arr([d["sp_ptr"] for d in mats]), arr([d["tcol"] for d in mats]),
                ctypes.cast(self._ntile, ctypes.c_void_p), lin_ptrs, self._ws.data_ptr(), self._ws.numel(),
                arr([o[0] for o in outs]), arr([o[1] for o in outs]), arr([o[2] for o in outs]),
                arr(rowmax) if rowmax else None, *(stamp or (None, None)), *(mirror or (0, 0, None, None)))

    def _prepare_batched(self):
        """Concatenate the rhs descriptors of A and G (one launch) and allocate
        the per-iteration outputs once."""
        import torch

        dA, dG = self._mats["A"], self._mats["G"]
        nA = dA["nrows"]
        cat = lambda k: torch.cat([dA[k], dG[k]])  # noqa: E731
        self._rhs = dict(rows=torch.cat([dA["r_row"], dG["r_row"] + nA]), form=cat("r_form"), vsrc=cat("r_vsrc"),
                         voff=cat("r_voff"), seg_src=cat("seg_src"), seg_off=cat("seg_off"), seg_len=cat("seg_len"),
                         seg_cb=torch.cat([dA["seg_cb"], dG["seg_cb"] + dA["cols"].numel()]),
                         cols=torch.cat([dA["cols"], dG["cols"]]), const=torch.cat([dA["rhs_const"], dG["rhs_const"]]),
                         n=dA["nlin"] + dG["nlin"], nA=nA)

    def assemble_device(self, lin, z_ref_dev, stream=None, precondition=False, reuse=False):
        """lin: dict of device tensors with the LIN_SOURCES fields.  Returns device
        tensors {A_indptr, A_indices, A_data, b, G_indptr, G_indices, G_data, h}
        (data/indices sized to the superset; valid prefix = indptr[-1]).
        ``reuse``: write into buffers owned by the assembler (no allocation per
        call; the previous call's result is overwritten) -- for iteration loops.
        Four kernel launches: count (A and G), scan, write, rhs.  With
        ``precondition`` the program is returned already row-scaled as
        cito.conic.precondition does (conic.py:290-338): the row inf-norms are
        fused into the CSC write and two more launches form and apply the row
        scales (+ ``row_scale_A`` / ``row_scale_G`` in the result)."""
        import torch

        if getattr(self, "_rhs", None) is None:
            self._prepare_batched()
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        if reuse:  # stable pointers: memoize the ctypes pointer tables (host launch overhead)
            memo = self.__dict__.setdefault("_ptr_memo", {})

            def arr(xs):
                key = tuple(x.data_ptr() for x in xs)
                a = memo.get(key)
                if a is None:
                    if len(memo) > 64:
                        memo.clear()
                    a = memo[key] = ctypes_ptr_array(list(key))
                return a
        else:
            arr = lambda xs: ctypes_ptr_array([x.data_ptr() if x is not None else None for x in xs])  # noqa: E731
        ptrs = arr([lin[k] for k in LIN_SOURCES])
        out = {}
        mats = [self._mats["A"], self._mats["G"]]
        outs = []
        owned = getattr(self, "_owned", None) if reuse else None
        if reuse and owned is None:
            owned = self._owned = {}
        for M, d in zip(("A", "G"), mats):
            if owned is not None and M in owned:
                indptr, rows, vals = owned[M]
            else:
                indptr = torch.empty(self.pat.n + 1, dtype=torch.int32, device=self.device)
                rows = torch.empty(max(1, d["nsup"]), dtype=torch.int32, device=self.device)
                vals = torch.empty(max(1, d["nsup"]), dtype=torch.float64, device=self.device)
                if owned is not None:
                    owned[M] = (indptr, rows, vals)
            out[f"{M}_indptr"], out[f"{M}_indices"], out[f"{M}_data"] = indptr, rows, vals
            outs.append((indptr, rows, vals))
        rowmax = None
        if precondition:
            nA, nG = mats[0]["nrows"], mats[1]["nrows"]
            rm = torch.zeros(max(1, nA + nG), dtype=torch.int64, device=self.device)
            rowmax = (rm[:nA], rm[nA:])
        # b/h of the linearized rows on a side stream, concurrently with the CSC compaction
        r = self._rhs
        cur = torch.cuda.current_stream(self.device) if stream is None else torch.cuda.ExternalStream(stream)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        side = self._side
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            if owned is not None:
                if "rhs" not in owned:
                    owned["rhs"] = torch.empty_like(r["const"])
                rhs = owned["rhs"]
                rhs.copy_(r["const"])
            else:
                rhs = r["const"].clone()
            _lib.check(_lib.lib().cito_rhs_dev(
                r["n"], r["rows"].data_ptr(), r["form"].data_ptr(), r["vsrc"].data_ptr(), r["voff"].data_ptr(),
                r["seg_src"].data_ptr(), r["seg_off"].data_ptr(), r["seg_len"].data_ptr(), r["seg_cb"].data_ptr(),
                r["cols"].data_ptr(), z_ref_dev.data_ptr(), ptrs, rhs.data_ptr(), 0, side.cuda_stream), "rhs")
        if _CSC_RECIPES:  # A/B: the warp-per-column recipe-table form
            _lib.check(_lib.lib().cito_csc_assemble2_dev(
                2, self.pat.n, arr([d["sp_ptr"] for d in mats]), arr([d["row"] for d in mats]),
                arr([d["src"] for d in mats]), arr([d["idx"] for d in mats]), arr([d["val"] for d in mats]),
                self.sigma_dev.data_ptr(), ptrs, arr([d["counts"] for d in mats]), arr([o[0] for o in outs]),
                arr([o[1] for o in outs]), arr([o[2] for o in outs]), arr(rowmax) if rowmax else None, s),
                "csc_assemble")
        else:
            _lib.check(_lib.lib().cito_csc_assemble_packed_dev(*self.packed_args(ptrs, outs, rowmax, arr), s),
                       "csc_assemble")
        cur.wait_stream(side)
        if owned is None:
            rhs.record_stream(cur)
        out["b"], out["h"] = rhs[: r["nA"]], rhs[r["nA"]:]
        if precondition:
            self._precondition(out, rowmax, s)
        return out

    def _soc_tables(self):
        if getattr(self, "_soc_dev", None) is None:
            self._soc_dev = soc_tables(self.pat.n_orthant, self.pat.soc_dims, self.device)
        return self._soc_dev

    def _precondition(self, out, rowmax, stream):
        start, dim = self._soc_tables()
        out["row_scale_A"], out["row_scale_G"] = precondition_device(
            self.pat.n, out, self._mats["A"]["nrows"], self._mats["G"]["nrows"], self.pat.n_orthant,
            len(self.pat.soc_dims), start, dim, rowmax, max(self._mats["A"]["nsup"], self._mats["G"]["nsup"]),
            stream)

    def to_program(self, dev_out, z_j):
        """Host ConicProgram (scipy CSC, the reference's types when loaded) + meta.
        One batched device->host copy into pinned staging, one synchronization.
        For a preconditioned ``dev_out`` returns (scaled program, Preconditioner, meta)."""
        import scipy.sparse as sp
        import torch

        ConicProgram, ConeSpec = _conic_types()
        pat = self.pat
        keys = ["A_indptr", "A_indices", "A_data", "b", "G_indptr", "G_indices", "G_data", "h"]
        scaled = "row_scale_A" in dev_out
        if scaled:
            keys = keys + ["row_scale_A", "row_scale_G"]
        if getattr(self, "_pinned", None) is None:
            self._pinned = {}
        for k in keys:
            if k not in self._pinned:
                self._pinned[k] = torch.empty(dev_out[k].shape, dtype=dev_out[k].dtype, pin_memory=True)
            self._pinned[k].copy_(dev_out[k], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        host = {k: self._pinned[k].numpy() for k in keys}
        mats = {}
        for M in ("A", "G"):
            indptr = host[f"{M}_indptr"].copy()
            nnz = int(indptr[-1])
            mats[M] = sp.csc_matrix((host[f"{M}_data"][:nnz].copy(), host[f"{M}_indices"][:nnz].copy(), indptr),
                                    shape=(self._mats[M]["nrows"], pat.n))
        dim = pat.lay.dim
        P_data = pat.P_diag[:dim]
        c = pat.objective_c(z_j)
        omega = 1.0
        if scaled:  # cost normalization (conic.py:311-316): host scalars
            omega = max(1.0, float(np.max(np.abs(c))) if c.size else 0.0)
            if P_data.size:
                omega = max(omega, float(np.max(np.abs(P_data))))
            P_data, c = P_data * (1.0 / omega), c / omega  # scipy's P / omega is P * (1 / omega)
        P = sp.csc_matrix((P_data, np.arange(dim, dtype=np.int32),
                           np.concatenate([np.arange(dim + 1), np.full(pat.n - dim, dim)]).astype(np.int32)),
                          shape=(pat.n, pat.n))
        prog = ConicProgram(P=P, c=c, A=mats["A"], b=host["b"].copy(), G=mats["G"],
                            h=host["h"].copy(), cones=ConeSpec(nonneg=pat.n_orthant, soc=pat.soc_dims))
        meta = _Meta(pat.z_idx, pat.sp_idx, pat.sm_idx, pat.t_idx)
        if scaled:
            prec = _preconditioner_type()(row_scale_A=host["row_scale_A"].copy(),
                                          row_scale_G=host["row_scale_G"].copy(), var_scale=np.ones(pat.n),
                                          cost_scale=omega)
            return prog, prec, meta
        self.last = (prog, dev_out)  # the precondition drop-in reuses the device copy
        return prog, meta


_LAZY_TYPES = {}


def _lazy_program_type(base):
    """A subclass of the (reference's) ConicProgram dataclass whose A, b, G, h are
    read from GpuSCPStep's device copy of the unscaled values on first access."""
    t = _LAZY_TYPES.get(base)
    if t is not None:
        return t

    def _field(name):
        def get(self):
            self._materialize()
            return self._host[name]

        def set_(self, v):
            self._materialize()
            self._host[name] = v

        return property(get, set_)

    class LazyProgram(base):
        @classmethod
        def _new(cls, step, hb, mats, nA, nG, P, c, cones):
            o = object.__new__(cls)
            o.__dict__.update(P=P, c=c, cones=cones, _step=step, _hb=hb, _mats=mats, _nA=nA, _nG=nG, _host=None)
            return o

        def _materialize(self):
            if self._host is not None:
                return
            import scipy.sparse as sp
            import torch

            u = self._hb.slot["unscaled"]
            h = {}
            o = 0
            for M in ("A", "G"):  # concatenated values: G's follow A's nonzeros
                ref = self._mats[M]
                nnz = ref.indices.size
                vals = u["vals"][o: o + nnz].cpu().numpy()
                o += nnz
                h[M] = sp.csc_matrix((vals, ref.indices.copy(), ref.indptr.copy()), shape=ref.shape)
            rhs = u["rhs"][: self._nA + self._nG].cpu().numpy()
            torch.cuda.current_stream(self._step.gt.device).synchronize()
            h["b"], h["h"] = rhs[: self._nA].copy(), rhs[self._nA:].copy()
            self._host = h

    for name in ("A", "b", "G", "h"):
        setattr(LazyProgram, name, _field(name))
    LazyProgram.__name__ = base.__name__
    _LAZY_TYPES[base] = LazyProgram
    return LazyProgram


def ctypes_ptr_array(ptrs):
    import ctypes

    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    return ctypes.cast(arr, ctypes.c_void_p)


_assemblers = {}


def build_subproblem(tr, lin, z_j, delta, config):
    """Drop-in for cito.scp.build_subproblem (scp.py:160-351): values assembled on
    the GPU from a host LinearizedProblem; returns (ConicProgram, meta)."""
    import torch

    from .scenario import build_scaling

    key = (id(tr), float(config.w_prox), float(config.w_ep))
    asm = _assemblers.get(key)
    if asm is None or getattr(asm, "owner", None) is not tr:  # the strong ref keeps id(tr) from being reused
        dev = torch.device("cuda", torch.cuda.current_device())
        scale_v = tr.scaling.scale if hasattr(tr, "scaling") else build_scaling(tr.scenario, tr.layout)[0]
        pat = SubproblemPattern(tr.scenario, tr.layout, scale_v, config.w_prox, config.w_ep)
        asm = SubproblemAssembler(pat, dev)
        asm.owner = tr
        _assemblers[key] = asm
    dev = asm.device
    from .linearize import _cache

    cached = _cache.get(id(tr))
    last = getattr(cached[1], "last", None) if cached and cached[0] is tr else None
    if hasattr(lin, "device_arrays") and lin.device_arrays() is not None:  # ours, buffers still current
        lin_dev = lin.device_arrays()
        z_ref = torch.as_tensor(np.ascontiguousarray(lin.z_ref, dtype=np.float64), device=dev)
    elif last is not None and last[0] is lin:
        lin_dev, z_ref = last[1], last[2]
    else:
        lin_dev = {k: torch.as_tensor(np.ascontiguousarray(getattr(lin, k), dtype=np.float64), device=dev)
                   for k in LIN_SOURCES}
        z_ref = torch.as_tensor(np.ascontiguousarray(lin.z_ref, dtype=np.float64), device=dev)
    out = asm.assemble_device(lin_dev, z_ref)
    return asm.to_program(out, z_j)


class _Packed:
    """One device buffer holding every per-iteration output of GpuSCPStep at fixed
    offsets, so the whole result comes back with a single device->host copy and
    every kernel argument is a constant pointer."""

    def __init__(self, fields, device):
        import torch

        off, self.layout = 0, {}
        for name, dtype, n in fields:
            isz = torch.empty((), dtype=dtype).element_size()
            off = (off + 255) // 256 * 256
            self.layout[name] = (off, dtype, int(n), isz)
            off += max(1, int(n)) * isz
        self.nbytes = (off + 255) // 256 * 256
        self.dev = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.d = {}
        for name, (o, dtype, n, isz) in self.layout.items():
            self.d[name] = self.dev[o: o + max(1, n) * isz].view(dtype)[:n]


class _Span:
    """Owner object of one handed-out array over pinned memory (numpy
    __array_interface__): the array's base, with `size` equal to the array's
    length so scipy's _prune_array never copies it, and weakly referenceable so
    the buffer knows when the caller has dropped the array.  It holds the pinned
    allocation itself, so an array outlives the GpuSCPStep that produced it."""

    def __init__(self, ptr, n, dtype, owner):
        self.owner = owner
        self.size = int(n)
        self.__array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": dtype.str,
                                    "version": 3}


class _HostBuf:
    """A pinned host mirror of a _Packed buffer whose arrays are handed out
    without copying.  It is free again once every array handed out from it has
    been dropped (weak references to their _Span owners)."""

    def __init__(self, pk):
        import torch

        self.host = torch.zeros(pk.nbytes, dtype=torch.uint8, pin_memory=True)
        self.nb = self.host.numpy()
        self.h, self.np_dtype, self.off = {}, {}, {}
        for name, (o, dtype, n, isz) in pk.layout.items():
            npdt = torch.empty((), dtype=dtype).numpy().dtype
            self.h[name] = self.nb[o: o + max(1, n) * isz].view(npdt)[:n]
            self.np_dtype[name], self.off[name] = (npdt, isz), o
        self.base_ptr = self.nb.ctypes.data
        self.graphs = {}
        self.live = []
        self.pat_gen = -1  # pattern generation of the CSC indices last copied into this buffer
        self.rhs_scaled = False  # b/h here were row-scaled by a preconditioned call (constant rows too)
        self.consts_ok = False  # the constant CSC entries here are current (unscaled, hb's pattern)

    def wrap(self, name, start, n):
        """Array of n elements of field `name` from element `start`, owned by a _Span."""
        import weakref

        npdt, isz = self.np_dtype[name]
        span = _Span(self.base_ptr + self.off[name] + start * isz, n, npdt, self.host)
        self.live.append(weakref.ref(span))
        return np.asarray(span)

    def free(self):
        self.live = [r for r in self.live if r() is not None]
        return not self.live


class GpuSCPStep:
    """One SCP iteration's pre-IPM work in a single device pass (public API).

    ``iterate(z, delta, z_j=None)`` = cito.scp.linearize_all + build_subproblem
    (scp.py:412-413) with host numpy in / host scipy out: one upload of z from pinned memory,
    the interval + node kernels, the whole-subproblem assembly (+ preconditioning,
    scp.py:414) whose last kernel stores the CSC values straight into a pinned
    host buffer (the fixed fields follow in one copy kernel), and a single
    synchronization.  All device buffers and kernel argument tables are built
    once; the host work per call is the C-ABI launches and the scipy wrappers.
    Raises FloatingPointError for non-finite interval end states like the
    reference (augmentation.py:231-233).
    Returns (LinearizedProblem (lazy, device-backed), ConicProgram, meta)."""

    def __init__(self, tr_or_scenario, w_prox=2000.0, w_ep=50000.0, device=None, use_graph=True):
        from .linearize import GpuTranscription, LazyLinearizedProblem
        from .scenario import build_scaling

        self.gt = tr_or_scenario if isinstance(tr_or_scenario, GpuTranscription) else GpuTranscription(
            tr_or_scenario, device=device)
        gt = self.gt
        scale_v = build_scaling(gt.scenario, gt.lay)[0]
        self.asm = SubproblemAssembler(SubproblemPattern(gt.scenario, gt.lay, scale_v, w_prox, w_ep), gt.device)
        self._Lazy = LazyLinearizedProblem
        self._plan = None
        self._last_lin = None
        self.use_graph = use_graph
        self.pattern_refetches = 0  # calls whose pattern moved after a values-only copy
        self.d2h_copied = 0  # bytes of every device->host copy the calls made

    # -- one-time plan: buffers + constant ctypes argument tables
    def _build_plan(self):
        import torch

        gt, asm, pat = self.gt, self.asm, self.asm.pat
        if getattr(asm, "_rhs", None) is None:
            asm._prepare_batched()
        lay, dev = gt.lay, gt.device
        NI = lay.N - 1
        f64 = dict(dtype=torch.float64, device=dev)
        dA, dG = asm._mats["A"], asm._mats["G"]
        nA, nG = dA["nrows"], dG["nrows"]
        i32, i64, fd = torch.int32, torch.int64, torch.float64
        # one result buffer, mirrored by each slot's pinned host buffer at the same offsets:
        # the fixed fields, then the CSC values of A and G concatenated (the compaction
        # writes G's entries right after A's nonzeros), then the row indices the same way.
        # The kernel that finalises the values (the compaction, or the row scaling) also
        # stores them into the host mirror; the fixed fields follow in one copy kernel.
        nsup = dA["nsup"] + dG["nsup"]
        pk = _Packed([("bad", i32, NI), ("changed_at", fd, 1), ("A_indptr", i32, pat.n + 1), ("G_indptr", i32, pat.n + 1),
                      ("rhs", fd, nA + nG), ("row_scale_A", fd, nA), ("row_scale_G", fd, nG),
                      ("vals", fd, nsup), ("indices", i32, nsup)], dev)
        # z followed by [delta, epsilon, stamp, rows wanted]: one H2D per call, read by the
        # kernels from device memory so a captured graph replays for any delta of the
        # homotopy; the stamp (call counter) is what the CSC compaction writes into
        # changed_at when the sparsity pattern moves; rows wanted != 0 makes it mirror the
        # row indices too (a host buffer that does not hold the current pattern)
        zde_dev = torch.empty(lay.dim + 5, **f64)
        zde_pin = torch.zeros(lay.dim + 5, dtype=torch.float64, pin_memory=True)
        z_dev = zde_dev[: lay.dim]
        rowmax = torch.zeros(max(1, nA + nG), dtype=i64, device=dev)  # zero between calls (k_row_scale resets it)
        arr = lambda xs: ctypes_ptr_array([x.data_ptr() if x is not None else None for x in xs])  # noqa: E731
        soc_start, soc_dim = soc_tables(pat.n_orthant, pat.soc_dims, dev)
        keep = []  # ctypes arrays must outlive the plan
        rhs_dev = pk.d["rhs"]  # b and h: rows [0, nA) = b, [nA, nA + nG) = h
        pc_args = (pat.n, pk.d["A_indptr"].data_ptr(), pk.d["indices"].data_ptr(), pk.d["vals"].data_ptr(), nA,
                   rhs_dev.data_ptr(), pk.d["G_indptr"].data_ptr(), None, None, nG, rhs_dev[nA:].data_ptr(),
                   pat.n_orthant, len(pat.soc_dims), soc_start.data_ptr(), soc_dim.data_ptr(),
                   rowmax[:nA].data_ptr(), rowmax[nA:].data_ptr(), 1, max(dA["nsup"], dG["nsup"]),
                   pk.d["row_scale_A"].data_ptr(), pk.d["row_scale_G"].data_ptr())
        dim = lay.dim
        P_idx = np.arange(dim, dtype=np.int32)
        P_ptr = np.concatenate([np.arange(dim + 1), np.full(pat.n - dim, dim)]).astype(np.int32)
        self._plan = dict(pk=pk, z_dev=z_dev, zde_dev=zde_dev, zde_pin=zde_pin, rowmax=rowmax, rhs_dev=rhs_dev,
                          hosts=[], graph_kernels={}, side=torch.cuda.Stream(dev), rhs_const=asm._rhs["const"],
                          rhs_const_host=asm._rhs["const"].cpu().numpy(),
                          pc_args=pc_args, keep=keep, L=_lib.lib(), nA=nA, nG=nG,
                          soc=(soc_start, soc_dim), P_idx=P_idx, P_ptr=P_ptr, arr=arr,
                          P_plain=None, meta=_Meta(pat.z_idx, pat.sp_idx, pat.sm_idx, pat.t_idx),
                          # with _Z_HOST the interval / node kernels and the compaction read z,
                          # delta, epsilon, stamp and the rows flag straight from the pinned
                          # buffer (no H2D before K1); k_rhs reads the device copy made on its
                          # own stream while K1 runs
                          zsrc=zde_pin if _Z_HOST else zde_dev,
                          stamp=((zde_pin if _Z_HOST else zde_dev)[lay.dim + 2:].data_ptr(),
                                 pk.d["changed_at"].data_ptr()), calls=0,
                          pat_gen=0, want_rows=(zde_pin if _Z_HOST else zde_dev)[lay.dim + 3:].data_ptr(),
                          want_consts=(zde_pin if _Z_HOST else zde_dev)[lay.dim + 4:].data_ptr())

    def _make_slot(self, hb):
        """Device buffers of one in-flight iteration, paired with the pinned host buffer hb:
        the linearization outputs (read lazily by the LinearizedProblem handed out)
        and the unscaled program values (read lazily by unscaled_program), plus the
        kernel argument tables that point at them.  A slot is reused only when every
        result handed out from it has been dropped, so nothing is ever overwritten
        under a live result and no copy-out is needed before the next iteration."""
        import torch

        gt, asm, pat, pl = self.gt, self.asm, self.asm.pat, self._plan
        lay, dev = gt.lay, gt.device
        N, nxt, nu, nq, nc = lay.N, lay.n_xt, lay.n_u, lay.n_q, lay.n_c
        n_psi = 3 * nc + lay.n_g_out
        NI = N - 1
        f64 = dict(dtype=torch.float64, device=dev)
        pk, arr = pl["pk"], pl["arr"]
        lin = dict(ends=torch.empty((NI, nxt), **f64), jx=torch.empty((NI, nxt, nxt), **f64),
                   ju=torch.empty((NI, nxt, 2 * nu), **f64), js=torch.empty((NI, nxt), **f64),
                   defects=torch.empty((NI, nxt), **f64),
                   psi=torch.empty((NI, n_psi), **f64), psi_jac=torch.empty((NI, n_psi, 2 * lay.n_y), **f64),
                   theta=torch.empty((N, 6 * nc), **f64), theta_jac=torch.empty((N, 6 * nc, 3 * nq + 3 * nc), **f64),
                   imp_v=torch.empty((N, nq), **f64), imp_jac=torch.empty((N, nq, 3 * nq + 2 * nc), **f64))
        lin["bad"] = pk.d["bad"]
        dA, dG = asm._mats["A"], asm._mats["G"]
        unscaled = dict(vals=torch.empty(max(1, dA["nsup"] + dG["nsup"]), **f64),
                        rhs=torch.empty(max(1, pl["nA"] + pl["nG"]), **f64))
        keep = []

        def k(a):
            if a is not None and not isinstance(a, int):
                keep.append(a)
            return a

        lin_ptrs = k(arr([lin[kk] for kk in LIN_SOURCES]))
        outs = [(pk.d["A_indptr"], pk.d["indices"], pk.d["vals"]), (pk.d["G_indptr"], None, None)]  # concatenated
        rowmax = pl["rowmax"]
        nA = pl["nA"]
        r = asm._rhs
        delta = hb.host.data_ptr() - pk.dev.data_ptr()  # device output -> its host mirror (bytes)
        slot = dict(
            lin=lin, unscaled=unscaled, keep=keep, delta=delta,
            # plain: the compaction mirrors the values (final) and, when wanted, the rows;
            # preconditioned: only the rows (the row scaling mirrors the scaled values)
            packed=tuple(k(a) for a in asm.packed_args(lin_ptrs, outs, None, arr, pl["stamp"],
                                                       (delta, delta, pl["want_rows"], pl["want_consts"]))),
            packed_pc=tuple(k(a) for a in asm.packed_args(lin_ptrs, outs, [rowmax[:nA], rowmax[nA:]], arr,
                                                          pl["stamp"], (0, delta, pl["want_rows"], None))),
            rhs_args=(r["n"], r["rows"].data_ptr(), r["form"].data_ptr(), r["vsrc"].data_ptr(),
                      r["voff"].data_ptr(), r["seg_src"].data_ptr(), r["seg_off"].data_ptr(),
                      r["seg_len"].data_ptr(), r["seg_cb"].data_ptr(), r["cols"].data_ptr(), pl["z_dev"].data_ptr(),
                      lin_ptrs, pl["rhs_dev"].data_ptr(), delta),
            lin_args=(gt.disc._h.ptr, N, 1, int(lay.dim), int(gt.base_u), int(gt.base_p), pl["zsrc"].data_ptr(),
                      pl["zsrc"][lay.dim:].data_ptr()),
            lin_outs=tuple(lin[kk].data_ptr() for kk in ("ends", "jx", "ju", "js", "defects", "bad", "psi",
                                                         "psi_jac", "theta", "theta_jac", "imp_v", "imp_jac")))
        return slot

    def _launch(self, precondition, hb):
        """The device work of one iteration on the current stream: H2D of
        [z, delta, epsilon, stamp, flags], K1 + K3, CSC assembly, rhs, optional row
        scaling (the unscaled values kept in the slot); the kernels that finalise
        each result field also store it into the pinned host buffer `hb` (outputs
        in hb's device slot)."""
        import torch

        pl, sl = self._plan, hb.slot
        L = pl["L"]
        s = torch.cuda.current_stream(self.gt.device).cuda_stream
        cur = torch.cuda.current_stream(self.gt.device)
        side = pl["side"]
        if _Z_HOST:  # the device copy of z for k_rhs, on the side stream while K1 runs
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                pl["zde_dev"].copy_(pl["zde_pin"], non_blocking=True)
        elif _Z_UPLOAD_KERNEL:
            # the upload as a kernel: K1 starts behind it by programmatic launch (and a graph
            # without copy-engine nodes: N = 200 e2e 0.48 -> 0.40 ms, same box)
            zd, zh = pl["zde_dev"], pl["zde_pin"]
            _lib.check(L.cito_copy_mirror(zd.data_ptr(), zh.data_ptr(), zd.numel() * 8, 0, s), "z upload")
        else:
            pl["zde_dev"].copy_(pl["zde_pin"], non_blocking=True)
        h = self.gt.disc._h  # the handle's own library (a run-time compiled topology has its own)
        h.check(h.L.cito_linearize_all_dev2(*sl["lin_args"], *sl["lin_outs"], s), "linearize_all")
        # b/h of the linearized rows on a side stream, concurrently with the CSC compaction
        side.wait_stream(cur)
        pk = pl["pk"]
        with torch.cuda.stream(side):  # every store also into hb's host mirror
            # the constant rows of b/h: device only -- the host buffer holds them since its
            # creation (restored after a preconditioned call scaled them there)
            rc = pl["rhs_const"]
            _lib.check(L.cito_copy_mirror(pl["rhs_dev"].data_ptr(), rc.data_ptr(), rc.numel() * 8, 0,
                                          side.cuda_stream), "rhs constants")
            _lib.check(L.cito_rhs_dev(*sl["rhs_args"], side.cuda_stream), "rhs")
            # K1's non-finite flags (final once the side stream starts)
            _lib.check(L.cito_copy_mirror(hb.host.data_ptr(), pk.dev.data_ptr(), pk.layout["changed_at"][0], 0,
                                          side.cuda_stream), "flags")
        # the compaction (A and G concatenated; the fused row norms accumulate into the
        # rowmax workspace, which the preconditioning leaves zero again)
        _lib.check(L.cito_csc_assemble_packed_dev(*(sl["packed_pc"] if precondition else sl["packed"]), s),
                   "csc_assemble")
        cur.wait_stream(side)
        if precondition:  # row scaling in place, the unscaled values kept in the slot by the same kernel
            u = sl["unscaled"]
            _lib.check(L.cito_precondition_dev(*pl["pc_args"], u["vals"].data_ptr(), u["rhs"].data_ptr(), None,
                                               u["rhs"][pl["nA"]:].data_ptr(), sl["delta"], s), "precondition")
        # no copy at the end: every result field reached hb's host mirror from the kernel
        # that wrote it (flags, rhs rows, column pointers, stamp, values, wanted row
        # indices; row scales and scaled values/rhs from the preconditioning)

    def _copy_pattern(self, hb, stream):
        """Copy-engine transfer of the CSC pattern (column pointers, then the row
        indices [0, nnz)) into hb: a call whose pattern moved although hb held the
        previous one, so the compaction did not store it there."""
        pk = self._plan["pk"]
        lay = pk.layout
        o0, o1 = lay["A_indptr"][0], lay["G_indptr"][0] + 4 * lay["G_indptr"][2]
        hb.host[o0:o1].copy_(pk.dev[o0:o1], non_blocking=True)
        stream.synchronize()
        nnz = int(hb.h["A_indptr"][-1]) + int(hb.h["G_indptr"][-1])
        o = lay["indices"][0]
        hb.host[o: o + 4 * nnz].copy_(pk.dev[o: o + 4 * nnz], non_blocking=True)
        ov = lay["vals"][0]  # the values too: the compaction skipped the constants at the old positions
        hb.host[ov: ov + 8 * nnz].copy_(pk.dev[ov: ov + 8 * nnz], non_blocking=True)
        stream.synchronize()
        self.d2h_copied += (o1 - o0) + 12 * nnz

    def d2h_bytes(self, precondition=False, indices=False):
        """Bytes one iteration moves device -> host at the last call's nonzero count:
        the fixed fields + the values (+ the pattern with ``indices``, as in a call
        whose buffer does not hold the current pattern).  An upper bound when the
        buffer already holds the constant entries (16-byte chunks of constants are
        then not sent, ~15 % of the values).  ``self.d2h_copied`` accumulates it per
        call (+ the copies of a pattern fetched after the synchronisation)."""
        pl = self._plan
        lay = pl["pk"].layout
        nnz = pl.get("last_nnz", lay["vals"][2])
        nrhs, nlin = pl["nA"] + pl["nG"], int(self.asm._rhs["n"])
        # flags, stamp, the linearized b/h rows (the constant ones stay in the host buffer),
        # values; the pattern (column pointers, row indices) only when wanted
        n = (4 * lay["bad"][2] + 8 + 8 * nlin + 8 * nnz
             + (4 * (lay["A_indptr"][2] + lay["G_indptr"][2] + nnz) if indices else 0))
        if precondition:  # the row scales and every b/h row once more (scaled)
            n += 16 * nrhs
        return int(n)

    def _host_buffer(self):
        """A pinned result buffer no live array points into (a new one when every
        buffer is still referenced by programs the caller kept)."""
        pl = self._plan
        for hb in pl["hosts"]:
            if hb.free():
                return hb
        hb = _HostBuf(pl["pk"])
        hb.slot = self._make_slot(hb)
        hb.h["rhs"][:] = pl["rhs_const_host"]
        pl["hosts"].append(hb)
        return hb

    def _capture(self, precondition, hb):
        """Capture _launch (D2H into `hb`) as a CUDA graph, after one eager run
        that performs the library's first-call setup; one replay per iteration."""
        import torch

        pl = self._plan
        pl["captures"] = pl.get("captures", 0) + 1
        self._launch(precondition, hb)
        torch.cuda.current_stream(self.gt.device).synchronize()
        hb.rhs_scaled |= bool(precondition)
        hb.consts_ok &= not precondition
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launch_count()
        with torch.cuda.graph(g):
            self._launch(precondition, hb)
        pl["graph_kernels"][precondition] = _lib.launch_count() - n0
        hb.graphs[precondition] = g
        return g

    def iterate(self, z, delta, z_j=None, epsilon=None, precondition=False):
        """Returns (lin, prog, meta); with ``precondition`` the program comes back
        row-scaled on the device (= cito.conic.precondition, scp.py:414) and the
        result is (lin, scaled_prog, Preconditioner, meta)."""
        import scipy.sparse as sp
        import torch

        z = np.asarray(z, dtype=float)
        # z . z finite <=> every entry finite (barring overflow, which the exact test then clears)
        if not np.isfinite(z @ z) and not np.all(np.isfinite(z)):
            raise FloatingPointError("non-finite reference point")
        if self._plan is None:
            self._build_plan()
        pl = self._plan
        gt, pat = self.gt, self.asm.pat
        if epsilon is None:
            epsilon = gt.scenario.ctcs_epsilon
        stream = torch.cuda.current_stream(gt.device)
        zp = pl["zde_pin"].numpy()
        dim = pat.lay.dim
        zp[:dim] = z
        zp[dim] = float(delta)
        zp[dim + 1] = float(epsilon)
        pl["calls"] += 1
        zp[dim + 2] = float(pl["calls"])  # the stamp of this call (changed_at)
        hb = self._host_buffer()
        # the CSC row indices come back only into a buffer that does not hold the current
        # pattern (the compaction mirrors them when asked; it stamps changed_at when the
        # pattern moves, and then they are fetched after the synchronization)
        idx_now = hb.pat_gen != pl["pat_gen"]
        zp[dim + 3] = 1.0 if idx_now else 0.0
        zp[dim + 4] = 0.0 if (_SKIP_CONSTS and hb.consts_ok and not idx_now) else 1.0  # constants already there
        if hb.rhs_scaled and not precondition:  # the constant b/h rows, scaled there by a preconditioned call
            hb.h["rhs"][:] = pl["rhs_const_host"]
            hb.rhs_scaled = False
        if self.use_graph:
            g = hb.graphs.get(bool(precondition))
            if g is None:
                g = self._capture(bool(precondition), hb)
            g.replay()
            _lib.add_graph_launches(pl["graph_kernels"][bool(precondition)])
        else:
            self._launch(bool(precondition), hb)
        hb.rhs_scaled |= bool(precondition)
        hb.consts_ok = not precondition  # (a moved pattern brings every value back below)
        nA = pl["nA"]
        # host work that does not depend on the device results runs while the GPU works:
        # the objective, the (scaled) P, the lazy LinearizedProblem
        zj = z if z_j is None else z_j
        c = pat.objective_c(zj)
        c_unscaled = c
        P_data = pat.P_diag[: pat.lay.dim]
        if precondition:  # cost normalization (conic.py:311-316)
            omega = max(1.0, float(np.max(np.abs(c))) if c.size else 0.0)
            if P_data.size:
                omega = max(omega, float(np.max(np.abs(P_data))))
            P = sp.csc_matrix((P_data * (1.0 / omega), pl["P_idx"], pl["P_ptr"]), shape=(pat.n, pat.n))
            c = c / omega
        else:
            if pl["P_plain"] is None:  # constant: one read-only matrix shared by every result
                Pm = sp.csc_matrix((P_data.copy(), pl["P_idx"].copy(), pl["P_ptr"].copy()), shape=(pat.n, pat.n))
                for arr in (Pm.data, Pm.indices, Pm.indptr):
                    arr.flags.writeable = False
                pl["P_plain"] = Pm
            P = pl["P_plain"]
        lin = self._Lazy(hb.slot["lin"], z.copy())
        # the scipy/program objects over the pinned buffer, built while the GPU works with
        # the nonzero counts of the previous call (the pattern rarely moves between SCP
        # iterations); checked after the synchronisation and rebuilt if they differ
        pred = pl.get("last_nnz_ag")
        early = pred is not None and bool(_CSC_FAST) and not _CSC_CHECK  # direct construction probed and on
        built = self._program(hb, pred, P, c, precondition, omega if precondition else None) if early else None
        stream.synchronize()  # the one synchronization
        hh = hb.h
        if hh["changed_at"][0] == zp[dim + 2]:  # the pattern moved in this call
            pl["pat_gen"] += 1
            if not idx_now:
                self._copy_pattern(hb, stream)
                self.pattern_refetches += 1
        hb.pat_gen = pl["pat_gen"]
        nnz_A, nnz_G = int(hh["A_indptr"][-1]), int(hh["G_indptr"][-1])
        nnz = pl["last_nnz"] = nnz_A + nnz_G
        pl["last_nnz_ag"] = (nnz_A, nnz_G)
        self.d2h_copied += self.d2h_bytes(precondition, idx_now)  # what the graph moved
        bad = hh["bad"]
        if bad.any():
            raise FloatingPointError(f"non-finite state in intervals {np.where(bad != 0)[0].tolist()}")
        self._c_last = (zj, c_unscaled)  # the unscaled objective, for unscaled_program(z_j) of the same point
        if (built is None or pred != (nnz_A, nnz_G) or hh["A_indptr"][0] != 0 or hh["G_indptr"][0] != 0
                or _CSC_CHECK):
            built = self._program(hb, (nnz_A, nnz_G), P, c, precondition, omega if precondition else None,
                                  check=True)
        mats, prog, prec = built
        import weakref

        hb.live.append(weakref.ref(lin))  # the slot's device outputs stay untouched while lin lives
        self._last_lin = weakref.ref(lin)
        if precondition:
            self._pc_parts = (mats, nA, pl["nG"], hb)
            return lin, prog, prec, pl["meta"]
        self._pc_parts = None
        return lin, prog, pl["meta"]

    def _program(self, hb, nnz_ag, P, c, precondition, omega, check=False):
        """(mats, ConicProgram, Preconditioner or None) over hb's pinned arrays for the
        given nonzero counts of A and G (no copy).  check=False skips the O(1) CSC
        invariants that need the device result (the caller compares the counts)."""
        pl, pat = self._plan, self.asm.pat
        nA, nG = pl["nA"], pl["nG"]
        ConicProgram, ConeSpec = _conic_types()
        if pl.get("cones") is None or type(pl["cones"]) is not ConeSpec:
            pl["cones"] = ConeSpec(nonneg=pat.n_orthant, soc=pat.soc_dims)
        nnz_A, nnz_G = nnz_ag
        mats = {}
        for M, nrows, o, nnz in (("A", nA, 0, nnz_A), ("G", nG, nnz_A, nnz_G)):
            mats[M] = _csc_direct(hb.wrap("vals", o, nnz), hb.wrap("indices", o, nnz),
                                  hb.wrap(f"{M}_indptr", 0, pat.n + 1), (nrows, pat.n), check=check)
        prog = ConicProgram(P=P, c=c, A=mats["A"], b=hb.wrap("rhs", 0, nA), G=mats["G"], h=hb.wrap("rhs", nA, nG),
                            cones=pl["cones"])
        prec = None
        if precondition:
            if pl.get("ones") is None:
                pl["ones"] = np.ones(pat.n)
                pl["ones"].flags.writeable = False
            prec = _preconditioner_type()(row_scale_A=hb.wrap("row_scale_A", 0, nA),
                                          row_scale_G=hb.wrap("row_scale_G", 0, nG), var_scale=pl["ones"],
                                          cost_scale=omega)
        return mats, prog, prec

    def reserve(self, n, precondition=False):
        """Make sure n result slots exist with their CUDA graphs captured for this
        mode, so a loop that keeps the previous result alive while computing the
        next (cito.scp.solve holds lin/prog of iteration k during k+1) never
        captures in the middle of the loop.  Uses the last [z, delta, epsilon].  A
        buffer that a live result still points into is never written (its capture
        runs the iteration once): new buffers are made instead."""
        import torch

        if self._plan is None or not self.use_graph:
            return
        pl = self._plan
        pc = bool(precondition)
        ready = sum(1 for hb in pl["hosts"] if pc in hb.graphs)
        for hb in list(pl["hosts"]):
            if ready >= n:
                break
            if pc not in hb.graphs and hb.free():
                self._capture(pc, hb)
                ready += 1
        while ready < n:
            hb = _HostBuf(pl["pk"])
            hb.slot = self._make_slot(hb)
            hb.h["rhs"][:] = pl["rhs_const_host"]
            pl["hosts"].append(hb)
            self._capture(pc, hb)
            ready += 1
        torch.cuda.current_stream(self.gt.device).synchronize()

    def unscaled_program(self, z_j):
        """The program of the last preconditioned iterate BEFORE row scaling
        (= cito.scp.build_subproblem's output), lazily: its A/G values and b/h come
        back from the slot's device copy only when first read (the program keeps
        its slot busy, so the copy stays valid).  P and c (host) are exact."""
        import weakref

        import scipy.sparse as sp

        if self._pc_parts is None:
            raise RuntimeError("unscaled_program needs a preceding iterate(..., precondition=True)")
        mats, nA, nG, hb = self._pc_parts
        pat = self.asm.pat
        pl = self._plan
        if pl["P_plain"] is None:
            P_data = pat.P_diag[: pat.lay.dim]
            Pm = sp.csc_matrix((P_data.copy(), pl["P_idx"].copy(), pl["P_ptr"].copy()), shape=(pat.n, pat.n))
            for arr in (Pm.data, Pm.indices, Pm.indptr):
                arr.flags.writeable = False
            pl["P_plain"] = Pm
        ConicProgram, ConeSpec = _conic_types()
        zl, cl = self._c_last
        c = cl if (z_j is zl or np.array_equal(z_j, zl)) else pat.objective_c(z_j)
        prog = _lazy_program_type(ConicProgram)._new(
            self, hb, mats, nA, nG, P=pl["P_plain"], c=c,
            cones=ConeSpec(nonneg=pat.n_orthant, soc=pat.soc_dims))
        hb.live.append(weakref.ref(prog))
        return prog
