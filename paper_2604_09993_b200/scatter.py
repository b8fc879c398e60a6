"""Multiple-shooting rows of the SCP subproblem, scattered on the GPU (K4).

Row (k, r) of A, built by cito.scp.build_subproblem (/root/reference/pkg/src/cito/scp.py:226-236
with eq() at :186-201) and assembled by cito.conic.canonicalize (conic.py:209-269), is

   +sigma_x[r]            at xm(k+1)[r]
   -jx[k,r,j] * sigma_x[j] at xp(k)[j]        (dropped when exactly zero)
   -ju[k,r,j] * sigma_u[j mod n_u] at u(k)[j] (dropped when exactly zero)
   -js[k,r]   * sigma_S   at s(k)             (dropped when exactly zero)
   -1 at slack+_{row}, +1 at slack-_{row}
   b[row] = ends[k,r] - (jx[k,r].z[xp(k)] + ju[k,r].z[u(k)] + js[k,r] z[s(k)])

with row = k*n_xt + r (dynamics rows come first in A, and their slacks are the
first n_int*n_xt equality slacks).  Columns: z in [0, lay.dim), slack+ at
lay.dim + i, slack- at lay.dim + n_eq_slack + i (scp.py:177-184).

``DynamicsCSC`` builds the CSC pattern (indptr/indices, int32, rows sorted
within each column) of those rows -- identical to the reference's
A[:n_dyn_rows] -- from the exact-zero pattern of one linearization, and the
slot map value-position for every (k, r, j).  ``slots_into`` maps the same
entries into any full-A CSC (e.g. the reference's own canonicalize output).
``DynamicsScatter`` then writes values and b on the device every iteration and
counts pattern mismatches (a value that became exactly zero or nonzero), in
which case the host rebuilds the pattern, as the reference implicitly does by
re-canonicalizing each iteration.
"""

import numpy as np

from . import _lib

__all__ = ["n_eq_slack", "DynamicsCSC", "DynamicsScatter"]


def n_eq_slack(lay):
    return (lay.N - 1) * lay.n_xt + lay.N * (lay.n_q + 2 * lay.n_c)  # scp.py:177


def n_cols(lay, n_psi):
    n_in = (lay.N - 1) * n_psi + lay.N * 4 * lay.n_c  # scp.py:178
    return lay.dim + 2 * n_eq_slack(lay) + n_in


def _entry_grid(lay):
    """(rows, cols) of every potential value entry, shaped (n_int, n_xt, n_xt+2n_u+1)."""
    n_int, nxt, nu2 = lay.N - 1, lay.n_xt, 2 * lay.n_u
    k = np.arange(n_int)[:, None, None]
    r = np.arange(nxt)[None, :, None]
    rows = np.broadcast_to(k * nxt + r, (n_int, nxt, nxt + nu2 + 1))
    xp = np.asarray(lay.xp_off)[:n_int] if hasattr(lay, "xp_off") else np.array([lay.xp(i)[0] for i in range(n_int)])
    uo = np.asarray(lay.u_off) if hasattr(lay, "u_off") else np.array([lay.u(i)[0] for i in range(n_int)])
    so = np.asarray(lay.s_off) if hasattr(lay, "s_off") else np.array([lay.s(i)[0] for i in range(n_int)])
    cols = np.empty((n_int, nxt, nxt + nu2 + 1), dtype=np.int64)
    cols[:, :, :nxt] = xp[:, None, None] + np.arange(nxt)[None, None, :]
    cols[:, :, nxt:nxt + nu2] = uo[:, None, None] + np.arange(nu2)[None, None, :]
    cols[:, :, -1] = so[:, None]
    return rows, cols


class DynamicsCSC:
    """CSC pattern of the dynamics rows of A (shape n_int*n_xt x n_cols) + value slots."""

    def __init__(self, lay, n_cols_total, state_scale, nz_x, nz_u, nz_s):
        n_int, nxt, nu2 = lay.N - 1, lay.n_xt, 2 * lay.n_u
        self.lay = lay
        self.n_rows = n_int * nxt
        self.n_cols = n_cols_total
        rows, cols = _entry_grid(lay)
        nz = np.concatenate([nz_x, nz_u, nz_s[:, :, None]], axis=2)
        # constant entries: +sigma at xm(k+1)[r], -1 at slack+, +1 at slack-
        xm = np.array([lay.xm(k + 1)[0] for k in range(n_int)])
        drow = np.arange(self.n_rows)
        c_rows = np.concatenate([drow, drow, drow])
        c_cols = np.concatenate([(xm[:, None] + np.arange(nxt)[None, :]).reshape(-1), lay.dim + drow,
                                 lay.dim + n_eq_slack(lay) + drow])
        c_vals = np.concatenate([np.tile(np.asarray(state_scale, dtype=float), n_int) * 1.0,
                                 -np.ones(self.n_rows), np.ones(self.n_rows)])
        v_rows = rows[nz]
        v_cols = cols[nz]
        all_rows = np.concatenate([c_rows, v_rows])
        all_cols = np.concatenate([c_cols, v_cols])
        order = np.lexsort((all_rows, all_cols))
        self.indices = all_rows[order].astype(np.int32)
        counts = np.bincount(all_cols, minlength=n_cols_total)
        self.indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        pos = np.empty(order.size, dtype=np.int64)
        pos[order] = np.arange(order.size)
        nc = c_rows.size
        self.const_pos = pos[:nc]
        self.const_vals = c_vals
        slots = np.full(nz.shape, -1, dtype=np.int32)
        slots[nz] = pos[nc:].astype(np.int32)
        self.slot_x = np.ascontiguousarray(slots[:, :, :nxt])
        self.slot_u = np.ascontiguousarray(slots[:, :, nxt:nxt + nu2])
        self.slot_s = np.ascontiguousarray(slots[:, :, -1])
        self.nnz = int(order.size)

    def template_data(self):
        data = np.zeros(self.nnz)
        data[self.const_pos] = self.const_vals
        return data

    @staticmethod
    def slots_into(indptr, indices, lay):
        """Slot maps of the dynamics value entries inside an arbitrary full-A CSC."""
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        ncol = indptr.size - 1
        nrow_big = int(indices.max()) + 1 if indices.size else 1
        col_of = np.repeat(np.arange(ncol), np.diff(indptr))
        keys = col_of * nrow_big + indices
        rows, cols = _entry_grid(lay)
        q = cols.reshape(-1) * nrow_big + rows.reshape(-1)
        p = np.searchsorted(keys, q)
        p = np.minimum(p, keys.size - 1)
        hit = keys[p] == q
        slots = np.where(hit, p, -1).astype(np.int32).reshape(rows.shape)
        nxt, nu2 = lay.n_xt, 2 * lay.n_u
        return (np.ascontiguousarray(slots[:, :, :nxt]), np.ascontiguousarray(slots[:, :, nxt:nxt + nu2]),
                np.ascontiguousarray(slots[:, :, -1]))


class DynamicsScatter:
    """Device-side value scatter of the dynamics rows (K4) for one layout."""

    def __init__(self, disc, lay, sigma_state, sigma_u, sigma_s, device):
        import torch

        self.disc = disc
        self.lay = lay
        self.device = device
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=device)
        n_int = lay.N - 1
        xp = np.array([lay.xp(k)[0] for k in range(n_int)], dtype=np.int64)
        uo = np.array([lay.u(k)[0] for k in range(n_int)], dtype=np.int64)
        so = np.array([lay.s(k)[0] for k in range(n_int)], dtype=np.int64)
        self._xp, self._u, self._s = t(xp, np.int64), t(uo, np.int64), t(so, np.int64)
        self._sig_x = t(sigma_state, np.float64)
        self._sig_u = t(sigma_u, np.float64)
        self.sig_s = float(sigma_s)
        self._mismatch = torch.zeros(1, dtype=torch.int32, device=device)
        self.pattern = None

    def set_slots(self, slot_x, slot_u, slot_s):
        import torch

        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=self.device)
        self._sx, self._su, self._ss = t(slot_x), t(slot_u), t(slot_s)

    def build_pattern(self, jx, ju, js, n_cols_total, state_scale):
        """Pattern from the exact-zero structure of one linearization (host arrays)."""
        self.pattern = DynamicsCSC(self.lay, n_cols_total, state_scale, np.asarray(jx) != 0.0,
                                   np.asarray(ju) != 0.0, np.asarray(js) != 0.0)
        self.set_slots(self.pattern.slot_x, self.pattern.slot_u, self.pattern.slot_s)
        return self.pattern

    def scatter(self, ends, jx, ju, js, z_dev, A_data, b_rows, stream=None):
        """Write the dynamics values into A_data / b_rows (device tensors).  Returns
        the device mismatch counter (int32[1]); nonzero means rebuild the pattern."""
        import torch

        self._mismatch.zero_()
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self.disc._h.check(self.disc._h.L.cito_scatter_dynamics_dev(
            self.disc._h.ptr, self.lay.N - 1, ends.data_ptr(), jx.data_ptr(), ju.data_ptr(), js.data_ptr(),
            z_dev.data_ptr(), self._xp.data_ptr(), self._u.data_ptr(), self._s.data_ptr(), self._sig_x.data_ptr(),
            self._sig_u.data_ptr(), self.sig_s, self._sx.data_ptr(), self._su.data_ptr(), self._ss.data_ptr(),
            A_data.data_ptr(), b_rows.data_ptr(), self._mismatch.data_ptr(), s), "scatter_dynamics")
        return self._mismatch
