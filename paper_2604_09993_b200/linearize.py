"""GPU-resident ``linearize_all`` (cito/scp.py:87-135) and node relations.

``GpuTranscription`` owns, for one scenario, the interval discretizer (K1/K2),
the node-relation kernel (K3) and the device-side index maps of the decision
vector layout (cito/ocp.py:131-203).  ``linearize_all`` gathers the interval
starts/controls/dilations and the node input vectors from z on the device,
runs K1 and K3, forms the multiple-shooting defects, and returns a
``LinearizedProblem`` with the reference's field names and shapes (numpy,
physical units) -- or keeps everything on the device (``to_host=False``) for
the CSC scatter (scatter.py).
"""

import sys
from dataclasses import dataclass

import numpy as np

from . import _lib
from .discretizer import Discretizer

__all__ = ["node_inputs", "LinearizedProblem", "GpuTranscription", "linearize_all", "NodeLinearizer",
           "initial_guess", "initial_guess_batch"]


def node_inputs(lay, z):
    """y pairs and packed node vectors exactly as Transcription._node_inputs (ocp.py:312-334)."""
    n_q = lay.n_q
    N = lay.N
    y_pairs = np.stack([np.concatenate([z[lay.y_of_xp(k)], z[lay.y_of_xm(k + 1)]]) for k in range(N - 1)])
    theta_vecs = np.stack([
        np.concatenate([z[lay.xm(k)][:n_q], z[lay.xm(k)][n_q: 2 * n_q], z[lay.xp(k)][n_q: 2 * n_q],
                        z[lay.phi(k)], z[lay.gam(k)]]) for k in range(N)])
    return y_pairs, theta_vecs


@dataclass
class LinearizedProblem:
    """Same fields as cito.scp.LinearizedProblem (scp.py:69-84)."""

    z_ref: np.ndarray
    ends: np.ndarray
    jx: np.ndarray
    ju: np.ndarray
    js: np.ndarray
    defects: np.ndarray
    psi: np.ndarray
    psi_jac: np.ndarray
    theta: np.ndarray
    theta_jac: np.ndarray
    imp_v: np.ndarray
    imp_jac: np.ndarray


class LazyLinearizedProblem:
    """LinearizedProblem (scp.py:69-84) whose arrays stay on the device until a
    field is read: the SCP loop hands it straight to build_subproblem (which
    assembles on the device), so the host never pays for the 2 MB of Jacobians
    unless it asks for them.  First access copies every field into fresh numpy
    arrays with one synchronization."""

    FIELDS = ("ends", "jx", "ju", "js", "defects", "psi", "psi_jac", "theta", "theta_jac", "imp_v", "imp_jac")

    def __init__(self, dev, z_ref):
        self._dev = dev
        self.z_ref = z_ref
        self._host = None

    def materialize(self):
        if self._host is None:
            import torch

            pinned = {k: torch.empty(self._dev[k].shape, dtype=self._dev[k].dtype, pin_memory=True)
                      for k in self.FIELDS}
            for k in self.FIELDS:
                pinned[k].copy_(self._dev[k], non_blocking=True)
            torch.cuda.current_stream(self._dev["jx"].device).synchronize()
            self._host = {k: v.numpy().copy() for k, v in pinned.items()}
        return self._host

    def __getattr__(self, name):
        if name in LazyLinearizedProblem.FIELDS:
            return self.materialize()[name]
        raise AttributeError(name)

    def device_arrays(self):
        """The device tensors behind this result, or None once the producer has
        reclaimed them for a later iteration (the host copy is then authoritative)."""
        return self._dev

    def release_device(self):
        """Take a host copy and drop the device references: called by the producer
        right before it overwrites the buffers with the next iteration."""
        self.materialize()
        self._dev = None


def _lp_type():
    mod = sys.modules.get("cito.scp")
    if mod is not None and hasattr(mod, "LinearizedProblem"):
        return mod.LinearizedProblem
    return LinearizedProblem


class NodeLinearizer:
    """Transcription.node_constraints + node_jacobians (ocp.py:336-365) via K3."""

    def __init__(self, disc):
        self.disc = disc

    def device(self, y_pairs, theta_vecs, delta, epsilon, out=None, stream=None):
        import torch

        h = self.disc._h
        d = h.dims
        n_c = len(self.disc.model.contacts)
        n_q, n_y = d.n_q, d.n_y
        n_psi = 3 * n_c + (n_y - 5 * n_c)
        Np, Nn = y_pairs.shape[0], theta_vecs.shape[0]
        dev = theta_vecs.device
        f64 = dict(dtype=torch.float64, device=dev)
        if out is None:
            out = (torch.empty((Np, n_psi), **f64), torch.empty((Np, n_psi, 2 * n_y), **f64),
                   torch.empty((Nn, 6 * n_c), **f64), torch.empty((Nn, 6 * n_c, 3 * n_q + 3 * n_c), **f64),
                   torch.empty((Nn, n_q), **f64), torch.empty((Nn, n_q, 3 * n_q + 2 * n_c), **f64))
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        yp = y_pairs if Np else theta_vecs
        h.check(h.L.cito_node_linearize_dev(h.ptr, Np, Nn, yp.data_ptr(), theta_vecs.data_ptr(),
                                                      float(delta), float(epsilon),
                                                      *[o.data_ptr() for o in out], s), "node_linearize")
        return out

    def host(self, y_pairs, theta_vecs, delta, epsilon):
        import torch

        dev = torch.device("cuda", torch.cuda.current_device())
        yp = torch.as_tensor(np.ascontiguousarray(y_pairs, dtype=np.float64), device=dev)
        tv = torch.as_tensor(np.ascontiguousarray(theta_vecs, dtype=np.float64), device=dev)
        out = self.device(yp, tv, delta, epsilon)
        torch.cuda.current_stream(dev).synchronize()
        return tuple(o.cpu().numpy() for o in out)


class GpuTranscription:
    """Device-side workspace of one scenario (reference Transcription or our ScenarioSpec)."""

    def __init__(self, tr_or_scenario, device=None):
        import torch

        if hasattr(tr_or_scenario, "layout") and hasattr(tr_or_scenario, "discretizer"):
            tr = tr_or_scenario
            self.scenario = tr.scenario
            self.lay = tr.layout
            self.disc = Discretizer(tr.model, mixing=tr.mixing, path_fn=tr.path_fn, substeps=tr.scenario.substeps)
        else:
            from .scenario import Layout

            sc = tr_or_scenario
            self.scenario = sc
            self.lay = Layout(sc)
            g, n_g = sc.path_constraints()
            self.disc = Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=g, substeps=sc.substeps)
        self.nodes = NodeLinearizer(self.disc)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        lay = self.lay
        N, n_q = lay.N, lay.n_q
        idx_start = np.stack([lay.xp(k) for k in range(N - 1)])
        idx_end = np.stack([lay.xm(k + 1) for k in range(N - 1)])
        idx_u = np.stack([lay.u(k) for k in range(N - 1)])
        idx_s = np.array([lay.s(k)[0] for k in range(N - 1)])
        idx_yp = np.stack([np.concatenate([lay.y_of_xp(k), lay.y_of_xm(k + 1)]) for k in range(N - 1)])
        idx_th = np.stack([np.concatenate([lay.xm(k)[:n_q], lay.xm(k)[n_q: 2 * n_q], lay.xp(k)[n_q: 2 * n_q],
                                           lay.phi(k), lay.gam(k)]) for k in range(N)])
        # layout bases as used by the fused kernels (identical to ocp.Layout's formulas, ocp.py:154-174)
        self.base_u = 2 * N * lay.n_xt
        self.base_p = self.base_u + (N - 1) * (2 * lay.n_u + 1)
        if not (int(lay.u(0)[0]) == self.base_u and int(lay.phi(0)[0]) == self.base_p
                and int(lay.xp(N - 1)[0]) == (2 * (N - 1) + 1) * lay.n_xt):
            raise ValueError("decision-vector layout differs from cito.ocp.Layout (ocp.py:154-174)")
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=self.device)
        self._i_start, self._i_end, self._i_u, self._i_s = t(idx_start), t(idx_end), t(idx_u), t(idx_s)
        self._i_yp, self._i_th = t(idx_yp), t(idx_th)
        self.n_imp = 3 * n_q + 2 * lay.n_c

    def _alloc_out(self, P):
        """Device result buffers of linearize_device for P problems (problem-major)."""
        import torch

        lay = self.lay
        N, nxt, nu, nq, nc = lay.N, lay.n_xt, lay.n_u, lay.n_q, lay.n_c
        NI, NN = P * (N - 1), P * N
        n_psi = 3 * nc + lay.n_g_out
        f64 = dict(dtype=torch.float64, device=self.device)
        out = dict(ends=torch.empty((NI, nxt), **f64), jx=torch.empty((NI, nxt, nxt), **f64),
                   ju=torch.empty((NI, nxt, 2 * nu), **f64), js=torch.empty((NI, nxt), **f64),
                   defects=torch.empty((NI, nxt), **f64),
                   bad=torch.empty((NI,), dtype=torch.int32, device=self.device),
                   psi=torch.empty((NI, n_psi), **f64), psi_jac=torch.empty((NI, n_psi, 2 * lay.n_y), **f64),
                   theta=torch.empty((NN, 6 * nc), **f64), theta_jac=torch.empty((NN, 6 * nc, 3 * nq + 3 * nc), **f64),
                   imp_v=torch.empty((NN, nq), **f64), imp_jac=torch.empty((NN, nq, 3 * nq + 2 * nc), **f64))
        return out

    def linearize_device(self, z_dev, delta, epsilon=None, k1_events=None, out=None):
        """Everything on the device in one C-ABI call (cito_linearize_all_dev): the
        interval kernel and the node-relation kernel read z directly and run
        concurrently.  ``z_dev`` is (dim,) or a multi-start batch (P, dim); outputs
        are stacked problem-major ((P*(N-1), ...) / (P*N, ...)).  Returns a dict of
        torch tensors.  ``k1_events`` = (start, end) CUDA events recorded around
        the call on the current stream."""
        import torch

        if epsilon is None:
            epsilon = self.scenario.ctcs_epsilon
        lay = self.lay
        P = 1 if z_dev.dim() == 1 else z_dev.shape[0]
        if z_dev.shape[-1] != lay.dim or not z_dev.is_contiguous():
            raise ValueError(f"z must be contiguous with last dimension {lay.dim}")
        N = lay.N
        if out is None:
            out = self._alloc_out(P)
        stream = torch.cuda.current_stream(self.device)
        if k1_events is not None:
            k1_events[0].record(stream)
        o = out
        self.disc._h.check(self.disc._h.L.cito_linearize_all_dev(
            self.disc._h.ptr, N, P, int(lay.dim), int(self.base_u), int(self.base_p), z_dev.data_ptr(), float(delta),
            float(epsilon), o["ends"].data_ptr(), o["jx"].data_ptr(), o["ju"].data_ptr(), o["js"].data_ptr(),
            o["defects"].data_ptr(), o["bad"].data_ptr(), o["psi"].data_ptr(), o["psi_jac"].data_ptr(),
            o["theta"].data_ptr(), o["theta_jac"].data_ptr(), o["imp_v"].data_ptr(), o["imp_jac"].data_ptr(),
            stream.cuda_stream), "linearize_all")
        if k1_events is not None:
            k1_events[1].record(stream)
        return out

    def linearize_to_host(self, Z, delta, epsilon=None, out=None):
        """Multi-start linearization with host arrays in and out (the configs[3] path):
        ``Z`` (P, dim) decision vectors, one per start; returns a dict of numpy arrays
        stacked problem-major like ``linearize_device`` (written into ``out``, a dict of
        caller-owned -- e.g. page-locked -- arrays, when given).  The problems run as
        chunks of about one wave of the interval kernel (3 intervals per CTA x #SMs;
        the last chunk takes the remainder), each chunk's results copied back on a
        side stream while the next chunks compute.  Raises FloatingPointError like
        linearize_all (scp.py:116-118) for non-finite end states."""
        import torch

        Zt = Z if torch.is_tensor(Z) else torch.from_numpy(np.ascontiguousarray(np.asarray(Z, dtype=np.float64)))
        if Zt.dim() == 1:
            Zt = Zt[None]
        P, N = Zt.shape[0], self.lay.N
        dev = self.device
        z_dev = Zt.to(dev, non_blocking=True)
        if getattr(self, "_host_plan", (None,))[0] != P:
            self._host_plan = (P, self._alloc_out(P))  # device result buffers
        dbuf = self._host_plan[1]
        if out is None:
            out = {k: np.empty(tuple(v.shape), dtype=np.int32 if v.dtype == torch.int32 else np.float64)
                   for k, v in dbuf.items()}
        hout = {k: torch.from_numpy(v) for k, v in out.items()}
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        per = max(1, (3 * n_sm) // (N - 1))
        nch = max(1, P // per)
        stream = torch.cuda.current_stream(dev)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(dev)
        cs = self._copy_stream

        def rows(v, p0, p1):  # interval arrays have N-1 rows per problem, node arrays N
            per_p = N - 1 if v.shape[0] == P * (N - 1) else N
            return slice(p0 * per_p, p1 * per_p)

        chunks = []
        for c in range(nch):  # all launches first: pageable destinations make the copies block the host
            p0, p1 = c * per, (P if c == nch - 1 else (c + 1) * per)
            self.linearize_device(z_dev[p0:p1], delta, epsilon, out={k: v[rows(v, p0, p1)] for k, v in dbuf.items()})
            ev = torch.cuda.Event()
            ev.record(stream)
            chunks.append((p0, p1, ev))
        for p0, p1, ev in chunks:
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                for k, v in dbuf.items():
                    hout[k][rows(v, p0, p1)].copy_(v[rows(v, p0, p1)], non_blocking=True)
        cs.synchronize()
        if out["bad"].any():
            raise FloatingPointError(f"non-finite state in intervals {np.where(out['bad'] != 0)[0].tolist()}")
        return out

    def linearize_all(self, z, delta, epsilon=None, jobs=1):
        """Drop-in for cito.scp.linearize_all(tr, z, delta, epsilon, jobs) (scp.py:87-135)."""
        import torch

        z = np.asarray(z, dtype=float)
        if not np.all(np.isfinite(z)):
            raise FloatingPointError("non-finite reference point")
        z_dev = torch.as_tensor(np.ascontiguousarray(z), device=self.device)
        r = self.linearize_device(z_dev, delta, epsilon)
        bad = r["bad"].cpu().numpy()  # the reference's end-state check (augmentation.py:231-233)
        if bad.any():
            raise FloatingPointError(f"non-finite state in intervals {np.where(bad != 0)[0].tolist()}")
        lin = LazyLinearizedProblem(r, z.copy())
        # keep the device copy so build_subproblem (subproblem.py) can assemble from it
        # without another host->device round trip
        self.last = (lin, r, z_dev)
        return lin


def initial_guess(scenario, disc, lay=None, seed=None):
    """Transcription.initial_guess (cito/ocp.py:461-505) with the y forward pass on the GPU.

    Same RNG draw order as the reference, so U/S/impulses are bit-identical; the
    auxiliary channels come from the N-1 sequential K2 propagations."""
    from .scenario import Layout

    lay = lay or Layout(scenario)
    n_q = lay.n_q
    z = _initial_guess_no_y(scenario, lay, seed)
    z[lay.y_of_xm(0)] = np.zeros(lay.n_y)
    for k in range(lay.N):
        z[lay.y_of_xp(k)] = z[lay.y_of_xm(k)]
        if k == lay.N - 1:
            break
        start = np.concatenate([z[lay.xp(k)][: 2 * n_q], z[lay.y_of_xp(k)]])
        end = disc.propagate(start, z[lay.u(k)].reshape(2, -1), float(z[lay.s(k)][0]))
        z[lay.y_of_xm(k + 1)] = end[2 * n_q:]
    return z


def initial_guess_batch(scenario, disc, seeds, lay=None):
    """Multi-start initial guesses (cito/ocp.py:461-505 for each seed), with the y
    forward pass batched across problems: N-1 propagate launches (one per
    interval index, all problems at once) instead of P*(N-1).  Row p equals
    initial_guess(scenario, disc, lay, seed=seeds[p])."""
    from .scenario import Layout

    lay = lay or Layout(scenario)
    n_q, N = lay.n_q, lay.N
    Z = np.stack([_initial_guess_no_y(scenario, lay, s) for s in seeds])
    for k in range(N):
        Z[:, lay.y_of_xp(k)] = Z[:, lay.y_of_xm(k)]
        if k == N - 1:
            break
        starts = np.concatenate([Z[:, lay.xp(k)[: 2 * n_q]], Z[:, lay.y_of_xp(k)]], axis=1)
        ends = disc.propagate_batch(starts, Z[:, lay.u(k)], Z[:, lay.s(k)[0]])
        Z[:, lay.y_of_xm(k + 1)] = ends[:, 2 * n_q:]
    return Z


def _initial_guess_no_y(sc, lay, seed):
    """Everything of initial_guess except the y forward pass (same RNG draw order)."""
    model = sc.model
    rng = np.random.default_rng(sc.seed if seed is None else seed)
    n_q = lay.n_q
    z = np.zeros(lay.dim)
    q_i, q_f = sc.x_init[:n_q], sc.x_final[:n_q]
    for k in range(lay.N):
        frac = k / (lay.N - 1)
        pose = (1.0 - frac) * q_i + frac * q_f
        z[lay.xm(k)[:n_q]] = pose
        z[lay.xp(k)[:n_q]] = pose
    for k in range(lay.N - 1):
        u = np.zeros(2 * lay.n_u)
        for side in range(2):
            base = side * lay.n_u + lay.n_a
            for i in range(lay.n_c):
                mu = model.contacts[i].friction_mu
                fn = rng.uniform(0.0, sc.guess_force_scale)
                ft = rng.uniform(-mu * fn, mu * fn) if fn > 0 else 0.0
                u[base + 2 * i] = ft
                u[base + 2 * i + 1] = fn
        z[lay.u(k)] = u
        z[lay.s(k)] = sc.s_nominal
    for k in range(lay.N):
        blk = np.zeros(2 * lay.n_c)
        for i in range(lay.n_c):
            mu = model.contacts[i].friction_mu
            pn = rng.uniform(0.0, sc.guess_impulse_scale) if sc.guess_impulse_scale else 0.0
            pt = rng.uniform(-mu * pn, mu * pn) if pn > 0 else 0.0
            blk[2 * i] = pt
            blk[2 * i + 1] = pn
        z[lay.phi(k)] = blk
    return z


_cache = {}


def transcription_for(tr):
    """The cached GpuTranscription of a reference Transcription (one per tr)."""
    key = id(tr)
    g = _cache.get(key)
    if g is None or g[0] is not tr:
        g = (tr, GpuTranscription(tr))
        _cache[key] = g
    return g[1]


def linearize_all(tr, z, delta, epsilon=None, jobs=1):
    """Module-level drop-in for cito.scp.linearize_all: caches one GpuTranscription per tr."""
    return transcription_for(tr).linearize_all(z, delta, epsilon, jobs)
