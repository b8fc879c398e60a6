"""GPU replay audit of a solved trajectory.

Drop-in for ``cito.verifier.replay_check`` (/root/reference/pkg/src/cito/verifier.py:236-346).
The reference walks the N-1 intervals in Python: per interval one fine
re-integration at 10x substeps (:283-285), ``grid`` sequential FOH-restricted
segment propagations at the nominal substeps (:220-233, :292), and jitted
per-sample audits (signed distances, joint residuals, auxiliary rates,
:257-272, :293-318).  Here every interval is one GPU thread of the primal
kernel K2: one fine launch for all intervals, ``grid`` chained segment launches
(all intervals per launch), and one K5 audit launch over all
(N-1)(grid+1) samples.  Only the final max/products over a few thousand
numbers and the cone margins of the decision vector stay on the host.
"""

import sys
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .discretizer import Discretizer

__all__ = ["FeasibilityReport", "replay_check", "ReplayAuditor"]

# auxiliary channel offsets within one contact block and the complementarity
# pairs of the psi rows (verifier.py:38-41)
_CH_PHIN, _CH_LAM, _CH_GAM, _CH_RHO, _CH_SD = range(5)
_PAIRS = ((_CH_PHIN, _CH_SD), (_CH_PHIN, _CH_LAM), (_CH_GAM, _CH_RHO))


@dataclass
class FeasibilityReport:
    """Same fields as cito.verifier.FeasibilityReport (verifier.py:160-216)."""

    max_penetration: float
    max_joint_drift: float
    pair_residuals: np.ndarray
    ctcs_increments: np.ndarray
    ctcs_epsilon: float
    cone_violation: float
    refinement_drift: float
    cross_products: np.ndarray = field(repr=False)


def _report_type():
    mod = sys.modules.get("cito.verifier")
    return getattr(mod, "FeasibilityReport", FeasibilityReport) if mod is not None else FeasibilityReport


class ReplayAuditor:
    """Per-transcription state of the replay audit: the nominal and the 10x
    discretizers (the reference's ``tr._replay_cache``, verifier.py:243-274)."""

    def __init__(self, model, mixing, path_fn, substeps, layout, state_scale, device=None):
        import torch

        self.model = model
        self.lay = layout
        self.nominal = Discretizer(model, mixing=mixing, path_fn=path_fn, substeps=substeps)
        self.fine = Discretizer(model, mixing=mixing, path_fn=path_fn, substeps=10 * substeps)
        self.state_scale = np.asarray(state_scale, dtype=float)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    def launch_count(self):
        return self.nominal.launch_count() + self.fine.launch_count()

    def _audit(self, xs, us):
        import torch

        lay = self.lay
        B = xs.shape[0]
        n_j = len(self.model.joints)
        f64 = dict(dtype=torch.float64, device=self.device)
        sds = torch.empty((B, max(1, lay.n_c)), **f64)
        cj = torch.empty((B, max(1, 2 * n_j)), **f64)
        om = torch.empty((B, max(1, lay.n_y)), **f64)
        s = torch.cuda.current_stream(self.device).cuda_stream
        self.nominal._h.check(self.nominal._h.L.cito_audit_dev(self.nominal._h.ptr, B, xs.data_ptr(), int(xs.stride(0)), us.data_ptr(),
                                             sds.data_ptr(), cj.data_ptr(), om.data_ptr(), s), "audit")
        return sds[:, : lay.n_c], cj[:, : 2 * n_j], om[:, : lay.n_y]

    def device_pass(self, z, grid):
        """Fine ends (N-1, n_xt), segment samples (grid+1, N-1, n_xt) and the
        per-sample audits, all on the device; returns host numpy arrays."""
        import torch

        lay = self.lay
        K = lay.N - 1
        xt0 = np.stack([z[lay.xp(k)] for k in range(K)])
        U = np.stack([z[lay.u(k)] for k in range(K)])                   # (K, 2 n_u) = [U-, U+]
        S = np.array([float(z[lay.s(k)][0]) for k in range(K)])
        U0, U1 = U[:, : lay.n_u], U[:, lay.n_u:]
        taus = np.linspace(0.0, 1.0, grid + 1)
        # segment inputs exactly as _segment_states forms them (verifier.py:225-231)
        seg_U = np.empty((grid, K, 2 * lay.n_u))
        seg_S = np.empty((grid, K))
        for idx, (a, b) in enumerate(zip(taus[:-1], taus[1:])):
            seg_U[idx, :, : lay.n_u] = (1.0 - a) * U0 + a * U1
            seg_U[idx, :, lay.n_u:] = (1.0 - b) * U0 + b * U1
            seg_S[idx] = S * (b - a)
        us = (1.0 - taus[:, None, None]) * U0[None] + taus[:, None, None] * U1[None]  # (grid+1, K, n_u), :294
        dev = self.device
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)  # noqa: E731
        x0_d, U_d, S_d = t(xt0), t(U), t(S)
        segU_d, segS_d, us_d = t(seg_U), t(seg_S), t(us)
        fine_end, fine_bad = self.fine.propagate_batch_device(x0_d, U_d, S_d)
        samples = torch.empty((grid + 1, K, lay.n_xt), dtype=torch.float64, device=dev)
        samples[0] = x0_d
        bads = [fine_bad]
        for idx in range(grid):  # chained: segment idx starts where idx-1 ended
            _, b_ = self.nominal.propagate_batch_device(samples[idx], segU_d[idx], segS_d[idx],
                                                        out=(samples[idx + 1], torch.empty(K, dtype=torch.int32,
                                                                                           device=dev)))
            bads.append(b_)
        flat = samples.view(-1, lay.n_xt)
        sds, cj, om = self._audit(flat, us_d.view(-1, lay.n_u))
        host = [a.cpu().numpy() for a in (fine_end, samples, sds, cj, om)]
        bad = torch.stack(bads).cpu().numpy()
        if bad.any():
            raise FloatingPointError("non-finite state during interval integration")
        return taus, host

    def check(self, z, grid=20, ctcs_epsilon=0.0):
        lay = self.lay
        model = self.model
        z = np.asarray(z, dtype=float)
        if z.shape != (lay.dim,):
            raise ValueError(f"expected decision vector of dimension {lay.dim}")
        K, n_c, n_y, n_q = lay.N - 1, lay.n_c, lay.n_y, lay.n_q
        taus, (fine_end, samples, sds, cj, om) = self.device_pass(z, grid)
        G1 = grid + 1
        sds, cj, om = sds.reshape(G1, K, -1), cj.reshape(G1, K, -1), om.reshape(G1, K, -1)
        pair_res = np.zeros((K, 3 * n_c))
        cross = np.zeros((K, 3 * n_c))
        ctcs = np.zeros((K, lay.n_g_out))
        max_pen = max_drift = max_joint = 0.0
        for k in range(K):  # verifier.py:283-318, reductions over the device results
            diff = (fine_end[k, : 2 * n_q] - z[lay.xm(k + 1)][: 2 * n_q]) / self.state_scale
            max_drift = max(max_drift, float(np.max(np.abs(diff))))
            dy = z[lay.y_of_xm(k + 1)] - z[lay.y_of_xp(k)]
            for i in range(n_c):
                for p, (a, b) in enumerate(_PAIRS):
                    pair_res[k, 3 * i + p] = max(0.0, min(dy[5 * i + a], dy[5 * i + b]))
            ctcs[k] = np.maximum(dy[5 * n_c: n_y], 0.0)
            if n_c:
                max_pen = max(max_pen, float(np.max(-sds[:, k])))
            if cj.shape[2]:
                max_joint = max(max_joint, float(np.max(np.linalg.norm(cj[:, k], axis=1))))
            rates = om[:, k]
            for i in range(n_c):
                for p, (a, b) in enumerate(_PAIRS):
                    ra = np.maximum(rates[:, 5 * i + a], 0.0)
                    rb = np.maximum(rates[:, 5 * i + b], 0.0)
                    cross[k, 3 * i + p] = float(np.max(ra) * np.max(rb))
        cone = 0.0  # friction-cone margins of the decision vector (verifier.py:320-333)
        n_a = lay.n_a
        for k in range(K):
            for u in z[lay.u(k)].reshape(2, -1):
                phi = u[n_a: n_a + 2 * n_c].reshape(n_c, 2)
                for i in range(n_c):
                    mu = model.contacts[i].friction_mu
                    cone = max(cone, abs(phi[i, 0]) - mu * phi[i, 1], -phi[i, 1])
        for k in range(lay.N):
            phi = z[lay.phi(k)].reshape(n_c, 2)
            for i in range(n_c):
                mu = model.contacts[i].friction_mu
                cone = max(cone, abs(phi[i, 0]) - mu * phi[i, 1], -phi[i, 1])
        return _report_type()(max_penetration=max(0.0, max_pen), max_joint_drift=max_joint,
                              pair_residuals=pair_res, ctcs_increments=ctcs, ctcs_epsilon=ctcs_epsilon,
                              cone_violation=max(0.0, cone), refinement_drift=max_drift, cross_products=cross)


_auditors = {}


def auditor_for(scenario):
    """One ReplayAuditor per scenario: from the reference's Transcription when
    cito.ocp is loaded (get_transcription, as verifier.py:238 does), else from
    this package's ScenarioSpec mirror."""
    key = id(scenario)
    hit = _auditors.get(key)
    if hit is not None and hit[0] is scenario:
        return hit[1]
    ocp = sys.modules.get("cito.ocp")
    if ocp is not None and hasattr(ocp, "get_transcription") and not _is_local(scenario):
        tr = ocp.get_transcription(scenario)
        lay = tr.layout
        aud = ReplayAuditor(tr.model, tr.mixing, tr.path_fn, scenario.substeps, lay,
                            tr.scaling.scale[lay.xm(0)][: 2 * lay.n_q])
    else:
        from .scenario import Layout, build_scaling

        lay = Layout(scenario)
        g, n_g = scenario.path_constraints()
        aud = ReplayAuditor(scenario.model, scenario.mixing_matrix(n_g), g, scenario.substeps, lay,
                            build_scaling(scenario, lay)[1][: 2 * lay.n_q])
    _auditors[key] = (scenario, aud)
    return aud


def _is_local(scenario):
    from .scenario import ScenarioSpec

    return isinstance(scenario, ScenarioSpec)


def replay_check(z, model, scenario, grid=20):
    """Drop-in for cito.verifier.replay_check(z, model, scenario, grid=20)
    (verifier.py:236-346): same FeasibilityReport, re-integration and sample
    audits on the GPU."""
    aud = auditor_for(scenario)
    if aud.model is not model and getattr(aud.model, "n_q", None) != getattr(model, "n_q", None):
        raise ValueError("model does not match the scenario's model")
    return aud.check(z, grid=grid, ctcs_epsilon=scenario.ctcs_epsilon)
