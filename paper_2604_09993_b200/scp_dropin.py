"""The three pre-IPM calls of the reference's SCP loop served from ONE device pass.

cito.scp.solve (/root/reference/pkg/src/cito/scp.py:383-467) calls, per attempt,

    lin = linearize_all(tr, z, delta_j, jobs=config.jobs)          scp.py:412
    prog, meta = build_subproblem(tr, lin, z, delta_j, config)      scp.py:413
    scaled_prog, prec = precondition(prog)                          scp.py:414

``install_scp()`` replaces those three module globals of ``cito.scp``:

  linearize_all     runs the whole iteration on the GPU -- GpuSCPStep.iterate with
                    preconditioning: one upload of [z, delta, epsilon, ...] from pinned memory, one CUDA
                    graph replay (K1 + K3, CSC assembly, rhs, row scaling; the result
                    written into a pinned host buffer) -- and returns the device-backed
                    LinearizedProblem
  build_subproblem  for that lin: the program before row scaling, whose A/G/b/h
                    stay on the device until read (scp.solve never reads them)
  precondition      for that program: the scaled program + Preconditioner already
                    on the host (cost scaling from the program's own c and P)

Any other argument (a foreign lin or program, other SCPConfig weights) falls
back to the general drop-ins (subproblem.build_subproblem / precondition), so
the patched functions stay correct for every caller.  ``uninstall()`` restores
the originals.
"""

import numpy as np

__all__ = ["install_scp", "SCPDropIns"]


class SCPDropIns:
    def __init__(self, scp_module, w_prox=2000.0, w_ep=50000.0):
        self.scp = scp_module
        self.w = (float(w_prox), float(w_ep))
        self._steps = {}  # id(tr) -> (tr, GpuSCPStep)
        self._last = None  # (lin, step, scaled, prec, meta)
        self._served = None  # (prog, scaled, prec)
        self.orig = None
        self.iterations = 0

    def _step(self, tr):
        from .subproblem import GpuSCPStep

        e = self._steps.get(id(tr))
        if e is None or e[0] is not tr:
            e = (tr, GpuSCPStep(tr, w_prox=self.w[0], w_ep=self.w[1]))
            self._steps[id(tr)] = e
        return e[1]

    def linearize_all(self, tr, z, delta, epsilon=None, jobs=1):
        step = self._step(tr)
        first = step._plan is None
        lin, scaled, prec, meta = step.iterate(z, delta, epsilon=epsilon, precondition=True)
        if first:  # solve keeps iteration k's results alive during k+1: two slots, both captured now
            step.reserve(2, precondition=True)
        self._last = (lin, step, scaled, prec, meta)
        self._served = None
        self.iterations += 1
        return lin

    def build_subproblem(self, tr, lin, z_j, delta, config):
        from . import subproblem

        last = self._last
        if (last is not None and last[0] is lin and (float(config.w_prox), float(config.w_ep)) == self.w):
            _, step, scaled, prec, meta = last
            prog = step.unscaled_program(np.asarray(z_j, dtype=float))
            self._served = (prog, scaled, prec)
            return prog, meta
        return subproblem.build_subproblem(tr, lin, z_j, delta, config)

    def precondition(self, prog):
        import scipy.sparse as sp

        from . import subproblem

        served = self._served
        if served is None or served[0] is not prog:
            return subproblem.precondition(prog)
        _, scaled, prec = served
        if prog.c is self._last[1]._c_last[1]:  # the objective the iterate scaled (z_j = z, as scp.solve passes)
            return scaled, prec
        # cost normalization of this program's own c and P (conic.py:311-316)
        c = prog.c
        omega = max(1.0, float(np.max(np.abs(c))) if c.size else 0.0)
        if prog.P.nnz:
            omega = max(omega, float(np.max(np.abs(prog.P.data))))
        if omega != prec.cost_scale or not np.array_equal(c / omega, scaled.c):
            P = sp.csc_matrix((prog.P.data * (1.0 / omega), prog.P.indices, prog.P.indptr), shape=prog.P.shape)
            scaled = type(scaled)(P=P, c=c / omega, A=scaled.A, b=scaled.b, G=scaled.G, h=scaled.h,
                                  cones=scaled.cones)
            prec = type(prec)(row_scale_A=prec.row_scale_A, row_scale_G=prec.row_scale_G, var_scale=prec.var_scale,
                              cost_scale=omega)
        return scaled, prec

    def uninstall(self):
        if self.orig is not None:
            self.scp.linearize_all, self.scp.build_subproblem, self.scp.precondition = self.orig
            self.orig = None


def install_scp(scp_module=None, w_prox=2000.0, w_ep=50000.0):
    """Patch ``cito.scp`` (or the given module) so its SCP loop runs each iteration's
    linearize + build + precondition as one device pass.  Returns the SCPDropIns
    (call ``.uninstall()`` to restore).  The transcription's own discretizer (used by
    initial_guess) is left alone; combine with ``install(tr)`` for that."""
    if scp_module is None:
        import cito.scp as scp_module  # noqa: PLC0415 (the reference package)
    d = SCPDropIns(scp_module, w_prox, w_ep)
    d.orig = (scp_module.linearize_all, scp_module.build_subproblem, scp_module.precondition)
    scp_module.linearize_all = d.linearize_all
    scp_module.build_subproblem = d.build_subproblem
    scp_module.precondition = d.precondition
    return d
