"""B200-native (sm_100a, fp64) re-implementation of CI-SCVX's per-SCP-iteration
discretize + linearize hot path (arxiv 2604.09993, reference package ``cito``).

Public surface (drop-in for the reference's Python call sites):
  Discretizer            -- cito.augmentation.Discretizer (augmentation.py:172-255)
  install(tr)            -- put it into a reference cito.ocp.Transcription
  linearize_all          -- cito.scp.linearize_all (scp.py:87-135), GPU-resident
  NodeLinearizer         -- Transcription.node_constraints/node_jacobians on the GPU
  DynamicsScatter        -- multiple-shooting rows straight into CSC values (scp.py:226-236)
"""

__version__ = "0.1.0"


def __getattr__(name):
    if name in ("Discretizer", "install", "AugmentedState", "IntervalParameterization", "IntervalResult"):
        from . import discretizer

        return getattr(discretizer, name)
    if name in ("linearize_all", "NodeLinearizer", "GpuTranscription", "LinearizedProblem"):
        from . import linearize

        return getattr(linearize, name)
    if name in ("DynamicsScatter",):
        from . import scatter

        return getattr(scatter, name)
    raise AttributeError(name)
