"""``jax.core.Tracer`` mapped to ``torch.Tensor`` (TEST INFRASTRUCTURE ONLY)."""

import torch

Tracer = torch.Tensor
