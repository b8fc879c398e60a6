"""Import the UNMODIFIED reference package ``cito`` through the jax shim.

TEST INFRASTRUCTURE ONLY.  Works only in the build container (where
``/root/reference`` exists); used to generate the golden fixtures under
``tests/golden/`` (see ``tests/golden/make_golden.py``) and to pin the C
oracle.  The GPU box never has ``/root/reference``; nothing on the product
path imports this module.
"""

import os
import sys

REF_SRC = os.environ.get("CITO_REF_SRC", "/root/reference/pkg/src")
SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "jaxshim")


def available():
    return os.path.isdir(os.path.join(REF_SRC, "cito"))


def import_cito():
    """Return the reference ``cito`` package (modules loaded under the shim)."""
    if not available():
        raise ImportError(f"reference source not found at {REF_SRC}")
    for p in (SHIM, REF_SRC):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch

    torch.set_default_dtype(torch.float64)
    import cito  # noqa: F401
    import cito.augmentation  # noqa: F401
    import cito.conic  # noqa: F401
    import cito.contact_dynamics  # noqa: F401
    import cito.multibody  # noqa: F401
    import cito.ocp  # noqa: F401
    import cito.scp  # noqa: F401

    return cito


def assets_dir():
    return os.path.join(REF_SRC, "cito", "assets")
