"""Kernel-backend selector, mirroring the reference's ``mpcg.backend``
(pkg/src/mpcg/backend.py:1-48).

Callers look kernels up through the module attribute ``backend.kernels``.
The only implementation here is ``"b200"`` (libmpbjac.so, sm_100a); there
is deliberately no CPU fallback, so asking for anything else raises.
"""
import os
import warnings

from . import kernels_b200

kernels = kernels_b200
name = "b200"


def use_backend(which):
    """Bind the named kernel implementation (only 'b200' exists)."""
    global kernels, name
    if which != "b200":
        raise ValueError(f"unknown backend {which!r}, expected 'b200'")
    kernels = kernels_b200
    name = "b200"
    return kernels


_requested = os.environ.get("MPCG_BACKEND", "b200").strip().lower()
if _requested not in ("b200", ""):
    warnings.warn(f"MPCG_BACKEND={_requested!r} ignored: this build only has "
                  "the 'b200' backend", stacklevel=1)
