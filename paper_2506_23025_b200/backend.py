"""Kernel backend selection (mirror of reference tritpack/backend.py:21-63).

The reference resolves a *kernel module* by name ("compiled" / "python") with
the TRITPACK_BACKEND environment variable re-read on every call.  This package
registers exactly one backend, "cuda" (paper_2506_23025_b200.cuda_kernels): the
same duck-typed surface with bit-identical results, executed on the B200.
There is deliberately no CPU backend here -- a missing CUDA library raises.
To reroute the *reference* package's callers, insert the module into its
registry: ``tritpack.backend._BY_NAME["cuda"] = cuda_kernels``.
"""

from __future__ import annotations

import os
from types import ModuleType

ENV_VAR = "TRITPACK_BACKEND"

_BY_NAME: dict[str, ModuleType | None] = {}


def _registry() -> dict[str, ModuleType | None]:
    if not _BY_NAME:
        from . import cuda_kernels

        _BY_NAME["cuda"] = cuda_kernels
    return _BY_NAME


def available() -> tuple[str, ...]:
    """Backend names usable in this process, preferred first."""
    return tuple(name for name, mod in _registry().items() if mod is not None)


def default_name() -> str:
    """TRITPACK_BACKEND if set (validated), else "cuda"."""
    reg = _registry()
    forced = os.environ.get(ENV_VAR)
    if forced is not None:
        if forced not in reg:
            raise ValueError(f"{ENV_VAR}={forced!r}: unknown backend, expected one of {sorted(reg)}")
        return forced
    return "cuda"


def resolve(name: str | None = None) -> ModuleType:
    """Return the kernel module for ``name`` (default: `default_name()`)."""
    reg = _registry()
    if name is None:
        name = default_name()
    if name not in reg or reg[name] is None:
        raise ValueError(f"unknown backend {name!r}, expected one of {sorted(reg)}")
    return reg[name]
