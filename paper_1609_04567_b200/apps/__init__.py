"""The paper's workloads on the device engine (reference: apps/__init__.py)."""

from .helmholtz import HelmholtzConfig, helmholtz_kernel, helmholtz_solve

__all__ = ["HelmholtzConfig", "helmholtz_solve", "helmholtz_kernel"]
