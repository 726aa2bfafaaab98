"""Test-side access to the problem builders (paper_2410_09663_b200/configs.py) plus the two
module sets they are built from: the product's host types or the reference's own ``enksmpc``.
"""
from __future__ import annotations

from types import SimpleNamespace

from paper_2410_09663_b200.configs import (  # noqa: F401
    CONFIGS, make_burgers_problem, make_cnn_problem, make_constraint, make_linear_setup,
    sine_field)


def product_modules():
    import paper_2410_09663_b200 as pkg

    return SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)


def reference_modules(path: str = "/root/reference/pkg/src"):
    """The reference package: read-only from /root/reference (this container) or the unmodified
    installed copy in baseline/_ref (__graft_entry__.install_reference; travels to the GPU box)."""
    import importlib
    import sys

    if path not in sys.path:
        sys.path.insert(0, path)
    return SimpleNamespace(dynamics=importlib.import_module("enksmpc.dynamics"),
                           virtualsys=importlib.import_module("enksmpc.virtualsys"),
                           matvar=importlib.import_module("enksmpc.matvar"),
                           enks=importlib.import_module("enksmpc.enks"))
