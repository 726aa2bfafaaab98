"""B200-native matrix-variate EnKS for optimal inferential control (arXiv 2410.09663).

A drop-in for the reference package's smoother hot path (``enksmpc.enks``):
``from paper_2410_09663_b200 import enks`` exposes init_ensemble / predict /
update / smooth_horizon with the reference signatures, backed by sm_100a
kernels behind the C-ABI in include/enks_b200.h.  Host-side mirrors of the
reference's configuration types live in ``matvar``, ``virtualsys`` and
``dynamics``.
"""
__version__ = "0.1.0"

from . import dynamics, matvar, virtualsys  # noqa: F401  (host-only, no device needed)

__all__ = ["dynamics", "matvar", "virtualsys", "enks", "engine", "ops"]
