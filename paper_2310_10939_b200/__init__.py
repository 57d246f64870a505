"""B200-native one-vector graph clustering (arXiv 2310.10939), a drop-in for the
reference package's ``fast_spectral_cluster`` entry point (specluster/__init__.py:12-27).

The hot path -- Irwin-Hall start vector, T lazy-random-walk steps over the CSR, D^-1
normalisation, 1-D k-means -- runs in hand-written sm_100a CUDA behind the C-ABI of
include/sc_b200.h (libsc_b200.so).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (ConvergenceError, DeviceError, GraphFormatError, InputError,  # noqa: F401
                     RankDeficiencyError, SpeclusterError, UndefinedConductanceError)
from .graph import Graph, from_csr, from_edges  # noqa: F401
from .kmeans import KMeans1D, Partition, PointSet, lloyd  # noqa: F401
from .pipeline import MODES, PipelineResult, SpectralParams, fast_spectral_cluster  # noqa: F401
from .spectral import (DeviceGraph, EmbeddingMatrix, RandomWalkOp,  # noqa: F401
                       SignlessLaplacianOp, irwin_hall_key, power_method, sample_irwin_hall)

__all__ = [
    "Graph", "Partition", "PointSet", "SpectralParams", "PipelineResult", "MODES",
    "fast_spectral_cluster", "lloyd", "power_method", "RandomWalkOp", "SignlessLaplacianOp",
    "DeviceGraph", "KMeans1D", "EmbeddingMatrix", "sample_irwin_hall", "irwin_hall_key",
    "from_edges", "from_csr", "__version__",
]
