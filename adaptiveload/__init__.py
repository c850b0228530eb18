"""Drop-in import path: ``adaptiveload`` backed by the B200 build.

Code written against the reference package (``from adaptiveload import adaln``,
``from adaptiveload.adaln import adaln_forward, ...``, ``from adaptiveload.errors import
ShapeMismatch``; reference pkg/src/adaptiveload/__init__.py and adaln/__init__.py:23-35) runs
unchanged on this package.  Every module here only re-exports ``paper_2605_17923_b200``: the
operator computes in the sm_100a kernels, the scheduler / shapes / sampler are the restatements
pinned bit-exact to the reference.  There is no numba or numpy backend (``adaln.BACKEND`` names
the CUDA library).
"""

from . import adaln, cluster_sim, costfit, errors, io, manifest, scheduler, shapes

__version__ = "0.1.0+b200"

__all__ = ["adaln", "cluster_sim", "costfit", "errors", "io", "manifest", "scheduler", "shapes",
           "__version__"]
