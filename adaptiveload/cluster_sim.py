"""``adaptiveload.cluster_sim`` -> the parts of the reference's simulator module that sit on the
B200 hot path: the per-rank bucket draw (``sample_assignments``, bit-exact with
cluster_sim.py:113-131), the imbalance metrics (``cv_step``, ``compute_cv``,
cluster_sim.py:161-174) and the default catalog / policies (cluster_sim.py:309-336).  The
measured data-parallel step that replaces ``simulate_step`` is ``paper_2605_17923_b200.dp_step``.
"""

from paper_2605_17923_b200.catalogs import reference_default_catalog as _default
from paper_2605_17923_b200.sampler import compute_cv, cv_step, sample_assignments  # noqa: F401

__all__ = ["sample_assignments", "cv_step", "compute_cv", "default_catalog",
           "default_token_budget", "default_dual_constraint"]


def default_catalog(geom=None):
    """The reference's default long-tail catalog (six 640x640 buckets) and its weights."""
    catalog, weights, _, _ = _default(geom)
    return catalog, weights


def default_token_budget():
    return _default()[2]


def default_dual_constraint():
    return _default()[3]
