"""Bucket catalogs and policies used by the benchmarks and the DP step.

* ``reference_default_catalog`` -- the reference's default long-tail workload
  (cluster_sim.py:309-336): six 640x640 buckets S = 1600 ... 52800 (lambda = 8), weights by
  sample count, equal-token budget 480 000, dual constraint (480 000, 3e9, p = 2).
* ``wan21_catalog`` -- Wan-2.1 shapes under the Wan VAE geometry (lambda = 4): 480x832 and
  720x1280 stills and 17..81-frame videos, S = 1560 ... 75600 (BASELINE configs[2], [3]).
"""

from __future__ import annotations

from .scheduler import DualConstraint, TokenBudget
from .shapes import WAN21_GEOMETRY, LatentGeometry, MediaShape, build_catalog

_REFERENCE_DEFAULT = [((1, 640, 640), 30), ((17, 640, 640), 25), ((41, 640, 640), 20),
                      ((113, 640, 640), 15), ((233, 640, 640), 7), ((257, 640, 640), 3)]

_WAN21 = ([((1, 480, 832), 40), ((1, 720, 1280), 20)]
          + [((f, 480, 832), c) for f, c in [(17, 24), (33, 16), (49, 10), (65, 6), (81, 4)]]
          + [((f, 720, 1280), c) for f, c in [(17, 8), (33, 5), (49, 3), (81, 2)]])


def _weights(catalog):
    total = sum(b.sample_count for b in catalog)
    return [b.sample_count / total for b in catalog]


def reference_default_catalog(geom: LatentGeometry | None = None):
    catalog = build_catalog([(MediaShape(*s), c) for s, c in _REFERENCE_DEFAULT],
                            geom or LatentGeometry())
    return catalog, _weights(catalog), TokenBudget(480_000), DualConstraint(480_000, 3e9, 2.0)


def wan21_catalog(token_budget: int = 480_000, m_comp: float = 3e9, p: float = 2.0):
    catalog = build_catalog([(MediaShape(*s), c) for s, c in _WAN21], WAN21_GEOMETRY)
    return (catalog, _weights(catalog), TokenBudget(token_budget),
            DualConstraint(float(token_budget), m_comp, p))
