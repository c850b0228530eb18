"""``adaptiveload.costfit`` -> paper_2605_17923_b200.costfit (re-export; see adaptiveload/__init__.py)."""

from paper_2605_17923_b200.costfit import *  # noqa: F401,F403
