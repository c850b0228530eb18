"""``adaptiveload.scheduler`` -> paper_2605_17923_b200.scheduler (re-export; see adaptiveload/__init__.py)."""

from paper_2605_17923_b200.scheduler import *  # noqa: F401,F403
