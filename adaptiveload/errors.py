"""``adaptiveload.errors`` -> paper_2605_17923_b200.errors (re-export; see adaptiveload/__init__.py)."""

from paper_2605_17923_b200.errors import *  # noqa: F401,F403
