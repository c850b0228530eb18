"""``adaptiveload.shapes`` -> paper_2605_17923_b200.shapes (re-export; see adaptiveload/__init__.py)."""

from paper_2605_17923_b200.shapes import *  # noqa: F401,F403
