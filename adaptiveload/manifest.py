"""``adaptiveload.manifest`` -> paper_2605_17923_b200.manifest (re-export)."""

from paper_2605_17923_b200.manifest import *  # noqa: F401,F403
