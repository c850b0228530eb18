"""``adaptiveload.io`` -> the reference file formats as written by the B200 tools
(paper_2605_17923_b200.traces: catalogs, cluster config, plans, models, trial traces, metrics,
summaries, manifest sidecars)."""

from paper_2605_17923_b200.traces import *  # noqa: F401,F403
