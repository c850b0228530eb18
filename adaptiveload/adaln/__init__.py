"""``adaptiveload.adaln`` -> the B200 operator (paper_2605_17923_b200.adaln): same names,
arguments, result dataclasses and exceptions as the reference's adaln/__init__.py:23-35."""

from paper_2605_17923_b200.adaln import *  # noqa: F401,F403
from paper_2605_17923_b200.adaln import __all__  # noqa: F401
