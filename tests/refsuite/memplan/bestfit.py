"""`memplan.bestfit` alias (see memplan/__init__.py)."""
from paper_1804_10001_b200.bestfit import *  # noqa: F401,F403
from paper_1804_10001_b200.bestfit import solve_bestfit  # noqa: F401
from paper_1804_10001_b200.skyline import (OffsetLine, OffsetLineSet, _RemainingBlocks,  # noqa: F401
                                           find_block)
