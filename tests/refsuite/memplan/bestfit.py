"""`memplan.bestfit` alias (see memplan/__init__.py)."""
from paper_1804_10001_b200.bestfit import *  # noqa: F401,F403
from paper_1804_10001_b200.bestfit import solve_bestfit  # noqa: F401

from . import OffsetLine, OffsetLineSet, _OutOfScopeType, find_block  # noqa: F401


class _RemainingBlocks(_OutOfScopeType):
    _name = "_RemainingBlocks (host window index debug type)"
