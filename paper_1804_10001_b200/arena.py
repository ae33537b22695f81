"""Replay arena (placeholder: exceptions only; full version follows)."""
from .core import MemplanError


class InvalidPlan(MemplanError):
    pass


class ExtraRequest(MemplanError):
    pass


class AllocAfterClose(MemplanError):
    pass


class LiveBlocksAtReset(MemplanError):
    pass


class UnknownId(MemplanError):
    pass


class OutOfMemory(MemplanError):
    pass
