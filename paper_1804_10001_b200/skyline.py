"""Host-side skyline types for step-by-step inspection of the best-fit
heuristic — the reference's public debug surface (`OffsetLine`,
`OffsetLineSet`, `find_block`, `_RemainingBlocks`; bestfit.py:42-273).

The planner never uses these: `solve_bestfit` runs on the GPU
(csrc/plan.cu).  They exist so code (and tests) that drive the heuristic
one operation at a time keep working against this package.  The skyline
is held the way the GPU kernel holds it — a time-ordered array of lines
[lo, hi) at a height, adjacent lines touching — and every operation
follows the rules the kernel implements:

  R3 choose_offset  lowest line, leftmost on equal heights (bestfit.py:115-122)
  R4 find_block     contained blocks only; best key (life, size, -id)
                    (bestfit.py:204-220, 243-262)
  R5 lift_up        only neighbour -> merge into it; equal neighbours ->
                    merge all three; else into the lower one (bestfit.py:180-201)
  R6 place          offset = line height; [lo, alloc) keeps the height,
                    [alloc, free) is raised by the size, [free, hi) keeps
                    it; only the raised segment re-merges with an
                    equal-height previous, then next line (bestfit.py:149-178)
"""

from __future__ import annotations

from dataclasses import dataclass

from .bestfit import ContainmentViolation, IllegalLift


@dataclass(eq=False)
class OffsetLine:
    """One skyline segment [time_lo, time_hi) at `height` (a view: the
    owning set keeps it current while it is part of the skyline)."""

    time_lo: int
    time_hi: int
    height: int

    def __repr__(self) -> str:
        return f"OffsetLine([{self.time_lo}, {self.time_hi}) @ {self.height})"


class OffsetLineSet:
    """The skyline over [t_lo, t_hi): starts as one line at height 0."""

    def __init__(self, t_lo: int, t_hi: int):
        if t_hi <= t_lo:
            raise ValueError(f"empty skyline span [{t_lo}, {t_hi})")
        self._lines = [OffsetLine(t_lo, t_hi, 0)]

    @classmethod
    def from_lines(cls, tiles) -> "OffsetLineSet":
        """Skyline from (lo, hi, height) tiles that cover a span without gaps."""
        tiles = [tuple(int(x) for x in t) for t in tiles]
        if not tiles:
            raise ValueError("no lines")
        for (_, hi, _), (lo, _, _) in zip(tiles, tiles[1:]):
            if hi != lo:
                raise ValueError("lines must tile their span")
        s = cls.__new__(cls)
        s._lines = [OffsetLine(lo, hi, h) for lo, hi, h in tiles]
        return s

    # ---- views ----
    def lines(self) -> list:
        return list(self._lines)

    def as_tuples(self) -> list:
        return [(l.time_lo, l.time_hi, l.height) for l in self._lines]

    def _index(self, line: OffsetLine) -> int:
        for i, l in enumerate(self._lines):
            if l is line:
                return i
        raise ValueError(f"{line!r} is not part of this skyline")

    # ---- R3 ----
    def choose_offset(self) -> OffsetLine:
        return min(self._lines, key=lambda l: (l.height, l.time_lo))

    # ---- R5 ----
    def lift_up(self, line: OffsetLine) -> OffsetLine:
        c = self._index(line)
        L = self._lines
        has_p, has_n = c > 0, c + 1 < len(L)
        if not has_p and not has_n:
            raise IllegalLift("cannot lift the only offset line")
        hp = L[c - 1].height if has_p else None
        hn = L[c + 1].height if has_n else None
        if has_p and has_n and hp == hn:      # merge all three
            merged = OffsetLine(L[c - 1].time_lo, L[c + 1].time_hi, hp)
            L[c - 1:c + 2] = [merged]
        elif has_n and (not has_p or hn < hp):  # into the next (lower) line
            merged = OffsetLine(line.time_lo, L[c + 1].time_hi, hn)
            L[c:c + 2] = [merged]
        else:                                 # into the previous (lower) line
            merged = OffsetLine(L[c - 1].time_lo, line.time_hi, hp)
            L[c - 1:c + 1] = [merged]
        return merged

    # ---- R6 ----
    def place(self, line: OffsetLine, block) -> int:
        c = self._index(line)
        a, f = block.alloc_time, block.free_time
        if not (line.time_lo <= a and f <= line.time_hi):
            raise ContainmentViolation(
                f"block {block.id} [{a}, {f}) does not fit line [{line.time_lo}, {line.time_hi})")
        h = line.height
        raised = OffsetLine(a, f, h + block.size)
        new = ([OffsetLine(line.time_lo, a, h)] if line.time_lo < a else []) + [raised] + \
              ([OffsetLine(f, line.time_hi, h)] if f < line.time_hi else [])
        L = self._lines
        L[c:c + 1] = new
        r = c + (1 if line.time_lo < a else 0)
        if r > 0 and L[r - 1].height == raised.height:       # re-merge with previous
            raised = OffsetLine(L[r - 1].time_lo, raised.time_hi, raised.height)
            L[r - 1:r + 1] = [raised]
            r -= 1
        if r + 1 < len(L) and L[r + 1].height == raised.height:  # then with next
            L[r:r + 2] = [OffsetLine(raised.time_lo, L[r + 1].time_hi, raised.height)]
        return h


def _key(b):
    """R4 selection key: longest lifetime, then larger size, then smaller id."""
    return (b.free_time - b.alloc_time, b.size, -b.id)


def find_block(line: OffsetLine, blocks):
    """The best block whose lifetime lies within the line (R4), or None."""
    fits = [b for b in blocks if line.time_lo <= b.alloc_time and b.free_time <= line.time_hi]
    return max(fits, key=_key) if fits else None


class _RemainingBlocks:
    """Unplaced blocks answering best-fit queries (the reference's window
    index, bestfit.py:223-273): `take_best(lo, hi)` returns the best block
    contained in [lo, hi) and removes it, or None."""

    def __init__(self, blocks):
        self._live = {b.id: b for b in blocks}

    def __len__(self) -> int:
        return len(self._live)

    def take_best(self, lo: int, hi: int):
        best = None
        for b in self._live.values():
            if lo <= b.alloc_time and b.free_time <= hi and (best is None or _key(b) > _key(best)):
                best = b
        if best is not None:
            del self._live[best.id]
        return best
