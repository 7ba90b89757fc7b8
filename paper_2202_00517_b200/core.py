"""Domain types of the drop-in API — mirrors rankdescent.core (core.py:23-113).

Only the parts the hot path's boundary needs: the error type, the dataset
wrapper and the ranking-system ABCs whose ``(score, id)`` total order the
device kernels implement.
"""

from __future__ import annotations

from abc import ABC, abstractmethod
from typing import Generic, Iterable, Iterator, Mapping, Sequence, TypeVar

import numpy as np

T = TypeVar("T")
ItemId = int


class ConfigError(ValueError):
    """A run parameter violates a structural precondition (core.py:23-24)."""


class Dataset(Generic[T]):
    """Indexed, immutable collection of n >= 2 items (core.py:27-59)."""

    def __init__(self, items: Sequence[T]):
        if len(items) < 2:
            raise ConfigError(f"a dataset needs at least 2 items, got {len(items)}")
        self._items = items

    @property
    def items(self) -> Sequence[T]:
        return self._items

    @property
    def n(self) -> int:
        return len(self._items)

    def __len__(self) -> int:
        return len(self._items)

    def __getitem__(self, i: int) -> T:
        return self._items[i]

    def __iter__(self) -> Iterator[T]:
        return iter(self._items)

    def __repr__(self) -> str:
        return f"Dataset(n={self.n})"


class RankingSystem(ABC):
    """Per-anchor strict total order over the other items (core.py:62-81)."""

    @abstractmethod
    def compare(self, x: ItemId, y: ItemId, z: ItemId) -> int:
        """Negative iff y ranks before z from x's viewpoint."""

    def comparator_for(self, x: ItemId):
        return lambda y, z: self.compare(x, y, z)


class ScoredRankingSystem(RankingSystem):
    """Order by ``(score(x, y), y)`` ascending (core.py:83-113)."""

    @property
    @abstractmethod
    def size(self) -> int: ...

    @abstractmethod
    def batch_scores(self, x: ItemId, ids: np.ndarray | None = None) -> np.ndarray: ...

    def score(self, x: ItemId, y: ItemId) -> float:
        return float(self.batch_scores(x, np.array([y], dtype=np.int64))[0])

    def compare(self, x: ItemId, y: ItemId, z: ItemId) -> int:
        if x == y or x == z or y == z:
            raise ValueError(f"compare needs pairwise distinct ids, got ({x}, {y}, {z})")
        return -1 if (self.score(x, y), y) < (self.score(x, z), z) else 1


def build_cofriends(friends: Mapping[ItemId, Iterable[ItemId]]) -> dict[ItemId, set[ItemId]]:
    """core.py:196-206 — transpose a friends digraph given as a mapping: y in
    friends[x] iff x in cofriends[y]; every input key appears, possibly empty.
    (The device path builds the same transpose as a CSR, knnd_csr_build.)"""
    cofriends: dict[ItemId, set[ItemId]] = {x: set() for x in friends}
    for x, targets in friends.items():
        for y in targets:
            cofriends.setdefault(y, set()).add(x)
    return cofriends


def verify_total_order(rs: RankingSystem, anchor: ItemId, ids: Sequence[ItemId]) -> bool:
    """core.py:209-235 — exhaustive anti-symmetry and transitivity check of the
    anchor's order over `ids` (O(m^3); a desk-scale diagnostic)."""
    others = [i for i in ids if i != anchor]
    for y in others:
        for z in others:
            if y < z and (rs.compare(anchor, y, z) < 0) == (rs.compare(anchor, z, y) < 0):
                return False
    for y in others:
        for z in others:
            for w in others:
                if len({y, z, w}) == 3 and rs.compare(anchor, y, z) < 0 and rs.compare(anchor, z, w) < 0 \
                        and not rs.compare(anchor, y, w) < 0:
                    return False
    return True
