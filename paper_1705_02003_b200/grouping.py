"""Drop-in for ``uqgroup.grouping``'s plan construction, with the sort on the GPU.

* ``GroupingPlan``  <- ``grouping.py:39-80`` (same fields, same validation);
* ``group_natural`` <- ``grouping.py:98-102``;
* ``group_by_key``  <- ``grouping.py:105-122``: the stable ascending key sort
  and the width-S chunking with last-group replica padding run on the device
  (``uqg_group_sort``: a stable LSD radix sort of order-preserving 64-bit key
  images, O(n) per level); sample ids may be any hashable objects, the device
  works on their generation-order indices.

The reference's post-hoc accounting is not on the hot path: ``compute_R``
(``grouping.py:156-193``) is restated in ``report.py`` for the run files
(``r_table.csv``); ``group_oracle`` and ``predicted_speedup``
(``grouping.py:125-154,196-204``) are not rebuilt.
The reference's own functions accept these plans unchanged
(``tests/test_ref_conformance.py``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from .errors import GroupingError

__all__ = ["GroupingError", "GroupingPlan", "group_natural", "group_by_key", "device_group"]


@dataclass(frozen=True)
class GroupingPlan:
    level: int
    ensemble_size: int
    ensembles: tuple
    padding: tuple
    strategy_tag: str

    def __post_init__(self) -> None:
        S = self.ensemble_size
        if S < 1:
            raise GroupingError(f"ensemble size must be >= 1, got {S}")
        if len(self.padding) != len(self.ensembles):
            raise GroupingError("padding must give one count per ensemble")
        last = len(self.ensembles) - 1
        for k, (grp, pad) in enumerate(zip(self.ensembles, self.padding)):
            if len(grp) != S:
                raise GroupingError(f"group {k} has {len(grp)} slots, expected {S}")
            if pad and k != last:
                raise GroupingError("only the last group may be padded")
            if not 0 <= pad < S:
                raise GroupingError(f"invalid padding count {pad}")
            if pad and any(x != grp[S - pad - 1] for x in grp[S - pad:]):
                raise GroupingError("padding must replicate the last real sample")

    @property
    def n_samples(self) -> int:
        return self.ensemble_size * len(self.ensembles) - sum(self.padding)

    def sample_ids(self) -> list:
        out = []
        for grp, pad in zip(self.ensembles, self.padding):
            out.extend(grp[: self.ensemble_size - pad])
        return out


def device_group(n: int, size: int, d_keys=None, sync: bool = True):
    """Device sort + chunk of n generation-order indices.

    Returns device int32 tensors (groups [K*size], padding [K]); ``d_keys``
    (float64 device tensor [n]) or None for natural order.  ``sync=False``
    (the level pipeline) never waits for the device: a non-finite key sets
    status bit 1, which the caller's next status check turns into
    ``GroupingError``.
    """
    if size < 1:
        raise GroupingError(f"ensemble size must be >= 1, got {size}")
    if n < 1:
        raise GroupingError("cannot group an empty sample set")
    torch = _lib._torch()
    K = (n + size - 1) // size
    groups = torch.empty((K * size,), dtype=torch.int32, device=_lib.device())
    pad = torch.empty((K,), dtype=torch.int32, device=_lib.device())
    _lib.call("uqg_group_sort" if sync else "uqg_group_sort_async", _lib.ctx(), _lib.ptr(d_keys),
              n, size, None, _lib.ptr(groups), _lib.ptr(pad), _lib.stream(),
              invalid=GroupingError)
    return groups, pad


def _plan(ids, groups, pad, size, level, tag) -> GroupingPlan:
    g = groups.cpu().numpy().reshape(-1, size)
    ens = tuple(tuple(ids[int(j)] for j in row) for row in g)
    return GroupingPlan(level, size, ens, tuple(int(p) for p in pad.cpu().numpy()), tag)


def group_natural(ids: Sequence, size: int, level: int = 0, tag: str = "nat") -> GroupingPlan:
    ids = list(ids)
    if not ids:
        raise GroupingError("cannot group an empty sample set")
    groups, pad = device_group(len(ids), size)
    return _plan(ids, groups, pad, size, level, tag)


def group_by_key(ids: Sequence, keys: Mapping, size: int, level: int = 0, tag: str = "sur"
                 ) -> GroupingPlan:
    ids = list(ids)
    if not ids:
        raise GroupingError("cannot group an empty sample set")
    try:
        karr = np.array([float(keys[i]) for i in ids], dtype=np.float64)
    except KeyError as err:
        raise GroupingError(f"no key supplied for sample {err.args[0]}") from None
    if size < 1:
        raise GroupingError(f"ensemble size must be >= 1, got {size}")
    groups, pad = device_group(len(ids), size, _lib.to_dev(karr))
    return _plan(ids, groups, pad, size, level, tag)
