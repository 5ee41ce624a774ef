"""Oracle: sample-to-ensemble chunking (TEST INFRA ONLY).

Restates ``grouping.py:83-122`` of the reference: ``group_natural`` chunks in
generation order; ``group_by_key`` sorts by ascending key, stable in generation
order (``np.argsort(kind="stable")``, ``grouping.py:121``), then chunks; a short
last chunk is padded by replicating its own last real sample
(``grouping.py:91-92``).  Returns plain tuples ``(ensembles, padding)``.
"""

from __future__ import annotations

import numpy as np


def chunk(ordered, size):
    if size < 1:
        raise ValueError("ensemble size must be >= 1")
    groups, pads = [], []
    for lo in range(0, len(ordered), size):
        g = list(ordered[lo:lo + size])
        short = size - len(g)
        g += [g[-1]] * short
        groups.append(tuple(g))
        pads.append(short)
    return tuple(groups), tuple(pads)


def natural(ids, size):
    if not ids:
        raise ValueError("empty sample set")
    return chunk(list(ids), size)


def by_key(ids, keys, size):
    if not ids:
        raise ValueError("empty sample set")
    k = np.array([float(keys[i]) for i in ids])
    if not np.all(np.isfinite(k)):
        raise ValueError("keys must be finite")
    order = sorted(range(len(ids)), key=lambda j: (k[j], j))  # stable ascending
    return chunk([ids[j] for j in order], size)
