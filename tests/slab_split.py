"""Test-only host-side slab split for sharding the observation array along its LAST mode
(SURVEY.md §8(e)), the same slicing kg_design_create applies per rank:
rank g owns the contiguous slab [lo_g, hi_g) of mode d, i.e. rows lo_g..hi_g of
X_d, and the flat cells [cell_base_g, cell_base_g + n_g) of every n-array.

H is local (eta[..., slab] needs only the slab rows of X_d); G is a sum of
per-slab partials, so one p-sized all-reduce per gradient (plus scalar
all-reduces for the objective partials and max(v)) reproduces the
single-device maps.  torch.distributed provides the collectives (NCCL on GPUs,
gloo in the CPU tests)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    lo: int          # first owned index of the last mode
    hi: int          # one past the last owned index
    cell_base: int   # global flat index of the first local cell
    n_local: int     # local cells


def slab(extents, rank: int, world: int) -> Slab:
    """Contiguous near-even split of the last mode: [nd*r/W, nd*(r+1)/W)."""
    extents = list(extents)
    nd = extents[-1]
    if world > nd:
        raise ValueError("sharded design: fewer last-mode slices than ranks")
    lo, hi = nd * rank // world, nd * (rank + 1) // world
    inner = int(np.prod(extents[:-1])) if len(extents) > 1 else 1
    return Slab(rank, world, lo, hi, lo * inner, (hi - lo) * inner)


def shard_design(design, s: Slab):
    """Slice the last-mode factor of every component to the slab's rows."""
    return [[np.asfortranarray(x[s.lo:s.hi]) if j == len(comp) - 1 else x for j, x in enumerate(comp)]
            for comp in design]


def shard_array(a, s: Slab):
    """The rank's slab of an n-array (last mode)."""
    return np.asfortranarray(np.asarray(a)[..., s.lo:s.hi])
