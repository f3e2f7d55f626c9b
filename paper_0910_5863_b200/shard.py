"""Sharding plan of the adaptive-BDDC hot path over ranks (one GPU per rank).

The path shards by substructure and by face pair:
  * substructures: 3D block partition of the subdomain lattice (`partition`,
    used by the engine's owner map in bench.py and the tests);
  * face pairs: owned by the rank of the lower-numbered substructure
    (`pair_owner`); the neighbours they need (ghosts) receive their Schur
    complements from the owning rank;
  * interface vectors: every rank holds the interface dofs its substructures
    touch; after the per-substructure work the copies shared with other ranks
    are summed by a point-to-point halo exchange, contributions added in
    ascending rank order;
  * dot products: each interface dof is owned by exactly one rank (the lowest
    rank holding a copy); local sums are all-reduced;
  * primal tree: every rank factors the nested-dissection boxes inside its own
    block; only the top front (the unknowns shared between the depth-1 boxes)
    is summed over the ranks by an all-reduce (engine.cu, coarse_tree.hpp).
The device engine implements this plan in C++ (host.cpp `halo_plan`,
engine.cu `halo_exchange` over NCCL send/recv); `HaloPlan` below is the same
plan restated in Python with torch.distributed, the checker of the engine's
plan in the world_size-2 gloo test (tests/test_multirank.py).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np


def process_grid(sub_axes: Sequence[int], world: int) -> Tuple[int, int, int]:
    """Factor `world` into a 3D process grid that divides the lattice as evenly
    as possible and minimizes the cut surface (ties: larger splits on x)."""
    best = None
    for px in range(1, world + 1):
        if world % px:
            continue
        for py in range(1, world // px + 1):
            if (world // px) % py:
                continue
            pz = world // (px * py)
            if px > sub_axes[0] or py > sub_axes[1] or pz > sub_axes[2]:
                continue
            blocks = [(-(-sub_axes[a] // g)) for a, g in zip(range(3), (px, py, pz))]
            imbalance = np.prod(blocks) * world / np.prod(sub_axes)
            surface = ((px - 1) * sub_axes[1] * sub_axes[2] + (py - 1) * sub_axes[0] * sub_axes[2] +
                       (pz - 1) * sub_axes[0] * sub_axes[1])
            key = (imbalance, surface, -px, -py)
            if best is None or key < best[0]:
                best = (key, (px, py, pz))
    if best is None:
        raise ValueError("cannot partition %s subdomains over %d ranks" % (tuple(sub_axes), world))
    return best[1]


def partition(sub_axes: Sequence[int], world: int) -> np.ndarray:
    """Rank of every subdomain (x-fastest numbering, mesh.cpp:68-70)."""
    px, py, pz = process_grid(sub_axes, world)
    nx, ny, nz = sub_axes
    owner = np.empty(nx * ny * nz, dtype=np.int64)
    for k, j, i in itertools.product(range(nz), range(ny), range(nx)):
        bi, bj, bk = i * px // nx, j * py // ny, k * pz // nz
        owner[(k * ny + j) * nx + i] = (bk * py + bj) * px + bi
    return owner


def pair_owner(pairs: Sequence[Tuple[int, int]], owner: np.ndarray) -> np.ndarray:
    """Face pairs (adaptive.cpp:12-20) go to the rank of the lower subdomain."""
    return np.array([owner[min(si, sj)] for si, sj in pairs], dtype=np.int64)


@dataclass
class HaloPlan:
    """Interface-dof bookkeeping of one rank.

    `local_iface` lists the global interface indices this rank touches
    (ascending); `owned` marks the ones it owns (lowest copy rank);
    `send[peer]`/`recv[peer]` are positions in `local_iface` exchanged with
    `peer` (identical index lists on both sides, so the exchange is symmetric).
    """
    rank: int
    local_iface: np.ndarray
    owned: np.ndarray
    peers: List[int] = field(default_factory=list)
    shared: Dict[int, np.ndarray] = field(default_factory=dict)

    @staticmethod
    def build(rank: int, copy_ranks: Sequence[Sequence[int]]) -> "HaloPlan":
        """copy_ranks[i] = ranks holding a copy of interface dof i (any order)."""
        local = [i for i, rs in enumerate(copy_ranks) if rank in rs]
        local_arr = np.array(local, dtype=np.int64)
        pos = {g: t for t, g in enumerate(local)}
        owned = np.array([min(copy_ranks[g]) == rank for g in local], dtype=bool)
        shared: Dict[int, List[int]] = {}
        for g in local:
            for r in sorted(set(copy_ranks[g])):
                if r != rank:
                    shared.setdefault(r, []).append(pos[g])
        plan = HaloPlan(rank, local_arr, owned)
        plan.peers = sorted(shared)
        plan.shared = {r: np.array(v, dtype=np.int64) for r, v in shared.items()}
        return plan

    def exchange(self, partial, dist):
        """Sum the copies of shared interface dofs across ranks (in place).

        `partial` is a float64 torch tensor over `local_iface`.  Peer sums are
        added in ascending rank order on every rank, so all copies of a dof end
        bitwise identical."""
        import torch
        incoming = {}
        reqs = []
        for r in self.peers:
            idx = torch.from_numpy(self.shared[r])
            out = partial.index_select(0, idx).contiguous()
            inc = torch.empty_like(out)
            reqs.append(dist.isend(out, r))
            reqs.append(dist.irecv(inc, r))
            incoming[r] = (idx, out, inc)
        for q in reqs:
            q.wait()
        # zero-padded contributions added in ascending rank order: x + 0.0 == x,
        # so every dof gets exactly the ordered sum over the ranks holding it
        total = torch.zeros_like(partial)
        for r in sorted(self.peers + [self.rank]):
            if r == self.rank:
                total += partial
            else:
                idx, _, inc = incoming[r]
                padded = torch.zeros_like(partial)
                padded.index_copy_(0, idx, inc)
                total += padded
        partial.copy_(total)
        return partial

    def owned_dot(self, a, b, dist) -> float:
        """Global dot product of two interface vectors (local views)."""
        import torch
        m = torch.from_numpy(self.owned)
        s = torch.sum(a[m] * b[m]).reshape(1).to(torch.float64)
        dist.all_reduce(s)
        return float(s.item())


def root_sum(local_root, dist):
    """Sum of the ranks' leaf contributions to the root (matrix or vector)."""
    dist.all_reduce(local_root)
    return local_root
