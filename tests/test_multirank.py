"""Multi-rank (N > 1) logic on CPU with torch.distributed/gloo, world_size 2.

Covers the sharding plan of the path (paper_0910_5863_b200/shard.py: block
partition, pair ownership, interface halo exchange, owned-dof dot products,
root sums) against the single-process oracle, checks that the sharded
engine's own halo plan (C++ host layer, bddc_b200_halo_plan) is the same plan,
and bench.py's multi-rank harness (barrier, max over ranks).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0910_5863_b200 import shard


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_shapes():
    assert shard.process_grid((12, 12, 12), 8) == (2, 2, 2)
    own = shard.partition((12, 12, 12), 8)
    assert np.all(np.bincount(own) == 216)  # 6^3 subdomains per GPU
    own = shard.partition((6, 6, 6), 8)
    assert np.all(np.bincount(own) == 27)
    own = shard.partition((8, 8, 8), 4)
    assert np.all(np.bincount(own) == 128)
    own = shard.partition((3, 3, 3), 2)
    assert sorted(np.bincount(own)) in ([9, 18], [12, 15], [13, 14])
    # blocks are contiguous boxes: every rank's subdomains form one lattice box
    own = shard.partition((6, 4, 2), 4)
    for r in range(4):
        ids = np.nonzero(own == r)[0]
        i, j, k = ids % 6, (ids // 6) % 4, ids // 24
        assert len(ids) == (i.max() - i.min() + 1) * (j.max() - j.min() + 1) * (k.max() - k.min() + 1)


def _subdomain_contribution(itf, s, x):
    """InterfaceProblem::apply (schur.cpp:12-36) restricted to substructure s."""
    sys = itf.systems[s]
    h = itf.h
    out = np.zeros(itf.size)
    xl = np.zeros(sys.dim)
    bnd, inn = h.boundary[s], h.interior[s]
    xl[bnd] = x[itf.bidx[s]]
    if len(inn):
        xl[inn] = h.interior_solve(s, -(h.coupling[s] @ xl[bnd]))
    y = sys.stiffness @ xl
    np.add.at(out, itf.bidx[s], y[bnd])
    return out


def _worker(rank, world, port, errors):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import fem
        from oracle.adaptive import face_pairs
        from oracle.experiment import build_pipeline, cube_spec
        from oracle.spaces import HarmonicExtension, InterfaceProblem
        sub = (3, 2, 2)
        p = build_pipeline(cube_spec(sub, 3, fem.SCALAR))
        h = HarmonicExtension(p.systems, p.maps)
        itf = InterfaceProblem(p.systems, p.maps, h)
        owner = shard.partition(sub, world)
        copy_ranks = [[int(owner[s]) for s, _ in p.maps.dof_copies[g]] for g in p.maps.interface_dofs]
        plan = shard.HaloPlan.build(rank, copy_ranks)
        # the sharded engine's own plan (C++ host layer, through the ABI) is the same
        import paper_0910_5863_b200 as pb
        cplan = pb.BDDC(pb.Problem.cube(sub, 3, "scalar")).halo_plan(owner, rank, world)
        assert np.array_equal(np.nonzero(cplan["touched"])[0], plan.local_iface)
        assert np.array_equal(cplan["owned"][plan.local_iface], plan.owned)
        assert cplan["peers"] == plan.peers
        for r in plan.peers:
            assert np.array_equal(cplan["shared"][r], plan.local_iface[plan.shared[r]])
        x = np.random.default_rng(7).standard_normal(itf.size)
        # each rank applies only its substructures, then the halo exchange sums copies
        part = np.zeros(itf.size)
        for s in np.nonzero(owner == rank)[0]:
            part += _subdomain_contribution(itf, int(s), x)
        local = torch.from_numpy(part[plan.local_iface].copy())
        plan.exchange(local, dist)
        ref = itf.apply(x)
        got = local.numpy()
        assert np.allclose(got, ref[plan.local_iface], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        # shared dofs are bitwise identical on both ranks after the exchange
        sums = torch.from_numpy(np.zeros(itf.size))
        sums[torch.from_numpy(plan.local_iface)] = local
        other = sums.clone()
        dist.all_reduce(other, op=dist.ReduceOp.MAX)
        mine = sums.clone()
        dist.all_reduce(mine, op=dist.ReduceOp.MIN)
        for r, idx in plan.shared.items():
            g = plan.local_iface[idx]
            assert torch.equal(other[g], mine[g])
        # owned-dof dot product equals the global one
        xl = torch.from_numpy(x[plan.local_iface].copy())
        d = plan.owned_dot(local, xl, dist)
        assert abs(d - float(ref @ x)) <= 1e-12 * abs(float(ref @ x))
        # every face pair has exactly one owner rank
        pairs = face_pairs(p.globset)
        po = shard.pair_owner(pairs, owner)
        mine_pairs = torch.tensor([int(np.sum(po == rank))], dtype=torch.int64)
        dist.all_reduce(mine_pairs)
        assert int(mine_pairs.item()) == len(pairs)
        # root sum: per-rank coarse contributions (corner-dof incidence) add to the global count
        root = np.zeros(p.maps.corner_dof_count)
        for s in np.nonzero(owner == rank)[0]:
            for l, cid in enumerate(p.maps.local_to_wc[int(s)]):
                if p.maps.local_is_corner[int(s)][l]:
                    root[cid] += 1.0
        rt = shard.root_sum(torch.from_numpy(root), dist)
        glob = np.zeros(p.maps.corner_dof_count)
        for s in range(len(p.systems)):
            for l, cid in enumerate(p.maps.local_to_wc[s]):
                if p.maps.local_is_corner[s][l]:
                    glob[cid] += 1.0
        assert np.array_equal(rt.numpy(), glob)
        # distributed primal tree: this rank's fronts and the
        # other rank's partition the primal unknowns outside the top front, the
        # top front is the same list on both ranks and equals the single plan's
        tb = pb.BDDC(pb.Problem.cube((4, 2, 2), 3, "scalar"))
        tb.arithmetic_constraints(True, True)
        town = shard.partition((4, 2, 2), world)
        single = tb.primal_tree_plan(town, 0, 1, 1)
        tplan = tb.primal_tree_plan(town, rank, world, 1)
        assert tplan["depth"] == 1 and np.array_equal(tplan["top"], single["top"])
        n_primal = len(single["top"]) + sum(len(o) for _, o in single["fronts"])
        mine = np.zeros(n_primal)
        for _, o in tplan["fronts"]:
            mine[o] += 1.0
        both = torch.from_numpy(mine.copy())
        dist.all_reduce(both)
        expect = np.ones(n_primal)
        expect[single["top"]] = 0.0
        assert np.array_equal(both.numpy(), expect)  # every eliminated unknown on exactly one rank
        assert mine.sum() > 0 and mine.sum() < expect.sum()
        # bench.py's multi-rank harness
        import bench
        bench.barrier(dist)
        assert bench.max_over_ranks(dist, float(rank + 1)) == float(world)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errors.put("rank %d: %s\n%s" % (rank, e, traceback.format_exc()))


def test_sharded_interface_operations_gloo():
    ctx = mp.get_context("spawn")
    errors = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errors)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    msgs = []
    while not errors.empty():
        msgs.append(errors.get())
    assert not msgs, "\n".join(msgs)
    assert all(pr.exitcode == 0 for pr in procs)


@pytest.mark.parametrize("sub,world,depth", [((4, 4, 4), 2, 2), ((4, 4, 4), 4, 2), ((4, 4, 4), 8, 2),
                                              ((3, 3, 3), 2, 1), ((6, 6, 6), 8, 2), ((6, 4, 2), 4, 1)])
def test_distributed_primal_tree_plan(sub, world, depth):
    """Every rank plans the boxes of the primal tree from the unknowns' global
    bounds and keeps the fronts inside its own block: together the ranks hold
    exactly the single-GPU plan's fronts (same unknowns per front, each on one
    rank, every front inside its owner's block), and all share its top front."""
    import paper_0910_5863_b200 as pb
    b = pb.BDDC(pb.Problem.cube(sub, 2, "scalar"))
    b.arithmetic_constraints(True, True)
    owner = shard.partition(sub, world)
    single = b.primal_tree_plan(owner, 0, 1, depth)
    assert single["depth"] == depth
    want = sorted((lvl, tuple(o)) for lvl, o in single["fronts"] if len(o))
    got = []
    for r in range(world):
        p = b.primal_tree_plan(owner, r, world, depth)
        assert p["depth"] == depth and np.array_equal(p["top"], single["top"])
        got += [(lvl, tuple(o)) for lvl, o in p["fronts"] if len(o)]
    assert sorted(got) == want


def test_misaligned_partition_keeps_dense_root():
    """A partition whose blocks cut through the depth-1 boxes (three ranks along
    x on a lattice the boxes halve) falls back to depth 0 on every rank."""
    import paper_0910_5863_b200 as pb
    b = pb.BDDC(pb.Problem.cube((6, 2, 2), 2, "scalar"))
    b.arithmetic_constraints(True, True)
    owner = shard.partition((6, 2, 2), 3)
    for r in range(3):
        p = b.primal_tree_plan(owner, r, 3, 2)
        assert p["depth"] == 0 and not p["fronts"]
