"""Multi-rank NESA product on CPU: partition, halo exchange, gloo.

The exchange code (paper_1801_03589_b200.dist.exchange_s) is the one the GPU
ranks run over NCCL; here each rank's kernels are emulated in numpy
(tests/dist_emulator.py) and the union of the partitioned outputs must equal
the single-device oracle product.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_03589_b200 import geometry as geo
from paper_1801_03589_b200.dist import (build_exchange, exchange_s, leaf_costs, local_ranges,
                                        partition_leaves)
from paper_1801_03589_b200.operators import NesaParams, build_all
from paper_1801_03589_b200.quadtree import TreeParams, build_tree


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=6000, P=24, Q=12, kind="ellipse-plates", seed=7):
    pts = geo.generate_sources(geo.CurveSpec(kind=kind, seed=seed), n)
    tree = build_tree(pts, TreeParams(P=P))
    ops = build_all(tree, NesaParams(Q=Q))
    q = geo.random_rhs(n, seed)
    return tree, ops, q


def _worker(rank, world, port, n, P, Q, kind, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from dist_emulator import stage1, stage2
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, ops, q = _problem(n, P, Q, kind)
        ranges = partition_leaves(tree, world, Q)
        xp = build_exchange(tree, ranges, rank)
        s = stage1(tree, ops, q, ranges[rank])
        st = torch.view_as_real(torch.from_numpy(s)).reshape(s.shape[0], -1).contiguous()
        exchange_s(st, xp)
        s2 = torch.view_as_complex(st.reshape(s.shape[0], s.shape[1], 2)).numpy()
        phi = stage2(tree, ops, q, ranges[rank], s2)
        pr = torch.view_as_real(torch.from_numpy(phi)).contiguous()
        dist.all_reduce(pr)
        if rank == 0:
            np.save(out, torch.view_as_complex(pr).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "ellipse-plates"), (3, "wave"), (4, "circle-random")])
def test_partitioned_product_matches_oracle(tmp_path, world, kind):
    from oracle.mvp_oracle import mvp_serial, rel_l2
    n, P, Q = 6000, 24, 12
    out = str(tmp_path / "phi.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, P, Q, kind, out), nprocs=world, join=True)
    tree, ops, q = _problem(n, P, Q, kind)
    ref = mvp_serial(tree, ops, q)
    assert rel_l2(np.load(out), ref) <= 1e-13


def test_partition_balanced_and_contiguous():
    tree, ops, q = _problem(20000, 32, 12)
    for world in (2, 4, 8):
        ranges = partition_leaves(tree, world, 12)
        assert ranges[0][0] == 0 and ranges[-1][1] == tree.n_leaves
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(ranges, ranges[1:]))
        c = leaf_costs(tree, 12)
        share = [c[b:e].sum() / c.sum() for b, e in ranges]
        assert max(share) <= 1.0 / world + c.max() / c.sum() + 1e-12


def test_local_ranges_are_ancestors():
    tree, ops, q = _problem(5000, 20, 10)
    ranges = partition_leaves(tree, 3, 10)
    a = tree.arrays
    for r in ranges:
        lr = local_ranges(tree, r)
        for leaf in range(*r):
            g = leaf
            while g >= 0:
                lo, hi = lr[int(a.level[g])]
                assert lo <= g <= hi
                g = int(a.parent[g])


def test_exchange_volume_small():
    # halo volume is a small fraction of G (<= 0.72 MB at 8 ranks)
    tree, ops, q = _problem(30000, 32, 12)
    for world in (2, 8):
        ranges = partition_leaves(tree, world, 12)
        for r in range(world):
            xp = build_exchange(tree, ranges, r)
            assert xp.export_ids.size < 0.2 * tree.arrays.n_groups


def _c4_exchange_worker(rank, world, port, out):
    # the halo exchange at the bench's own partition shape (C4: 2M points,
    # P = 64, Q = 64, 8 ranks): every rank holds random partial amplitudes
    # for its local groups (summing to a known total), runs the exchange over
    # gloo, and must end up with the full amplitude of every group its
    # translations read
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1801_03589_b200.dist import local_mask
        tree = _c4_tree()
        ranges = partition_leaves(tree, world, 64)
        xp = build_exchange(tree, ranges, rank)
        a = tree.arrays
        G = a.n_groups
        qr = 2
        rng = np.random.default_rng(11)
        total = rng.standard_normal((G, qr))
        masks = np.stack([local_mask(tree, r) for r in ranges])
        # partials: contributor k of group g holds total * w_k, sum_k w_k = 1
        w = np.where(masks, rng.random((world, G)) + 0.1, 0.0)
        w /= w.sum(axis=0, keepdims=True)
        s = torch.from_numpy(total * w[rank][:, None])
        exchange_s(s, xp)
        src = np.repeat(np.arange(G), np.diff(a.int_ptr))
        needed = np.unique(a.int_idx[masks[rank][src]])
        err = np.abs(s.numpy()[needed] - total[needed]).max()
        vol = xp.max_export * 64 * 2 * 4   # bytes per rank sent (Q = 64, complex64)
        res = torch.tensor([err, float(vol), float(xp.import_ids.size)], dtype=torch.float64)
        allr = [torch.zeros_like(res) for _ in range(world)]
        dist.all_gather(allr, res)
        if rank == 0:
            np.save(out, torch.stack(allr).numpy())
    finally:
        dist.destroy_process_group()


def _c4_tree():
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=3), 2_000_000)
    return build_tree(pts, TreeParams(P=64))


@pytest.mark.slow
def test_exchange_at_c4_partition_world8(tmp_path):
    world = 8
    out = str(tmp_path / "x.npy")
    mp.spawn(_c4_exchange_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r = np.load(out)
    assert (r[:, 0] <= 1e-12).all(), r[:, 0]        # every needed amplitude complete
    # well under a megabyte per rank per product (complex64, Q = 64)
    assert (r[:, 1] <= 2e6).all(), r[:, 1]
