"""Multi-rank host logic on CPU with gloo (world_size 2): LPT panel partition,
panel spans in the C ABI's order, and the all-gather that assembles a block-sparse
output slab from per-rank panels; sharding of independent units."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_01921_b200 import parallel as P


def test_lpt_is_deterministic_and_balanced():
    costs = [10, 7, 7, 3, 3, 2, 1, 1]
    owner = P.lpt_partition(costs, 3)
    assert owner == P.lpt_partition(costs, 3)
    loads = [sum(c for c, o in zip(costs, owner) if o == p) for p in range(3)]
    assert max(loads) - min(loads) <= max(costs)
    assert P.lpt_partition([5], 4) == [0]


def test_panels_follow_abi_order():
    panels = P.panels_of([(1, 1), (130, 7), (64, 3)], 1)
    assert [(o, r0, r1) for o, r0, r1, _, _ in panels] == [(0, 0, 1), (1, 0, 64), (1, 64, 128), (1, 128, 130),
                                                          (2, 0, 64)]
    assert P.panel_spans(panels, [0, 8, 1000])[2] == (8 + 64 * 7, 64 * 7)


def test_shard_covers_each_unit_once():
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i in P.shard(64, world, r))
        assert got == list(range(64))


def test_block_pair_k_c4():
    from paper_2401_01921_b200.workloads import c4_sectors
    import tnkit_np as oracle
    sec = c4_sectors()
    qv = [(q,) for q, _ in sec]
    deg = [d for _, d in sec]
    a_qns = oracle.zero_flux_combos([(1, qv, [0]), (1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    e_qns = oracle.zero_flux_combos([(1, qv, [0]), (-1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    out_qns = oracle.zero_flux_combos([(1, qv, [0]), (-1, qv, [0])])
    a_shapes = [(deg[q[0]], 1, deg[q[2]]) for q in a_qns]
    kt = P.block_pair_k(a_qns, a_shapes, [1, 2], e_qns, [1, 0], [0], [2], out_qns)
    e_shapes = [(deg[q[0]], 1, deg[q[2]]) for q in e_qns]
    macs = sum(k * deg[q[0]] * deg[q[1]] for k, q in zip(kt, out_qns))
    assert macs == 169073208


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shapes = [(1, 1), (130, 7), (64, 3), (3, 3), (200, 5)]
        ktot = [1, 40, 9, 0, 77]
        panels, owner = P.panel_plan(shapes, 1, ktot, world)
        sizes = [r * c for r, c in shapes]
        offs = list(np.cumsum([0] + [((s + 7) // 8) * 8 for s in sizes])[:-1])
        total = int(offs[-1] + sizes[-1])
        full = torch.arange(total, dtype=torch.float64) * 0.5 + 1.0
        slab = torch.full((total,), -7.0, dtype=torch.float64)
        spans = P.panel_spans(panels, offs)
        for (s, n), o in zip(spans, owner):
            if o == rank:
                slab[s:s + n] = full[s:s + n]
        P.gather_panels(slab, spans, owner, rank, world)
        covered = torch.zeros(total, dtype=torch.bool)
        for s, n in spans:
            covered[s:s + n] = True
        ok = bool(torch.equal(slab[covered], full[covered]))
        q.put((rank, ok, owner))
    finally:
        dist.destroy_process_group()


def test_gather_panels_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    owners = [o for _, _, o in res]
    assert owners[0] == owners[1] and set(owners[0]) == {0, 1}
