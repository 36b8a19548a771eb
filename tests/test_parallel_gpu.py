"""(e) C4 sharded end to end on the GPU: two ranks (gloo, host-staged gather buffers)
both on cuda:0 each compute their LPT share of output panels through the masked grouped
launch, pack with tnb_copy2d_batched, all-gather, unpack; the assembled output must
equal the single-rank contract_pair. The ranks' kernels never wait on one another
(the exchange is on the host), so sharing one GPU is safe."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2401_01921_b200 as tnb
        from paper_2401_01921_b200 import parallel
        errs = []
        for seed in (777, 1001):
            A, E = bench.c4_tensors(tnb, seed=seed)
            got = parallel.contract_sharded(A, E)
            want = tnb.contract_pair(A, E)
            assert got.labels == want.labels and got._qns == want._qns
            for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
                g, w = gb.numpy(), wb.numpy()
                errs.append(float(np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-300)))
        # repeated call: cached shard plan, same bits
        again = parallel.contract_sharded(A, E)
        same = all(np.array_equal(x.numpy(), y.numpy()) for x, y in zip(again.get_blocks_(), got.get_blocks_()))
        q.put((rank, max(errs), same, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_contract_sharded_two_ranks_matches_contract_pair(cuda):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, same, exc in res:
        assert exc is None, (rank, exc)
        assert err <= 1e-13, (rank, err)
        assert same, rank
