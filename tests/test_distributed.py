"""Multi-process (world size 2, gloo, CPU) tests of the column-sharded GEMM's host logic:
block-cyclic ownership, the A broadcast and the all-gather that reassembles C.  The per-rank
GEMM is the oracle (injected), so every rank's assembled C must equal the single-process
oracle product bit for bit -- partitioning never changes per-element arithmetic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from paper_1904_06376_b200.distributed import block_owner_layout, gemm_colsharded, local_columns


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_gemm(A, B, C, variant, flags=0, acc=None):
    import oracle
    assert flags == 0
    C.copy_(torch.from_numpy(oracle.gemm(A.numpy(), B.numpy(), variant=variant)))


def _worker(rank, world, port, m, n, k, sub_blocks, variant, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A_np = synthetic.uniform(m, k, seed=1)
        B_np = synthetic.uniform(k, n, seed=2)
        A = torch.from_numpy(A_np) if rank == 0 else torch.zeros((k, m), dtype=torch.float32).t()
        cols = local_columns(n, world, rank, sub_blocks)
        B_local = torch.from_numpy(np.asfortranarray(B_np[:, cols]))
        C = torch.full((n, m), float("nan"), dtype=torch.float32).t()      # column-major m x n
        gemm_colsharded(A, B_local, C, variant=variant, sub_blocks=sub_blocks, gemm_fn=_oracle_gemm)
        q.put((rank, C.numpy().copy(), A.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,sub_blocks", [(40, 64, 24, 1), (33, 70, 17, 3)])
def test_colsharded_world2_matches_single_process(orc, m, n, k, sub_blocks):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, sub_blocks, 6, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synthetic.uniform(m, k, seed=1)
    B = synthetic.uniform(k, n, seed=2)
    want = orc.gemm(A, B, variant=6)
    for rank, C, A_seen in results:
        assert np.array_equal(A_seen, A), rank            # broadcast delivered A
        assert np.array_equal(C, want), rank              # all-gather assembled C


def test_block_cyclic_layout():
    lay = block_owner_layout(100, 4, 3)
    # sub-round s covers a contiguous range, ranks in order, widths differ by <= 1
    flat = [blk for s in lay for blk in s]
    assert flat[0][0] == 0 and sum(w for _, w in flat) == 100
    for a, b in zip(flat, flat[1:]):
        assert a[0] + a[1] == b[0]
    widths = [w for _, w in flat]
    assert max(widths) - min(widths) <= 1
    cols = [c for r in range(4) for c in local_columns(100, 4, r, 3)]
    assert sorted(cols) == list(range(100))
