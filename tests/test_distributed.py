"""Multi-process (world size 2, gloo, CPU) tests of the column-sharded GEMM's host logic:
block-cyclic ownership, the A broadcast in k-chunks (contiguous transpose views, as NCCL
requires), the accumulator carry between chunks, and both all-gather branches that reassemble
C (in place into C for equal block widths, padded list otherwise).  The per-rank GEMM is
injected: the oracle (k_chunks = 1), or an exact FP64 product of small integers with the
FP32 carry (k_chunks > 1) -- partitioning and chunking must never change a result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from paper_1904_06376_b200.distributed import block_owner_layout, chunk_edges, gemm_colsharded, local_columns


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


def _exact_gemm(A, B, C, variant, flags=0, acc=None):
    """Exact product of small integers with the library's carry semantics: ACC_IN starts from
    acc, ACC_OUT stores the running sum to acc instead of C (exact, so chunking is invisible)."""
    Z = A.double() @ B.double()
    if flags & 1:
        Z = Z + acc.double()
    if flags & 2:
        acc.copy_(Z.float())
    else:
        C.copy_(Z.float())


def _worker(rank, world, port, m, n, k, sub_blocks, k_chunks, variant, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode == "oracle":
            A_np = synthetic.uniform(m, k, seed=1)
            B_np = synthetic.uniform(k, n, seed=2)
            fn = _oracle_gemm
        else:
            A_np = synthetic.small_ints(m, k, seed=1, bound=100)
            B_np = synthetic.small_ints(k, n, seed=2, bound=100)
            fn = _exact_gemm
        A = torch.from_numpy(A_np) if rank == 0 else torch.zeros((k, m), dtype=torch.float32).t()
        cols = local_columns(n, world, rank, sub_blocks)
        B_local = torch.from_numpy(np.asfortranarray(B_np[:, cols]))
        C = torch.full((n, m), float("nan"), dtype=torch.float32).t()      # column-major m x n
        gemm_colsharded(A, B_local, C, variant=variant, sub_blocks=sub_blocks, k_chunks=k_chunks, gemm_fn=fn)
        q.put((rank, C.numpy().copy(), A.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(m, n, k, sub_blocks, k_chunks, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, sub_blocks, k_chunks, 6, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("m,n,k,sub_blocks", [(40, 64, 24, 1), (33, 70, 17, 3), (40, 64, 24, 4)])
def test_colsharded_world2_matches_single_process(orc, m, n, k, sub_blocks):
    """(40, 64): equal block widths -> the in-place all_gather_into_tensor branch; (33, 70, S=3):
    ragged widths -> the padded list branch."""
    A = synthetic.uniform(m, k, seed=1)
    B = synthetic.uniform(k, n, seed=2)
    want = orc.gemm(A, B, variant=6)
    for rank, C, A_seen in _run(m, n, k, sub_blocks, 1, "oracle"):
        assert np.array_equal(A_seen, A), rank            # broadcast delivered A
        assert np.array_equal(C, want), rank              # all-gather assembled C


@pytest.mark.parametrize("m,n,k,sub_blocks,k_chunks", [(48, 64, 700, 2, 4), (30, 70, 300, 3, 4)])
def test_colsharded_world2_chunked_carry(m, n, k, sub_blocks, k_chunks):
    """A broadcast in k-chunks (edges at multiples of 128, deduplicated), the first sub-block's
    accumulator carried across them, the rest on the whole A: exact integer products must come
    out unchanged on every rank."""
    A = synthetic.small_ints(m, k, seed=1, bound=100).astype(np.float64)
    B = synthetic.small_ints(k, n, seed=2, bound=100).astype(np.float64)
    want = (A @ B).astype(np.float32)
    for rank, C, A_seen in _run(m, n, k, sub_blocks, k_chunks, "exact"):
        assert np.array_equal(A_seen, A.astype(np.float32)), rank
        assert np.array_equal(C, want), rank


def test_chunk_edges():
    """Interior edges are multiples of 128, strictly increasing (no empty chunk), cover [0, k]."""
    assert chunk_edges(300, 4) == [0, 128, 256, 300]          # 75 -> 128, 150 -> 256, 225 -> 256: deduplicated
    assert chunk_edges(1000, 1) == [0, 1000]
    assert chunk_edges(100, 4) == [0, 100]
    for k in (129, 700, 4096, 5000):
        for c in (2, 3, 8):
            e = chunk_edges(k, c)
            assert e[0] == 0 and e[-1] == k
            assert all(b > a for a, b in zip(e, e[1:]))
            assert all(x % 128 == 0 for x in e[1:-1])


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
