"""The column-sharded GEMM (paper_1904_06376_b200.distributed) on the GPU with the
NCCL backend in a world of one process: A split once into the piece buffer chunk by chunk, the
k-chunked first sub-block (FP32 promoted accumulator carried between chunks through
bf16x_gemm_ex ACC_IN / ACC_OUT) and the sub-block loop on the pre-split A run on the CUDA
library exactly as on every rank of a multi-GPU run, and must reproduce the one-call GEMM
(BF16X_NO_STREAM_K) bit for bit.  (The collectives themselves are exercised with gloo, world size 2, in
tests/test_distributed.py; more GPUs are not available to the test runs.)"""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1904_06376_b200 as bx
import synthetic
from paper_1904_06376_b200.distributed import gemm_colsharded, local_columns

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", [3, 6, 9])
@pytest.mark.parametrize("m,n,k,sub_blocks,k_chunks", [(512, 768, 1024, 1, 4), (1000, 1300, 700, 3, 3),
                                                        (2048, 2048, 2048, 4, 8), (4096, 4608, 1000, 2, 4),
                                                        (300, 400, 300, 2, 4)])
def test_colsharded_world1_bit_identical(nccl_world1, orc, m, n, k, sub_blocks, k_chunks, variant):
    A = synthetic.uniform(m, k, seed=m + k)
    B = synthetic.uniform(k, n, seed=n + k)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    want = bx.gemm(Ad, Bd, variant=variant, no_stream_k=True).cpu().numpy()
    cols = local_columns(n, 1, 0, sub_blocks)
    assert cols == list(range(n))
    C = torch.full((n, m), float("nan"), dtype=torch.float32, device="cuda").t()   # column-major
    gemm_colsharded(Ad, Bd, C, variant=variant, sub_blocks=sub_blocks, k_chunks=k_chunks)
    torch.cuda.synchronize()
    got = C.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # and the assembled product meets the oracle bar on sampled columns
    sc = np.linspace(0, n - 1, 8).astype(np.int64)
    C64 = orc.dgemm(A, B, cols=sc)
    eo = orc.normwise_error(orc.gemm(A, B, variant=variant, cols=sc), C64, A, B[:, sc])
    assert orc.normwise_error(got[:, sc], C64, A, B[:, sc]) <= 2.0 * eo


@pytest.mark.parametrize("P,sub_blocks", [(2, 2), (4, 2), (8, 2)])
def test_rank_shards_equal_one_gpu_columns(orc, P, sub_blocks):
    """Each rank's share of a P-GPU run (its block-cyclic columns, A split once into pieces,
    B_local's sub-blocks) computed here one rank after another on one GPU (no collectives):
    every shard must equal the same columns of the one-GPU call bit for bit, so the gathered C
    of a real P-GPU run is the one-GPU C.  4096 x 4608 x 1000 has 288 tiles: the one-GPU call
    would use stream-K without BF16X_NO_STREAM_K."""
    from paper_1904_06376_b200.distributed import _PieceGemm, block_owner_layout
    m, n, k = 4096, 4608, 1000
    A = synthetic.uniform(m, k, seed=3)
    B = synthetic.uniform(k, n, seed=4)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    want = bx.gemm(Ad, Bd, variant=6, no_stream_k=True).cpu().numpy()
    pg = _PieceGemm(Ad, 6)
    pg.split_chunk(Ad, 0, k)
    for q in range(P):
        cols = local_columns(n, P, q, sub_blocks)
        Bq = torch.from_numpy(np.asfortranarray(B[:, cols])).cuda()
        Cq = torch.empty_strided((m, len(cols)), (1, m), dtype=torch.float32, device="cuda")
        off = 0
        for owners in block_owner_layout(n, P, sub_blocks):
            w = owners[q][1]
            pg.gemm(0, k, Bq[:, off:off + w], Cq[:, off:off + w], 0)
            off += w
        torch.cuda.synchronize()
        assert np.array_equal(Cq.cpu().numpy().view(np.uint32), want[:, cols].view(np.uint32)), q


def _gloo_cuda_worker(rank, world, port, m, n, k, S, R, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A_np = synthetic.uniform(m, k, seed=1)
        B_np = synthetic.uniform(k, n, seed=2)
        A = torch.from_numpy(A_np).cuda() if rank == 0 else torch.zeros((k, m), device="cuda").t()
        cols = local_columns(n, world, rank, S)
        Bl = torch.from_numpy(np.asfortranarray(B_np[:, cols])).cuda()
        C = torch.full((n, m), float("nan"), device="cuda").t()
        gemm_colsharded(A, Bl, C, variant=6, sub_blocks=S, k_chunks=R)
        torch.cuda.synchronize()
        want = bx.gemm(torch.from_numpy(A_np).cuda(), torch.from_numpy(B_np).cuda(), variant=6, no_stream_k=True)
        torch.cuda.synchronize()
        q.put((rank, bool(torch.equal(C.contiguous().view(torch.int32), want.contiguous().view(torch.int32))),
               bool(torch.equal(A.contiguous().view(torch.int32),
                                torch.from_numpy(A_np).cuda().contiguous().view(torch.int32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,S,R", [(1024, 2048, 1536, 2, 3), (700, 1300, 900, 3, 4)])
def test_colsharded_world2_on_one_gpu(m, n, k, S, R):
    """The whole N > 1 data plane with real CUDA kernels: two processes share cuda:0 under the
    gloo backend (CUDA tensors), so the side-stream broadcast of A's chunks (contiguous transpose
    views), the per-chunk events, the chunked carry, the per-rank piece buffer and both all-gather
    branches (in place for equal block widths, padded for 1300 columns in 6 blocks) run exactly
    as they would across GPUs.  Each rank's kernels are independent (no kernel waits on another
    rank), so sharing one GPU only serialises them.  Both ranks' C must equal the one-GPU C."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cuda_worker, args=(r, 2, port, m, n, k, S, R, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, c_ok, a_ok in res:
        assert a_ok, rank
        assert c_ok, rank
