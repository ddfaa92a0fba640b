"""The column-sharded GEMM (paper_1904_06376_b200.distributed) on the GPU with the
NCCL backend in a world of one process: the k-chunked A path (FP32 promoted accumulator
carried between chunks through bf16x_gemm_ex ACC_IN / ACC_OUT) and the sub-block loop run on
the CUDA library exactly as on every rank of a multi-GPU run, and must reproduce the one-call
GEMM bit for bit.  (The collectives themselves are exercised with gloo, world size 2, in
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
                                                        (2048, 2048, 2048, 4, 8)])
def test_colsharded_world1_bit_identical(nccl_world1, orc, m, n, k, sub_blocks, k_chunks, variant):
    A = synthetic.uniform(m, k, seed=m + k)
    B = synthetic.uniform(k, n, seed=n + k)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    want = bx.gemm(Ad, Bd, variant=variant).cpu().numpy()
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
