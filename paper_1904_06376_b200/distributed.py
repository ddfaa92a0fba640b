"""Column-sharded multi-GPU split GEMM (north star: "partitioned across the 8 GPUs
of one box by output column blocks of C, with B sharded, A broadcast once and an NCCL
all-gather over NVLink only to reassemble C").

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.  Output columns
are independent, so the only exchanges are

  * broadcast of A (FP32, m x k) from `src`, sent as `k_chunks` contiguous column chunks
    A[:, Kc] (contiguous in column-major storage) so the first sub-block's GEMM can start on
    chunk c while chunk c+1 is in flight; the FP32 promoted accumulator is carried between
    chunks (bf16x_gemm_ex ACC_IN/ACC_OUT), which makes the chunked result bit-identical to a
    one-pass GEMM when chunk widths are multiples of the promotion interval (64 k by default, 128 k
    for the x1/x3 128-k tuning hook; chunk edges are aligned to 128);
  * one all-gather per sub-round of C's column blocks.  Ownership is block-cyclic: with P
    ranks and S sub-blocks of width w = n / (P*S), rank q owns blocks s*P + q, so sub-round s
    covers the contiguous column range [s*P*w, (s+1)*P*w) of C and the all-gather of C^T
    (row-major view of column-major C) writes straight into C -- no permute pass.  The
    all-gather of sub-round s runs on a side stream while sub-round s+1 computes.

There are no reductions: k is never split across GPUs.  `gemm_fn` is the per-rank GEMM
(default: the bf16x CUDA library); the CPU tests inject the oracle to exercise the partition
and collective logic with the gloo backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_owner_layout(n: int, world: int, sub_blocks: int):
    """Column ranges per (sub-round s, rank q): returns a list over s of lists over q of
    (start, width).  Widths differ by at most one column."""
    nb = world * sub_blocks
    edges = [(n * b) // nb for b in range(nb + 1)]
    return [[(edges[s * world + q], edges[s * world + q + 1] - edges[s * world + q]) for q in range(world)]
            for s in range(sub_blocks)]


def local_columns(n: int, world: int, rank: int, sub_blocks: int):
    """Global column indices owned by `rank`, in the order of its local B / C blocks."""
    cols = []
    for s in block_owner_layout(n, world, sub_blocks):
        st, w = s[rank]
        cols.extend(range(st, st + w))
    return cols


def _cuda_gemm(A, B, C, variant, flags=0, acc=None):
    """Per-rank split GEMM on column-major CUDA tensors (C = A B, or carry via flags)."""
    import paper_1904_06376_b200 as bx
    m, k = A.shape
    n = B.shape[1]
    bx.gemm_raw(m, n, k, 1.0, A.data_ptr(), max(1, A.stride(1) if k > 1 else m), B.data_ptr(),
                max(1, B.stride(1) if n > 1 else k), 0.0, C.data_ptr(), max(1, C.stride(1) if n > 1 else m),
                variant=variant, flags=flags, acc=None if acc is None else acc.data_ptr())


def gemm_colsharded(A: torch.Tensor, B_local: torch.Tensor, C: torch.Tensor, variant: int = 6,
                    group=None, src: int = 0, sub_blocks: int = 1, k_chunks: int = 1, gemm_fn=None):
    """C = A B with B's columns sharded over the ranks of `group`.

    A       : m x k FP32 column-major (valid on `src`; overwritten by the broadcast elsewhere)
    B_local : k x n_q FP32 column-major, this rank's owned columns in `local_columns` order
    C       : m x n FP32 column-major on every rank (the assembled product)
    Returns C.  With world size 1 no collective is issued."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m, k = A.shape
    n = C.shape[1]
    layout = block_owner_layout(n, world, sub_blocks)
    gemm = gemm_fn or _cuda_gemm
    on_cuda = A.is_cuda
    comm = torch.cuda.Stream(device=A.device) if (on_cuda and world > 1) else None

    # --- A broadcast in contiguous k-chunks; sub-block 0 consumes chunks as they land ---
    kc_edges = [(k * c) // max(1, k_chunks) for c in range(max(1, k_chunks) + 1)]
    if k_chunks > 1:
        kc_edges = [min(k, (e + 127) // 128 * 128) for e in kc_edges]   # promotion-interval aligned
        kc_edges[0] = 0
    chunk_events = []
    for c in range(len(kc_edges) - 1):
        a_chunk = A[:, kc_edges[c]:kc_edges[c + 1]]
        if world > 1:
            if comm is not None:
                comm.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(comm):
                    dist.broadcast(a_chunk, src=src, group=group)
                    ev = torch.cuda.Event()
                    ev.record(comm)
                chunk_events.append(ev)
            else:
                dist.broadcast(a_chunk, src=src, group=group)
                chunk_events.append(None)
        else:
            chunk_events.append(None)

    off = 0
    for s, owners in enumerate(layout):
        st, w = owners[rank]
        Bq = B_local[:, off:off + w]
        Cq = C[:, st:st + w]
        if s == 0 and len(kc_edges) > 2 and on_cuda:
            acc = torch.empty_strided((m, w), (1, max(1, m)), dtype=torch.float32, device=A.device)
            nchunk = len(kc_edges) - 1
            for c in range(nchunk):
                if chunk_events[c] is not None:
                    torch.cuda.current_stream().wait_event(chunk_events[c])
                k0, k1 = kc_edges[c], kc_edges[c + 1]
                flags = (1 if c > 0 else 0) | (2 if c < nchunk - 1 else 0)
                gemm(A[:, k0:k1], Bq[k0:k1, :], Cq, variant, flags=flags, acc=acc)
        else:
            for ev in chunk_events:
                if ev is not None:
                    torch.cuda.current_stream().wait_event(ev)
            chunk_events = [None] * len(chunk_events)
            gemm(A, Bq, Cq, variant)
        off += w
        if world > 1:
            widths = [wq for _, wq in owners]
            lo, hi = owners[0][0], owners[-1][0] + owners[-1][1]
            if len(set(widths)) == 1 and on_cuda:
                out = C[:, lo:hi].t()            # (P*w) x m row-major view == the columns, contiguous
                inp = Cq.t()
                if comm is not None:
                    comm.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(comm):
                        dist.all_gather_into_tensor(out, inp, group=group)
                else:
                    dist.all_gather_into_tensor(out, inp, group=group)
            else:                                # ragged widths (or gloo): padded list all-gather
                wmax = max(widths)
                inp = torch.zeros((wmax, m), dtype=C.dtype, device=C.device)
                inp[:w] = Cq.t()
                parts = [torch.empty((wmax, m), dtype=C.dtype, device=C.device) for _ in widths]
                dist.all_gather(parts, inp, group=group)
                for (sq, wq), part in zip(owners, parts):
                    C[:, sq:sq + wq] = part[:wq].t()
    if comm is not None:
        torch.cuda.current_stream().wait_stream(comm)
    return C
