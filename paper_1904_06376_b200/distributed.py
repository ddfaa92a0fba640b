"""Column-sharded multi-GPU split GEMM (north star: "partitioned across the 8 GPUs
of one box by output column blocks of C, with B sharded, A broadcast once and an NCCL
all-gather over NVLink only to reassemble C").

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.  Output columns
are independent, so the only exchanges are

  * broadcast of A (FP32, m x k, column-major with lda = m) from `src`, sent as `k_chunks`
    contiguous column chunks A[:, Kc] -- each sent as its transpose view A[:, Kc]^T, a
    row-major-contiguous (|Kc| x m) tensor over the same memory, as NCCL requires -- so the
    first sub-block's GEMM can start on chunk c while chunk c+1 is in flight.  Each rank splits
    every chunk ONCE, as it lands, into one piece buffer of the whole A in A's own layout
    (bf16x_split at column offset k0, no transpose); every GEMM of every sub-block then reads those
    pieces (bf16x_gemm_ex A_pieces with BF16X_A_PIECES_MN), so A is split exactly once per rank.  The first sub-block carries
    its FP32 promoted accumulator between chunks (bf16x_gemm_ex ACC_IN / ACC_OUT), which makes
    the chunked result bit-identical to a one-pass GEMM: chunk edges are multiples of 128 (the
    longest promotion interval), deduplicated;
  * one all-gather per sub-round of C's column blocks.  Ownership is block-cyclic: with P
    ranks and S sub-blocks of width w = n / (P*S), rank q owns blocks s*P + q, so sub-round s
    covers the contiguous column range [s*P*w, (s+1)*P*w) of C and the all-gather of C^T
    (row-major view of column-major C) writes straight into C -- no permute pass.  The
    all-gather of sub-round s runs on a side stream while sub-round s+1 computes.

Every GEMM is issued with BF16X_NO_STREAM_K, so each element depends only on its own row of A
and column of B: the assembled C equals a one-GPU bf16x_gemm_ex(..., BF16X_NO_STREAM_K) bit for
bit (tests/test_gpu_distributed.py), whatever P, S and the chunking.

There are no reductions: k is never split across GPUs.  `gemm_fn` replaces the per-rank GEMM
on FP32 operands (the CPU tests inject the oracle to exercise the partition and collective
logic with the gloo backend); by default the bf16x CUDA library runs it on pieces.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN_K = 128      # chunk edges: a multiple of every promotion interval (64 / 128 values of k)


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


def chunk_edges(k: int, k_chunks: int, align: int = ALIGN_K):
    """k-chunk boundaries of the A broadcast: k_chunks near-equal parts with interior edges
    rounded up to multiples of `align`, deduplicated (so no chunk is empty)."""
    if k_chunks <= 1 or k <= align:
        return [0, k]
    edges = {0, k}
    for c in range(1, k_chunks):
        edges.add(min(k, ((k * c) // k_chunks + align - 1) // align * align))
    return sorted(edges)


def _ld(t, rows):
    return max(1, t.stride(1) if t.shape[1] > 1 else rows)


class _PieceGemm:
    """The CUDA library path: A split once into pieces in A's own layout (MN-major, ld round_up(m, 8)),
    GEMMs on those pieces (bf16x_gemm_ex with BF16X_A_PIECES_MN)."""

    def __init__(self, A, variant):
        import paper_1904_06376_b200 as bx
        self.bx = bx
        m, k = A.shape
        self.m, self.k = m, k
        self.variant = variant
        self.pa = 2 if variant in (3, 5) else (1 if variant == 1 else 3)
        self.mp = (m + 7) // 8 * 8
        self.a_plane = self.mp * k
        self.P = torch.empty(max(1, self.pa * self.a_plane), dtype=torch.uint16, device=A.device)
        self.base = self.P.data_ptr()

    def split_chunk(self, A, k0, k1):
        """Pieces of A[:, k0:k1] into columns k0..k1 of the piece buffer."""
        if k1 <= k0 or self.m == 0:
            return
        es = 2   # bytes per piece element
        p = [self.base + (q * self.a_plane + k0 * self.mp) * es if q < self.pa else 0 for q in range(3)]
        self.bx.split_raw(self.m, k1 - k0, A.data_ptr() + k0 * A.stride(1) * 4, _ld(A, self.m), p[0], p[1], p[2],
                          self.mp)

    def gemm(self, k0, k1, Bq, Cq, flags, acc=None):
        n = Cq.shape[1]
        self.bx.gemm_raw(self.m, n, k1 - k0, 1.0, 0, self.m, Bq.data_ptr() + k0 * 4, _ld(Bq, Bq.shape[0]), 0.0,
                         Cq.data_ptr(), _ld(Cq, self.m), variant=self.variant,
                         flags=flags | self.bx.NO_STREAM_K | self.bx.A_PIECES_MN, A_pieces=self.base + k0 * self.mp * 2,
                         ldap=self.mp,
                         a_plane=self.a_plane, acc=None if acc is None else acc.data_ptr())


def gemm_colsharded(A: torch.Tensor, B_local: torch.Tensor, C: torch.Tensor, variant: int = 6,
                    group=None, src: int = 0, sub_blocks: int = 1, k_chunks: int = 1, gemm_fn=None):
    """C = A B with B's columns sharded over the ranks of `group`.

    A       : m x k FP32 column-major with lda = m (valid on `src`; overwritten by the broadcast
              elsewhere)
    B_local : k x n_q FP32 column-major, this rank's owned columns in `local_columns` order
    C       : m x n FP32 column-major on every rank (the assembled product)
    gemm_fn : None (bf16x CUDA library on pieces), or fn(A_chunk, B_chunk, C_block, variant,
              flags=0, acc=None) on FP32 operands (the CPU tests' oracle)
    Returns C.  With world size 1 no collective is issued."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m, k = A.shape
    n = C.shape[1]
    if A.numel() > 0 and not ((m <= 1 or A.stride(0) == 1) and (k <= 1 or A.stride(1) == m)):
        raise ValueError("A must be column-major with lda == m (contiguous columns)")
    layout = block_owner_layout(n, world, sub_blocks)
    on_cuda = A.is_cuda
    comm = torch.cuda.Stream(device=A.device) if (on_cuda and world > 1) else None
    cur = torch.cuda.current_stream() if on_cuda else None
    pg = _PieceGemm(A, variant) if gemm_fn is None else None

    # --- A broadcast in contiguous k-chunks (on the comm stream when there is one) ---
    edges = chunk_edges(k, k_chunks)
    nchunk = len(edges) - 1
    chunk_ready = [None] * nchunk
    for c in range(nchunk):
        a_t = A[:, edges[c]:edges[c + 1]].t()          # (|Kc| x m) row-major view of the columns
        if world > 1 and a_t.numel() > 0:
            if not a_t.is_contiguous():
                raise ValueError("A chunk view is not contiguous")
            if comm is not None:
                comm.wait_stream(cur)
                with torch.cuda.stream(comm):
                    dist.broadcast(a_t, src=src, group=group)
                    ev = torch.cuda.Event()
                    ev.record(comm)
                chunk_ready[c] = ev
            else:
                dist.broadcast(a_t, src=src, group=group)
    split_done = [False] * nchunk

    def need_chunk(c):
        if chunk_ready[c] is not None:
            cur.wait_event(chunk_ready[c])
            chunk_ready[c] = None
        if pg is not None and not split_done[c]:
            pg.split_chunk(A, edges[c], edges[c + 1])
            split_done[c] = True

    off = 0
    for s, owners in enumerate(layout):
        st, w = owners[rank]
        Bq = B_local[:, off:off + w]
        Cq = C[:, st:st + w]
        if w > 0 and m > 0:
            if s == 0 and nchunk > 1:
                acc = torch.empty_strided((m, w), (1, max(1, m)), dtype=torch.float32, device=A.device)
                for c in range(nchunk):
                    need_chunk(c)
                    k0, k1 = edges[c], edges[c + 1]
                    flags = (1 if c > 0 else 0) | (2 if c < nchunk - 1 else 0)
                    if pg is not None:
                        pg.gemm(k0, k1, Bq, Cq, flags, acc)
                    else:
                        gemm_fn(A[:, k0:k1], Bq[k0:k1, :], Cq, variant, flags=flags, acc=acc)
            else:
                for c in range(nchunk):
                    need_chunk(c)
                if pg is not None:
                    pg.gemm(0, k, Bq, Cq, 0)
                else:
                    gemm_fn(A, Bq, Cq, variant)
        else:
            for c in range(nchunk):
                need_chunk(c)
        off += w
        if world > 1:
            widths = [wq for _, wq in owners]
            lo, hi = owners[0][0], owners[-1][0] + owners[-1][1]
            if len(set(widths)) == 1:
                # equal widths: gather straight into C (its columns lo..hi are the contiguous
                # rows of the row-major view C^T)
                out = C[:, lo:hi].t()
                inp = Cq.t()
                if not (out.is_contiguous() and inp.is_contiguous()):
                    raise ValueError("C must be column-major with ldc == m")
                if comm is not None:
                    comm.wait_stream(cur)
                    with torch.cuda.stream(comm):
                        dist.all_gather_into_tensor(out, inp, group=group)
                else:
                    dist.all_gather_into_tensor(out, inp, group=group)
            else:                                # ragged widths: padded list all-gather
                if comm is not None:
                    cur.wait_stream(comm)
                wmax = max(widths)
                inp = torch.zeros((wmax, m), dtype=C.dtype, device=C.device)
                inp[:w] = Cq.t()
                parts = [torch.empty((wmax, m), dtype=C.dtype, device=C.device) for _ in widths]
                dist.all_gather(parts, inp, group=group)
                for (sq, wq), part in zip(owners, parts):
                    C[:, sq:sq + wq] = part[:wq].t()
    if comm is not None:
        cur.wait_stream(comm)
    return C
