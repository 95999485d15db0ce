"""Cross-rank plumbing of the distributed step (Alg. 1 lines 6-9 and 21,
PAPER.md:482-508): all-gather of the per-rank access counts C[v]_k into A,
the image-to-rank assignment W, the splat-row layouts of the all-to-all and
the two all_to_all_single exchanges (splat state forward, its gradient
backward).  Device-agnostic torch.distributed code: NCCL over NVLink on the
GPUs, gloo on CPU tensors in the multi-process tests.

Row layouts (B batch views, N ranks, A[v, k] = points of rank k visible in
view v, W[v] = rank rendering view v):
  send layout on rank k  views ordered by (W[v], v); view v holds A[v, k]
                         rows (ascending local point index) -> the chunk
                         for destination d is contiguous
  recv layout on rank k  for every source s (ascending): the views v with
                         W[v] = k (ascending), A[v, s] rows each
The backward exchange sends G_SP rows in the recv layout back to their
sources, so they land in the send layout where the projection backward
finds them by the same row index.  Split sizes follow from A alone; no
extra size exchange is needed.  With P = 1 the rows moved are exactly the
A-predicted transfers of account_iteration (simulator.py:134-183).

Asynchronous online placement:
with `prefetch`, the access counts of the NEXT batch (culled on the GPU at
the start of the current step, i.e. before its Adam update: stale by one
step, the staleness simulator.py:40-45 models) are all-gathered
asynchronously and a host thread computes its W while the GPU runs the
current step.  The next step still all-gathers its fresh counts, which fix
the split sizes; only W comes from the stale matrix, so the exchange stays
exact and the placement leaves the critical path.
"""

from __future__ import annotations

import concurrent.futures as cf
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .assign import CostCoefficients, hierarchical_place


@dataclass
class StepLayout:
    A: np.ndarray             # int64 [B, N]
    W: np.ndarray             # int64 [B]
    order: np.ndarray         # int32 [B] send-layout view order
    send_rows: list           # rows to each destination rank
    recv_rows: list           # rows from each source rank
    my_views: np.ndarray      # batch positions rendered here (ascending)
    seg_rows: np.ndarray      # int64 [n_segs] rows of each recv segment
    seg_slot: np.ndarray      # int32 [n_segs] render slot of each segment

    @property
    def n_recv(self) -> int:
        return int(sum(self.recv_rows))

    @property
    def n_send(self) -> int:
        return int(sum(self.send_rows))


def layout_for(A: np.ndarray, W: np.ndarray, rank: int) -> StepLayout:
    """Send/recv split sizes and segment tables of rank `rank`."""
    A = np.asarray(A, dtype=np.int64)
    W = np.asarray(W, dtype=np.int64)
    B, N = A.shape
    order = np.lexsort((np.arange(B), W)).astype(np.int32)
    send = [int(A[W == d, rank].sum()) for d in range(N)]
    mine = np.flatnonzero(W == rank)
    recv = [int(A[mine, s].sum()) for s in range(N)]
    seg_rows, seg_slot = [], []
    for s in range(N):
        for slot, v in enumerate(mine):
            seg_rows.append(int(A[v, s]))
            seg_slot.append(slot)
    return StepLayout(A, W, order, send, recv, mine, np.array(seg_rows, dtype=np.int64),
                      np.array(seg_slot, dtype=np.int32))


class SplatExchange:
    """Collectives of one rank; `group` defaults to the world group."""

    def __init__(self, inter_coeffs: CostCoefficients | None = None, intra_coeffs: CostCoefficients | None = None,
                 group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.inter = inter_coeffs if inter_coeffs is not None else CostCoefficients(p=4.0)
        self.intra = intra_coeffs if intra_coeffs is not None else CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1,
                                                                                    delta=1.0, p=4.0)
        self.bytes_fwd = 0
        self.bytes_bwd = 0
        # gloo (CPU tests, several ranks sharing one GPU) moves host tensors only
        self.host_staging = dist.get_backend(group) == "gloo"
        self._pool = cf.ThreadPoolExecutor(max_workers=1, thread_name_prefix="placement")
        self._ahead = {}         # batch key -> future of its W
        self.place_ms = []       # host placement time per W (ms)
        self.wait_ms = []        # time the step waited for a prefetched W (ms)
        self.prefetched = 0

    def _stage(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host_staging else t

    def gather_access(self, col: torch.Tensor) -> np.ndarray:
        """All-gather C[.]_k (int64 [B]) -> A int64 [B, N] on the host."""
        src = self._stage(col.contiguous())
        out = torch.empty(self.world * col.numel(), dtype=col.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        return out.view(self.world, -1).t().cpu().numpy().astype(np.int64)

    def _place(self, A: np.ndarray) -> np.ndarray:
        t = time.perf_counter()
        B, N = A.shape
        W = hierarchical_place(A, N, 1, self.inter, self.intra).assignment
        self.place_ms.append(1e3 * (time.perf_counter() - t))
        return W

    def assign(self, A: np.ndarray, key=None) -> np.ndarray:
        """W <- AssignImages(A): hierarchical_place on a one-box topology
        (N, 1); the W prefetched for `key` (stale by one step) when there is one."""
        fut = self._ahead.pop(key, None) if key is not None else None
        if fut is not None:
            t = time.perf_counter()
            W = fut.result()
            self.wait_ms.append(1e3 * (time.perf_counter() - t))
            self.prefetched += 1
            return W
        return self._place(A)

    def prefetch(self, col_next: torch.Tensor, key) -> None:
        """Start the all-gather of the next batch's counts and its placement
        on the host thread (collective issued here, in program order)."""
        src = self._stage(col_next.contiguous())
        out = torch.empty(self.world * col_next.numel(), dtype=col_next.dtype, device=src.device)
        work = dist.all_gather_into_tensor(out, src, group=self.group, async_op=True)
        if out.is_cuda:
            work.wait()  # stream-ordered: later work on this stream sees the result
            host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            host.copy_(out, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()

            def ready():
                ev.synchronize()
                return host
        else:
            def ready():
                work.wait()
                return out
        world = self.world

        def job():
            A = ready().view(world, -1).t().numpy().astype(np.int64)
            return self._place(A)

        for stale in list(self._ahead)[:-1]:  # keep at most two pending batches
            self._ahead.pop(stale)
        self._ahead[key] = self._pool.submit(job)

    def exchange_counts(self, counts: torch.Tensor) -> np.ndarray:
        """counts int64 [N, K] (row d: values for rank d) -> [N, K] on the host,
        row s: the values rank s addressed to this rank (one all_to_all)."""
        src = self._stage(counts.contiguous().view(-1))
        out = torch.empty_like(src)
        dist.all_to_all_single(out, src, group=self.group)
        return out.view(self.world, -1).cpu().numpy().astype(np.int64)

    def _a2a(self, send: torch.Tensor, send_rows, recv_rows, width: int) -> torch.Tensor:
        src = self._stage(send.view(-1, width))
        recv = torch.empty((int(sum(recv_rows)), width), dtype=send.dtype, device=src.device)
        dist.all_to_all_single(recv, src, output_split_sizes=list(recv_rows), input_split_sizes=list(send_rows),
                               group=self.group)
        return recv.to(send.device) if self.host_staging else recv

    def forward(self, sp_send: torch.Tensor, lay: StepLayout, width: int) -> torch.Tensor:
        """Splat state rows to the ranks that render them (line 9)."""
        remote = sum(r for d, r in enumerate(lay.send_rows) if d != self.rank)
        self.bytes_fwd += remote * width * sp_send.element_size()
        return self._a2a(sp_send, lay.send_rows, lay.recv_rows, width)

    def forward_ids(self, row_gid: torch.Tensor, lay: StepLayout) -> torch.Tensor:
        """Global point id (int32) of every row sent by forward(): the
        receiver's canonical tie order (4 B per row, counted in bytes_fwd)."""
        remote = sum(r for d, r in enumerate(lay.send_rows) if d != self.rank)
        self.bytes_fwd += remote * row_gid.element_size()
        return self._a2a(row_gid, lay.send_rows, lay.recv_rows, 1).view(-1)

    def backward(self, g_recv: torch.Tensor, lay: StepLayout, width: int) -> torch.Tensor:
        """Splat-state gradients back to the owners of the points (line 21)."""
        remote = sum(r for s, r in enumerate(lay.recv_rows) if s != self.rank)
        self.bytes_bwd += remote * width * g_recv.element_size()
        return self._a2a(g_recv, lay.recv_rows, lay.send_rows, width)
