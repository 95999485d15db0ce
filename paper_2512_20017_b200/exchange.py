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


class _Dev:
    """A raw device pointer where the C ABI wrappers expect a tensor."""

    def __init__(self, p: int):
        self.p = int(p)

    def data_ptr(self) -> int:
        return self.p


class PeerExchange(SplatExchange):
    """The two all-to-alls of the step through peer memory (csrc/peer.cu)
    instead of a collective library: every rank exports one device block
    (flags, splat-row receive buffer, global-id receive buffer, G_SP home
    buffer) over CUDA IPC and maps the others' blocks; the projection writes
    each splat row straight into the renderer's receive buffer
    (bs_proj_desc.view_sp / view_gid), bs_return_rows writes each gradient
    row straight into its owner's home buffer, and completion travels as
    stream-ordered flags (bs_stream_signal / bs_stream_wait, epoch per
    step).  Between GPUs the loads/stores run over NVLink / NVSwitch; ranks
    sharing one GPU (tests) map each other's memory the same way.  The host
    plumbing (access counts, IPC handles) stays on torch.distributed.

    Buffer sizes follow from A and W, which every rank holds, so a
    reallocation is decided identically everywhere (a collective step)."""

    peer = True

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        import ctypes

        from . import _native as nat

        self._nat, self._ct = nat, ctypes
        self.lib = nat.load()
        self.epoch = 0
        self.cap_recv = [0] * self.world   # rows each rank's receive buffer holds
        self.cap_home = [0] * self.world   # rows each rank's G_SP home buffer holds
        self.widths = None
        self.base = None                   # own block
        self.peers = [None] * self.world   # mapped blocks (own at [rank])
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.ok, self.why = self._preflight()

    @classmethod
    def create(cls, *args, **kw) -> "SplatExchange":
        """A PeerExchange when every rank can map every other rank's memory
        and its stream-ordered flag writes land (checked collectively by
        `_preflight`), else the collective SplatExchange."""
        ex = cls(*args, **kw)
        if ex.ok:
            return ex
        import warnings

        warnings.warn(f"peer-memory exchange unavailable ({ex.why}); using all-to-all collectives")
        return SplatExchange(*args, **kw)

    def _preflight(self):
        """Collective check: map every peer's block, write a flag into it
        from this rank's stream, read the own flags back on the host.  Any
        failure on any rank -> every rank falls back (no device-side wait is
        issued, so nothing can hang)."""
        ct, nat = self._ct, self._nat
        ok, why, base, opened = 1, "", None, []
        try:
            hb = int(self.lib.bs_ipc_handle_bytes())
            p = ct.c_void_p()
            handle = (ct.c_uint8 * hb)()
            nat.call("bs_ipc_alloc", 4 * self.world, ct.byref(p), handle)
            base = p.value
        except Exception as e:  # noqa: BLE001
            ok, why, handle = 0, f"alloc: {e}", None
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle) if handle is not None else None, group=self.group)
        if ok and any(h is None for h in handles):
            ok, why = 0, "a peer could not allocate"
        peers = [None] * self.world
        if ok:
            try:
                st = torch.cuda.current_stream().cuda_stream
                for r in range(self.world):
                    if r == self.rank:
                        peers[r] = base
                        continue
                    q = ct.c_void_p()
                    nat.call("bs_ipc_open", (ct.c_uint8 * hb).from_buffer_copy(handles[r]), ct.byref(q))
                    peers[r] = q.value
                    opened.append(q.value)
                for r in range(self.world):
                    if r != self.rank:
                        nat.call("bs_stream_signal", st, peers[r] + 4 * self.rank, 1234567)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                ok, why = 0, f"map/signal: {e}"
        dist.barrier(group=self.group)
        if ok:
            try:
                # the own flag words, copied on the device and read on the host
                tmp = torch.empty(self.world, dtype=torch.int32, device=self.dev)
                idx = torch.zeros(1, dtype=torch.int64, device=self.dev)
                nat.call("bs_gather_rows", base, self.world, nat.ptr(idx), 1, nat.ptr(tmp),
                         torch.cuda.current_stream().cuda_stream)
                got = tmp.cpu().numpy()
                if any(int(got[s]) != 1234567 for s in range(self.world) if s != self.rank):
                    ok, why = 0, "flag writes did not land"
            except Exception as e:  # noqa: BLE001
                ok, why = 0, f"read back: {e}"
        flag = torch.tensor([ok], dtype=torch.int32)
        if dist.get_backend(self.group) != "gloo":
            flag = flag.to(self.dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for q in opened:
            try:
                nat.call("bs_ipc_close", q)
            except Exception:  # noqa: BLE001
                pass
        if base is not None:
            nat.call("bs_ipc_free", base)
        if int(flag.item()) == 0 and ok:
            why = "a peer failed the check"
        return bool(int(flag.item())), why

    # block layout: [fwd flags N u32 | bwd flags N u32 | pad to 256 B] [sp rows] [gid] [gsp home]
    def _offsets(self, cap_r, cap_h):
        spf, gspf = self.widths
        o_sp = 256
        o_gid = o_sp + ((cap_r * spf * 4 + 255) // 256) * 256
        o_gsp = o_gid + ((cap_r * 4 + 255) // 256) * 256
        end = o_gsp + cap_h * gspf * 4
        return o_sp, o_gid, o_gsp, max(end, 512)

    def _ensure(self, need_recv, need_home, sp_floats, gsp_floats):
        if (self.widths == (sp_floats, gsp_floats) and all(n <= c for n, c in zip(need_recv, self.cap_recv))
                and all(n <= c for n, c in zip(need_home, self.cap_home))):
            return
        # identical decision on every rank; nobody may still use the old blocks
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self._release()
        self.widths = (sp_floats, gsp_floats)
        self.cap_recv = [max(int(n * 1.25) + 1024, c) for n, c in zip(need_recv, self.cap_recv)]
        self.cap_home = [max(int(n * 1.25) + 1024, c) for n, c in zip(need_home, self.cap_home)]
        ct, nat = self._ct, self._nat
        hb = int(self.lib.bs_ipc_handle_bytes())
        size = self._offsets(self.cap_recv[self.rank], self.cap_home[self.rank])[3]
        p = ct.c_void_p()
        handle = (ct.c_uint8 * hb)()
        nat.call("bs_ipc_alloc", size, ct.byref(p), handle)
        self.base = p.value
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        for r in range(self.world):
            if r == self.rank:
                self.peers[r] = self.base
            else:
                q = ct.c_void_p()
                nat.call("bs_ipc_open", (ct.c_uint8 * hb).from_buffer_copy(handles[r]), ct.byref(q))
                self.peers[r] = q.value
        self.epoch = 0  # fresh zeroed flags
        dist.barrier(group=self.group)

    def _release(self):
        if self.base is None:
            return
        for r, p in enumerate(self.peers):
            if p is not None and r != self.rank:
                self._nat.call("bs_ipc_close", p)
        self._nat.call("bs_ipc_free", self.base)
        self.base, self.peers = None, [None] * self.world

    def _flag(self, rank, kind, src):
        return self.peers[rank] + 4 * (kind * self.world + src)

    def plan(self, lay: StepLayout, sp_floats: int, gsp_floats: int):
        """Per-step plan from A and W: capacities, per-view destination
        pointers of this rank's rows, the return segments of the rows it
        renders.  Returns the device arrays the kernels read."""
        A, W, N, me = lay.A, lay.W, self.world, self.rank
        B = A.shape[0]
        need_recv = [int(A[W == d].sum()) for d in range(N)]
        need_home = [int(A[:, s].sum()) for s in range(N)]
        self._ensure(need_recv, need_home, sp_floats, gsp_floats)
        self.epoch += 1
        offs = [self._offsets(self.cap_recv[r], self.cap_home[r]) for r in range(N)]
        # receive layout of rank d: sources ascending, then its views ascending
        view_sp = np.zeros(B, dtype=np.int64)
        view_gid = np.zeros(B, dtype=np.int64)
        for v in range(B):
            d = int(W[v])
            mine_d = np.flatnonzero(W == d)
            before = int(A[mine_d, :me].sum()) + int(A[mine_d[mine_d < v], me].sum())
            view_sp[v] = self.peers[d] + offs[d][0] + before * sp_floats * 4
            view_gid[v] = self.peers[d] + offs[d][1] + before * 4
        # send layout of every source s: views ordered by (W, v)
        order = np.lexsort((np.arange(B), W))
        row0 = np.zeros((N, B), dtype=np.int64)
        for s in range(N):
            acc = 0
            for v in order:
                row0[s, v] = acc
                acc += int(A[v, s])
        seg_src, seg_dst0 = [], []
        for s in range(N):
            for v in lay.my_views:
                seg_src.append(s)
                seg_dst0.append(int(row0[s, v]))
        dst = np.array([self.peers[r] + offs[r][2] for r in range(N)], dtype=np.int64)
        host = np.concatenate([view_sp, view_gid, dst, np.asarray(seg_dst0, dtype=np.int64),
                               np.asarray(seg_src, dtype=np.int64)])
        # kernel-parameter upload (bs_upload): no stream synchronisation per
        # step; two alternating buffers, as a step's plan may still be read
        # by the previous step's kernels when the next one is queued
        self._plan_k = 1 - getattr(self, "_plan_k", 0)
        bufs = getattr(self, "_plan_bufs", [None, None])
        if bufs[self._plan_k] is None or bufs[self._plan_k].numel() < host.size:
            bufs[self._plan_k] = torch.empty(max(host.size, 256), dtype=torch.int64, device=self.dev)
        self._plan_bufs = bufs
        dev = self._nat.upload(host.astype(np.int64), bufs[self._plan_k][: host.size])
        n_segs = len(seg_src)
        return {"view_sp": dev[:B], "view_gid": dev[B:2 * B], "dst": dev[2 * B:2 * B + N],
                "seg_dst0": dev[2 * B + N:2 * B + N + n_segs],
                "seg_src": dev[2 * B + N + n_segs:].to(torch.int32),
                "sp_recv": _Dev(self.base + offs[me][0]), "gid_recv": _Dev(self.base + offs[me][1]),
                "gsp_home": _Dev(self.base + offs[me][2]), "n_segs": n_segs}

    def _signal_all(self, kind, st):
        for d in range(self.world):
            if d != self.rank:
                self._nat.call("bs_stream_signal", st, self._flag(d, kind, self.rank), self.epoch)

    def _wait_all(self, kind, st):
        for s in range(self.world):
            if s != self.rank:
                self._nat.call("bs_stream_wait", st, self._flag(self.rank, kind, s), self.epoch)

    def forward_done(self, lay: StepLayout, sp_floats: int, st) -> None:
        """After the projection wrote every row into its renderer's buffer:
        tell every rank, then wait until every rank's rows for this one are in."""
        remote = sum(r for d, r in enumerate(lay.send_rows) if d != self.rank)
        self.bytes_fwd += remote * (sp_floats + 1) * 4
        self._signal_all(0, st)
        self._wait_all(0, st)

    def backward_done(self, lay: StepLayout, wire: int, st) -> None:
        remote = sum(r for s, r in enumerate(lay.recv_rows) if s != self.rank)
        self.bytes_bwd += remote * wire * 4
        self._signal_all(1, st)
        self._wait_all(1, st)

    def close(self):
        if self.base is not None:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
            self._release()
