"""K2 tile binning through the bucket pipeline (csrc/bin_tiles.cu), shared by
the training-step executor (trainer.py) and the UDF wrappers (udf.py).

The lists equal a stable depth sort of the splat rows followed by a stable
sort by (slot, tile) ("sorts ... splats by their distance"):
per tile ascending depth, ties in row order."""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat


def bin_buckets(buf, sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams, tiles, model_id=nat.MODEL_3DGS,
                sort_cap=16384, before_sync=None, capacity_hint=None, records=None):
    """Atomics into (slot, tile) buckets, then a shared-memory sort of every
    bucket by (depth, row); buckets larger than the in-SM sort go through the
    device radix sort.  `buf` is a grow-only buffer cache with
    get(name, n, dtype).  `before_sync` (optional) queues independent GPU work
    ahead of the host read of the instance count, which it then overlaps.
    `capacity_hint` overrides the initial key-buffer size (tests of the
    overflow path).  `records` (single pass): the projection already counted
    the buckets into buf "bucket_counts" and wrote each row's tile rectangle
    (bs_proj_desc.bucket_counts / row_bin); the scatter reads those 16-byte
    records instead of the splat rows and there is no count pass.
    Returns (n_inst, inst_rows, ranges, largest bucket)."""
    st, lib = nat.stream_handle(), nat.load()
    nb = n_slots * tiles
    counts = buf.get("bucket_counts", nb, torch.int32)
    if records is None:
        nat.call("bs_bin_tiles_count", nat.ptr(sp), n_rows, nat.ptr(seg_row0), nat.ptr(seg_slot), len(seg_slot),
                 nat.ptr(slot_cams), tiles, nb, nat.ptr(counts), model_id, st)
    ranges = buf.get("ranges", nb * 2, torch.int32)
    cursor = buf.get("cursor", nb, torch.int32)
    stats = buf.get("bin_stats", 2, torch.int64)
    ows = buf.get("offsets_ws", lib.bs_bin_tiles_offsets_workspace(nb), torch.uint8)

    def offsets():
        nat.call("bs_bin_tiles_offsets", nat.ptr(counts), nb, nat.ptr(ranges), nat.ptr(cursor), nat.ptr(stats),
                 nat.ptr(ows), ows.numel(), st)

    offsets()
    # the instance count travels to the host while the GPU scatters into a
    # buffer sized from earlier steps (no idle gap at this read); on overflow
    # the offsets and the scatter run again with a larger buffer
    pin = getattr(buf, "bin_stats_pin", None)
    if pin is None:
        pin = torch.empty(2, dtype=torch.int64, pin_memory=True)
        buf.bin_stats_pin = pin
    nat.call("bs_copy_to_host", nat.ptr(stats), 16, pin.data_ptr(), st)  # by a kernel: no copy-engine queue
    ready = torch.cuda.Event()
    ready.record()
    if before_sync is not None:
        before_sync()
    # the key buffer is sized generously (6 tiles per row, or the largest
    # count seen) and the scatter may fill all of it: an overflow costs a
    # re-run and a reallocation, which at C4 sizes is milliseconds
    inst_cap = max(getattr(buf, "inst_cap", 0), 6 * n_rows, 1024) if capacity_hint is None else capacity_hint

    def scatter(capacity):
        k = buf.get("inst_keys", capacity, torch.int64)
        if capacity_hint is None:
            k = buf.bufs["inst_keys"]  # the whole cached allocation
        if records is None:
            nat.call("bs_bin_tiles_scatter", nat.ptr(sp), n_rows, nat.ptr(seg_row0), nat.ptr(seg_slot),
                     len(seg_slot), nat.ptr(slot_cams), tiles, nat.ptr(cursor), nat.ptr(k), k.numel(), model_id, st)
        else:
            nat.call("bs_bin_tiles_scatter_rec", nat.ptr(records), n_rows, nat.ptr(seg_row0), nat.ptr(seg_slot),
                     len(seg_slot), nat.ptr(slot_cams), tiles, nat.ptr(cursor), nat.ptr(k), k.numel(), st)
        return k

    keys = scatter(inst_cap)
    ready.synchronize()
    n_inst, biggest = (int(x) for x in pin.tolist())  # sizes the instance buffers
    if n_inst > keys.numel():
        inst_cap = int(n_inst * 1.25) + 1024
        offsets()
        keys = scatter(inst_cap)
    buf.inst_cap = max(getattr(buf, "inst_cap", 0), int(n_inst * 1.25) + 1024)
    irows = buf.get("irows", max(keys.numel(), 1), torch.int32)[: max(n_inst, 1)]
    cap = min(sort_cap, lib.bs_bin_tiles_max_sort())
    # no bucket exceeds `biggest`: size classes above it are not launched
    nat.call("bs_bin_tiles_sort_n", nat.ptr(keys), nat.ptr(ranges), nb, max(1, min(cap, biggest)), n_inst,
             nat.ptr(irows), st)
    if biggest > cap:  # rare: buckets beyond the shared-memory sort
        from .culling import radix_sort_u64

        rg = ranges.view(-1, 2).cpu().numpy()
        for b in np.flatnonzero(rg[:, 1] - rg[:, 0] > cap):
            s0, s1 = int(rg[b, 0]), int(rg[b, 1])
            k = keys[s0:s1]
            v = torch.empty(s1 - s0, dtype=torch.int32, device=keys.device)
            radix_sort_u64(k, v, 0, 64)
            nat.call("bs_keys_low32", nat.ptr(k), s1 - s0, nat.ptr(irows[s0:s1]), st)
    return n_inst, irows, ranges, biggest
