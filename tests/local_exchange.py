"""Test-only exchange: every rank's handle in one process ("virtual shards" on one GPU).

The collectives of paper_2111_04289_b200.dist's protocol (watermark MAX/MIN all-reduce, LR1
count SUM all-reduce, owner all-to-all) done with plain torch device ops across the handles of
one process, so that the protocol's kernels can be checked on a single GPU.  Not part of the
product (tests/ only).
"""
from __future__ import annotations

from paper_2111_04289_b200.dist import ROW_BYTES


class LocalExchange:
    """All ranks' handles in one process (virtual shards on one GPU)."""

    def setup_p2p(self, handles, device_watermark: bool = False):
        for h in handles:
            for o in handles:
                h.p2p_import_local(o)
        if device_watermark:
            for h in handles:
                h.p2p_device_watermark(True)

    def barrier(self, handles):
        pass                        # pushes are synchronous: nothing in flight

    def allreduce_watermarks(self, handles):
        import torch
        torch.cuda.synchronize()
        wms, tss = zip(*(h.watermark_tensors() for h in handles))
        wm = torch.stack(list(wms)).max(0).values
        ts = torch.stack(list(tss)).min(0).values
        for a, b in zip(wms, tss):
            a.copy_(wm)
            b.copy_(ts)
        torch.cuda.synchronize()

    def allreduce_sum(self, handles, tensors):
        import torch
        torch.cuda.synchronize()
        tot = torch.stack(list(tensors)).sum(0, dtype=tensors[0].dtype)
        for t in tensors:
            t.copy_(tot)
        torch.cuda.synchronize()

    def allreduce_dense(self, handles, arrays):
        import torch
        torch.cuda.synchronize()
        for i in range(2):
            tot = torch.stack([a[i] for a in arrays]).sum(0, dtype=arrays[0][i].dtype)
            for a in arrays:
                a[i].copy_(tot)
        torch.cuda.synchronize()

    def all_to_all(self, handles, sends):
        import torch
        world = len(handles)
        out = []
        for d in range(world):
            parts = []
            for rows, counts in sends:
                off = sum(counts[:d]) * ROW_BYTES
                parts.append(rows[off:off + counts[d] * ROW_BYTES])
            out.append(torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize()
        return out
