"""Two-sided (mailbox) halo exchange -- the message-passing comparison variant
of reference/pkg/src/diomp/apps/halo_twosided.py:12-58.

Same protocol as the reference: each rank sends its boundary slabs into
per-direction mailboxes on the neighbours (D2D puts over NVLink), completes
them, raises an 8-byte delivery tag (step+1) beside each mailbox, then waits
for the tags addressed to it and unpacks mailbox -> ghost planes with a local
device copy, and joins the group barrier.  Kept for API parity and the
code-size comparison (apps/loc.py); the fused kernel path does not use it.
"""

import struct

from ..global_memory import GlobalAddress, TransferKind

FROM_LEFT, FROM_RIGHT = 0, 1


def mailbox_bytes(halo, plane_bytes):
    """Symmetric allocation one rank needs: two slabs + two 8-byte tags."""
    return 2 * halo * plane_bytes + 16


def exchange(rt, group, u_addr, mail_addr, plane_bytes, halo, nx_local, rank, nranks, step):
    slab = halo * plane_bytes
    dev = u_addr.device
    tag = struct.pack("<q", step + 1)
    tags_at = mail_addr.offset + 2 * slab
    pending = []
    for nb, box, first_plane in ((rank - 1, FROM_RIGHT, halo), (rank + 1, FROM_LEFT, nx_local)):
        if 0 <= nb < nranks:
            h = rt.put(GlobalAddress(nb, dev, mail_addr.offset + box * slab),
                       GlobalAddress(rank, dev, u_addr.offset + first_plane * plane_bytes),
                       slab, TransferKind.D2D)
            pending.append((h, GlobalAddress(nb, dev, tags_at + 8 * box)))
    for h, tag_addr in pending:
        h.wait(rt.cfg.timeout)
        rt.put(tag_addr, tag, 8, TransferKind.H2D).wait(rt.cfg.timeout)
    for nb, box, ghost_plane in ((rank - 1, FROM_LEFT, 0), (rank + 1, FROM_RIGHT, halo + nx_local)):
        if 0 <= nb < nranks:
            at = tags_at + 8 * box
            rt.engine.wait_until(lambda at=at: rt.gm.view(dev, at, 8).tobytes() == tag,
                                 rt.cfg.timeout, "halo mailbox tag")
            rt.put(GlobalAddress(rank, dev, u_addr.offset + ghost_plane * plane_bytes),
                   GlobalAddress(rank, dev, mail_addr.offset + box * slab), slab,
                   TransferKind.D2D).wait(rt.cfg.timeout)
    rt.barrier(group)
