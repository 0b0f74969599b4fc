"""Multi-GPU orchestration (one process per GPU, DB row-sharded).

The path shards naturally: DB rows are independent, and every shard holds all
three parties' shares of its rows, so reshares and AND gates stay on the
device.  The only exchanges are the two below:

1. NCCL broadcast of the three query payloads from rank 0;
2. all-gather of each shard's per-person XOR-shared OR partial
   (3 x persons bytes), followed by the MPC-OR across shards and the open at
   P1 on rank 0 (``Session.or_open``).

Partial aggregates are never opened (OpenAudit semantics, rep3.hpp:131-134).
"""
from __future__ import annotations


def shard_rows(total_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range (offset, rows) of `rank`: an even split, the first
    `total_rows % world` ranks taking one extra row."""
    base, extra = divmod(total_rows, world)
    rows = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, rows


def sharded_batch_query(sess, qpay, persons: int, dist, world: int, rank: int, parts):
    """One query over the row-sharded DB.

    sess   : this rank's ``Session`` (or any object with ``batch_query_partial`` /
             ``or_open``), created with shard_rank / db_rows_total / db_row_offset
    qpay   : three uint8 tensors (query payloads; rank 0's are broadcast)
    parts  : uint8 tensor [world, 3, persons] receiving the gathered partials
    Returns person_match (numpy) on rank 0, None elsewhere."""
    import torch

    for d in qpay:                               # (1) query-share broadcast
        dist.broadcast(d, src=0)
    if qpay[0].is_cuda:
        torch.cuda.current_stream().synchronize()
    mine = torch.empty((3, persons), dtype=torch.uint8, device=qpay[0].device)
    sess.batch_query_partial(qpay, persons, mine)
    if dist.get_backend() == "nccl":                             # (2) gather shares
        dist.all_gather_into_tensor(parts.view(-1), mine.view(-1))
    else:  # gloo (CPU tests): list all-gather
        chunks = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(chunks, mine)
        for g in range(world):
            parts[g].copy_(chunks[g])
    if qpay[0].is_cuda:
        torch.cuda.current_stream().synchronize()
    if rank == 0:
        return sess.or_open(parts, world, persons)
    return None
