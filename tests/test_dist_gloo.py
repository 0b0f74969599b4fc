"""Multi-process (world_size 2, gloo on CPU) check of the sharded query plumbing
used by bench.py (paper_2405_04463_b200/dist.py): row-shard plan, query-payload
broadcast, all-gather of per-person XOR-shared partials and the final OR/open
on rank 0.  Each rank's shard engine is a stand-in built from the oracle's
per-lane match bits (the GPU engine itself is covered by tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as O
from paper_2405_04463_b200.dist import shard_rows, sharded_batch_query

L, S, PERSONS, ROT, SEED = 64, 37, 3, 3, 17


def _case():
    rng = O.Rng(SEED)
    dc, dm = O.records(rng, L, S, 0.85)
    qc, qm = O.records(rng, L, 2 * PERSONS, 0.85)
    qc[3], qm[3] = dc[30], dm[30]          # person 1 matches row 30 (on rank 1)
    cfg = O.make_config(O.REPLICATED, L, 0.375, ROT, debug_rows=True)
    ref = O.run_local(cfg, SEED, dc, dm, qc, qm, PERSONS)
    q = O.deal(O.REPLICATED, L, qc, qm, O.Rng(sub=(SEED, 2)))
    return ref, q


class OracleShard:
    """Stand-in shard engine: per-person OR over this shard's lanes, XOR-shared."""

    def __init__(self, row_bits, offset, rows, rank, expected_q):
        self.bits, self.offset, self.rows, self.rank, self.q = row_bits, offset, rows, rank, expected_q

    def batch_query_partial(self, qpay, persons, out):
        for a, b in zip(qpay, self.q):   # the broadcast delivered rank 0's payloads
            assert np.array_equal(a.numpy(), b)
        ncols = 2 * persons * ROT
        rng = np.random.default_rng(self.rank)
        for p in range(persons):
            b = 0
            for col in range(2 * ROT * p, 2 * ROT * (p + 1)):
                lanes = col * S + self.offset + np.arange(self.rows)
                b |= int(self.bits[lanes].any())
            if self.rank == 0:  # inner-batch pair lanes live on shard 0
                k = ncols * S
                for i in range(persons):
                    for j in range(i + 1, persons):
                        if p in (i, j):
                            b |= int(self.bits[k:k + 4 * ROT].any())
                        k += 4 * ROT
            r1, r2 = rng.integers(0, 2, 2)
            out[0, p], out[1, p], out[2, p] = b ^ r1 ^ r2, r1, r2

    def or_open(self, parts, G, persons):
        x = parts.numpy()
        return (np.bitwise_xor.reduce(x, axis=1) & 1).max(axis=0).astype(np.uint8)


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ref, q = _case()
    off, rows = shard_rows(S, world, rank)
    sess = OracleShard(ref.row_bits, off, rows, rank, q)
    qpay = [torch.from_numpy(x.copy()) if rank == 0 else torch.zeros(len(x), dtype=torch.uint8) for x in q]
    parts = torch.zeros((world, 3, PERSONS), dtype=torch.uint8)
    m = sharded_batch_query(sess, qpay, PERSONS, dist, world, rank, parts)
    if rank == 0:
        result.put((m.tolist(), ref.person_match.tolist()))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_plan_covers_rows():
    for total in (0, 1, 7, 100_000, 4_194_304):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(total, world, r) for r in range(world)]
            assert sum(n for _, n in spans) == total
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_two_rank_gloo_sharded_query():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got, want = q.get()
    assert got == want
    assert want[1] == 1
