"""DB-sharded query over the library's own NCCL communicator, one process per
GPU (torchrun), checked against the oracle on rank 0 (tools / tests only).

    torchrun --nproc-per-node G tools/sharded_nccl.py [--check]

Each rank holds a contiguous row range of one DB (all three parties' shares of
it); torch.distributed only ships the NCCL id."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--backend", default="shamir", choices=["shamir", "replicated"])
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2405_04463_b200 as P
    from oracle import pyoracle as O
    from paper_2405_04463_b200.dist import shard_rows

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    be = P.SHAMIR if a.backend == "shamir" else P.REPLICATED
    l, s, persons, seed = 12800, 1500, 3, 29
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2 * persons, 0.9)
    qc[1], qm[1] = dc[s - 3], dm[s - 3]   # person 0 matches a row of the last shard
    qc[4], qm[4] = dc[5], dm[5]           # person 2 matches a row of the first shard
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)))
    rec = O.record_bytes(be, l)
    off, rows = shard_rows(s, world, rank)
    sess = P.Session(P.EngineConfig(backend=be, l=l), master_seed=seed, device=local, shard_rank=rank,
                     db_rows_total=s, db_row_offset=off)
    sess.load_db([x[off * rec:(off + rows) * rec] for x in db], rows)
    idl = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(idl, src=0)
    sess.shard_attach_nccl(idl[0], world)
    qlen = [len(x) for x in q]
    m = sess.sharded_batch_query(q if rank == 0 else None, persons, qlen)
    qd = [torch.from_numpy(x).cuda() for x in q] if rank == 0 else None
    m2 = sess.sharded_batch_query(qd, persons, qlen)
    # streaming: three queries, two in flight (every collective stream-ordered)
    tk = [sess.sharded_batch_query_submit(qd, persons, qlen)]
    tk.append(sess.sharded_batch_query_submit(qd, persons, qlen))
    ms = [sess.batch_query_wait(tk[0])]
    tk.append(sess.sharded_batch_query_submit(qd, persons, qlen))
    ms += [sess.batch_query_wait(tk[1]), sess.batch_query_wait(tk[2])]
    if rank == 0:
        out = {"world": world, "person_match": [int(x) for x in m]}
        if a.check:
            ref = O.run_local(O.make_config(be, l), seed, dc, dm, qc, qm, persons)
            out["check"] = bool(np.array_equal(m, ref.person_match) and np.array_equal(m2, ref.person_match) and
                                all(np.array_equal(x, ref.person_match) for x in ms))
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
