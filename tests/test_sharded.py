"""DB-sharded queries through the C-ABI (irismpc_gpu_shard_attach_* +
irismpc_gpu_sharded_batch_query): G contexts each hold a row
range of the DB, the library broadcasts the query from shard 0, gathers the
per-person XOR-shared partials and opens on shard 0.  Here the shards are G
contexts of one process on one GPU, one host thread each, joined by an
in-process shard group (one NCCL communicator cannot hold two ranks of one
GPU; bench.py --gpus N runs the NCCL attach, one process per GPU)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2405_04463_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


def _run_threads(fns):
    out, err = [None] * len(fns), [None] * len(fns)

    def go(i):
        try:
            out[i] = fns[i]()
        except Exception as e:  # noqa: BLE001
            err[i] = e

    th = [threading.Thread(target=go, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("be,var,G,splits", [(O.SHAMIR, P.MPC_LIFT, 2, [333]), (O.REPLICATED, P.NO_LIFT, 3, [100, 512]),
                                             (O.SHAMIR, P.PLAIN_MASK, 2, [1])])
def test_sharded_batch_query_matches_oracle(be, var, G, splits):
    l, s, persons, seed = 12800, 700, 3, 43
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2 * persons, 0.9)
    qc[2], qm[2] = dc[600], dm[600]   # person 1 matches a row of the last shard
    qc[5], qm[5] = dc[0], dm[0]       # person 2 matches row 0
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)), variant=var)
    rec = O.record_bytes(be, l, var)
    bounds = [0] + splits + [s]
    cfg = P.EngineConfig(backend=be, l=l, variant=var)
    group = P.ShardGroup(G)
    shards = []
    for r in range(G):
        r0, r1 = bounds[r], bounds[r + 1]
        sh = P.Session(cfg, master_seed=seed, shard_rank=r, db_rows_total=s, db_row_offset=r0)
        sh.load_db([x[r0 * rec:r1 * rec] for x in db], r1 - r0)
        sh.shard_attach_inproc(group)
        shards.append(sh)
    qlen = [len(x) for x in q]
    outs = _run_threads([(lambda r=r: shards[r].sharded_batch_query(q if r == 0 else None, persons, qlen))
                         for r in range(G)])
    ref = O.run_local(O.make_config(be, l, variant=var), seed, dc, dm, qc, qm, persons)
    np.testing.assert_array_equal(outs[0], ref.person_match)
    assert outs[0][1] == 1 and outs[0][2] == 1
    # a second query on the same shards (device payloads on shard 0), persistent contexts
    qd = [torch.from_numpy(x).cuda() for x in q]
    outs = _run_threads([(lambda r=r: shards[r].sharded_batch_query(qd if r == 0 else None, persons, qlen))
                         for r in range(G)])
    np.testing.assert_array_equal(outs[0], ref.person_match)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_sharded_contexts_on_two_devices_one_process():
    """Two shard contexts on different GPUs of one process (per-device GEMM
    attribute / SM-count state, cross-device gather over UVA) and a plain
    single-GPU context on device 1 afterwards."""
    be, var, l, s, persons, seed = O.SHAMIR, P.MPC_LIFT, 12800, 600, 2, 47
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2 * persons, 0.9)
    qc[1], qm[1] = dc[450], dm[450]
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)), variant=var)
    rec = O.record_bytes(be, l, var)
    cfg = P.EngineConfig(backend=be, l=l, variant=var)
    group = P.ShardGroup(2)
    shards = []
    for r, (r0, r1) in enumerate([(0, 300), (300, s)]):
        sh = P.Session(cfg, master_seed=seed, device=r, shard_rank=r, db_rows_total=s, db_row_offset=r0)
        sh.load_db([x[r0 * rec:r1 * rec] for x in db], r1 - r0)
        sh.shard_attach_inproc(group)
        shards.append(sh)
    qlen = [len(x) for x in q]
    outs = _run_threads([(lambda r=r: shards[r].sharded_batch_query(q if r == 0 else None, persons, qlen))
                         for r in range(2)])
    ref = O.run_local(O.make_config(be, l, variant=var), seed, dc, dm, qc, qm, persons)
    np.testing.assert_array_equal(outs[0], ref.person_match)
    assert outs[0][0] == 1
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, device=1)
    np.testing.assert_array_equal(m, ref.person_match)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, persons), ref.agg)


def test_sharded_requires_attach_and_total_rows():
    cfg = P.EngineConfig(backend=P.SHAMIR, l=256, rotations=5)
    sh = P.Session(cfg, master_seed=1, shard_rank=1, db_rows_total=0)
    with pytest.raises(P.ConfigError):
        sh.shard_attach_inproc(P.ShardGroup(2))   # db_rows_total missing
    sh2 = P.Session(cfg, master_seed=1)
    with pytest.raises(P.ConfigError):
        sh2.sharded_batch_query([np.zeros(10, np.uint8)] * 3, 1)  # not attached


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("backend", ["shamir", "replicated"])
def test_sharded_over_nccl_two_processes(backend):
    """The same sharded query with the library's NCCL communicator, one process
    per GPU (tools/sharded_nccl.py --check); runs where >= 2 GPUs are visible."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + (backend == "shamir")),
           os.path.join(root, "tools", "sharded_nccl.py"), "--check", "--backend", backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["check"] is True and line["person_match"][0] == 1 and line["person_match"][2] == 1
