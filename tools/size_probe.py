"""Runs synthetic batch queries at a list of (rows, persons) sizes; prints ok/error per size."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_04463_b200 as P

L = 12800
for spec in sys.argv[1:]:
    s, persons = map(int, spec.split("x"))
    try:
        sess = P.Session(P.EngineConfig(backend=P.SHAMIR, l=L), master_seed=7)
        sess.synth_db(s)
        codes = torch.empty((2 * persons, L // 64), dtype=torch.int64, device="cuda")
        masks = torch.empty_like(codes)
        sess.synth_records(2, s, 2 * persons, 0.9, codes, masks)
        q = [torch.empty(2 * persons * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
        sess.deal_payload(7, 2, 0, codes, masks, q)
        m = sess.batch_query(q, persons)
        st = sess.last_stats
        print(spec, "ok", m.sum(), f"wall {st.wall_ms:.2f} gemm {st.gemm_ms:.2f} thr {st.threshold_ms:.2f} or {st.or_ms:.2f} prep {st.prep_ms:.2f}", flush=True)
        sess.close()
    except Exception as e:
        print(spec, "ERROR", e, flush=True)
        break
