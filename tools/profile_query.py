"""One configs[2]-shaped query for ncu captures (tools only): synthetic DB in HBM,
the bench's planted query batch, `--queries` synchronous batch queries.

    python tools/profile_query.py [--rows 1000000] [--persons 32] [--queries 1]

Kernel order per row chunk (host issue order, which ncu serialises):
k_limb_gemm_pair (hd), k_limb_gemm_pair (ml), k_gate_keystream, k_reshare, k_lift,
k_inject, k_msb -- so `-k regex:"k_limb|k_gate|k_reshare|k_lift|k_inject|k_msb" -s 14 -c 7`
captures one steady-state chunk."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--persons", type=int, default=32)
    ap.add_argument("--queries", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2405_04463_b200 as P
    from test_full_scale import planted_query
    sess = P.Session(P.EngineConfig(backend=P.SHAMIR, l=12800, rotations=31), master_seed=7)
    sess.synth_db(a.rows, rng_seed=2, first=0, mask_density=0.9, deal_seed=7)
    codes, masks = planted_query(sess, a.rows, a.persons)
    q = [torch.empty(2 * a.persons * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 2, 0, codes, masks, q)
    for _ in range(a.queries):
        m = sess.batch_query(q, a.persons)
    torch.cuda.synchronize()
    st = sess.last_stats
    print(f"ok person0={int(m[0])} lanes={st.lanes} wall_ms={st.wall_ms:.1f} launches={st.kernel_launches}")


if __name__ == "__main__":
    main()
